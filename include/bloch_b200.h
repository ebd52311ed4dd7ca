/*
 * bloch_b200.h — C-ABI of libbloch_b200.so, the sm_100a Bloch event-stream engine.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (pure Python, /root/reference/pkg/src/mrsim) has no FFI of its own; the seam
 * it exposes — and that its tests monkeypatch (tests/test_engine.py:214-222) —
 * is
 *
 *     engine.compute_block(tables: OperatorTables, block: SpinBlock)
 *         -> (echoes complex128 (n_acq, max_ns), [snapshot (n,3) f64 | None])
 *                                                   (engine.py:259-310)
 *
 * fed by the master precompute engine.precompute_sequence_tables
 * (engine.py:83-164) and folded by engine.run / _run_pool (engine.py:465-595).
 * The entry points below replace exactly that seam; the ctypes binding that
 * the reference side would add is shown in INTEGRATION.md.
 *
 *   reference                                     this ABI
 *   --------------------------------------------  --------------------------------
 *   OperatorTables / EsTable (engine.py:51-80)    bloch_set_tables()
 *   compute_block (engine.py:259-310)             bloch_compute_block()
 *   worker exception -> WorkerPanic               status < 0 + bloch_last_error()
 *     (engine.py:455-459, 575-577; errors.py:57)
 *   InvalidParameter (engine.py:467-473)          BLOCH_E_INVALID
 *
 * Conventions: plain pointers and sizes only; every call returns an int
 * status (0 = ok, < 0 = error) and leaves a thread-local message readable via
 * bloch_last_error().  A context is bound to one CUDA device and is not
 * re-entrant: serialise calls per context.  The caller owns every buffer it
 * passes; the context owns only its scratch (compiled program, staged spins,
 * partial k-space) and retains no caller pointer past a call.
 */
#ifndef BLOCH_B200_H
#define BLOCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLOCH_ABI_VERSION 1

/* status codes */
#define BLOCH_OK 0
#define BLOCH_E_INVALID -1 /* bad argument          -> mrsim InvalidParameter      */
#define BLOCH_E_CUDA -2    /* CUDA error / no device -> mrsim WorkerPanic          */
#define BLOCH_E_STATE -3   /* call out of order (e.g. compute before set_tables)  */
#define BLOCH_E_NOMEM -4   /* device allocation failed                            */

/* precision of the per-spin state inside the kernel */
#define BLOCH_PREC_F32 32 /* fp64 spin state and phases; fp32 ADC sample sums (tensor cores) (default) */
#define BLOCH_PREC_F64 64 /* fp64 everywhere, sample sums included (the reference's 1e-12 unit tests) */

/* bloch_compute_block flags */
#define BLOCH_IN_DEVICE 1u  /* spin arrays are device pointers (else host)          */
#define BLOCH_OUT_DEVICE 2u /* echoes/snapshot outputs are device pointers (else host) */
#define BLOCH_NO_SYNC 4u    /* return without synchronising the stream; with host buffers they must be
                               pinned and stay untouched until bloch_synchronize (pipelined callers) */

typedef struct bloch_ctx bloch_ctx;

/* Library / ABI identification. */
const char* bloch_version(void);
int bloch_abi_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* bloch_last_error(void);
/* Number of visible CUDA devices (0 when none; status BLOCH_E_CUDA if the driver fails). */
int bloch_device_count(int* out);

/* pseudo-device of a compile-only context (no CUDA calls; set_tables / program_stats only) */
#define BLOCH_HOST_ONLY -1

/* Create a context on `device` (or BLOCH_HOST_ONLY) with state precision BLOCH_PREC_F32 / _F64. */
int bloch_create(int device, int precision, bloch_ctx** out);
int bloch_destroy(bloch_ctx* ctx);

/*
 * A device set (the reference's domain decomposition over spins, engine.py:229-251 and
 * 540-595, across the GPUs of one box, from one host thread).  The context holds one sub-context per
 * device, in rank order.  bloch_set_tables compiles the program once per device; bloch_compute_block
 * (host spin arrays only) cuts the block into contiguous shards with np.linspace bounds — rank r takes
 * [floor(r n/k), floor((r+1) n/k)) exactly as partition_blocks — evolves them concurrently, each on its
 * own device and stream, copies each shard's final magnetisation rows into place (rank order is the
 * reference's block order, engine.py:497-504) and performs the one exchange: every partial k-space is
 * pulled to the first device (peer copies over NVLink/NVSwitch) and summed there in rank order in fp64
 * (the reference's ordered fold, engine.py:493-496, 594-595).  Outputs are host buffers, or device
 * buffers on the first device.  Listing a device twice is allowed (two shards on one GPU).
 */
int bloch_create_multi(const int32_t* devices, int32_t n_devices, int precision, bloch_ctx** out);
/* Devices of a context (1 for a single-device context); `devices` may be NULL or hold n entries. */
int bloch_device_count_of(const bloch_ctx* ctx, int32_t* n_devices, int32_t* devices);
/* Per-device integrator and whole-call device time (ms) of the last synchronous call, rank order:
 * `capacity` entries at most (the reference's per-worker busy time, engine.py:516-525). */
int bloch_last_device_times(const bloch_ctx* ctx, int32_t capacity, float* kernel_ms, float* device_ms);
/* Stream used for all work of this context (a cudaStream_t; NULL = context-owned). */
int bloch_set_stream(bloch_ctx* ctx, void* stream);

/*
 * Upload the event tables of one sequence — the flattened OperatorTables.
 * For elementary sequence i (0 <= i < n_es) its events are
 * [es_ev_offset[i], es_ev_offset[i+1]) of the ev_* arrays (EsTable.ev_*,
 * engine.py:51-70); es_has_pulse[i] != 0 means EsTable.pulse_mat is the 3x3
 * row-major matrix at es_pulse_mat + 9*i; es_acq[i] is EsTable.acq (-1 when
 * the ES does not acquire).  The library compiles the stream into its device
 * program (rotations, generic intervals, uniform ADC windows).
 */
int bloch_set_tables(bloch_ctx* ctx, int32_t n_es, const int64_t* es_ev_offset,
                     const uint8_t* es_has_pulse, const double* es_pulse_mat,
                     const int32_t* es_acq, const double* ev_dt, const double* ev_dmom,
                     const uint8_t* ev_sample, const int32_t* ev_snap, int32_t n_acq,
                     int32_t max_samples, int32_t n_snap);

/* Statistics of the compiled program: events E (reference table size incl.
 * pulses), ADC samples, pulses, generic intervals (evaluated one by one),
 * uniform ADC windows and the samples they cover, samples covered by
 * linear-increment (chirp) runs, and pulse+interval pairs folded into RF
 * trains.  Any pointer may be NULL. */
int bloch_program_stats(const bloch_ctx* ctx, int64_t* n_events, int64_t* n_samples,
                        int64_t* n_rot, int64_t* n_interval, int64_t* n_window_ops,
                        int64_t* n_window_samples, int64_t* n_chirp_samples,
                        int64_t* n_train_pairs);

/* Layout of the compiled program: ops in the device stream, rotation classes
 * (tabulated per-spin propagators), relax classes (tabulated exponentials), and
 * intervals evaluated on the fly (unique intervals after fusion). */
int bloch_program_layout(const bloch_ctx* ctx, int64_t* n_ops, int64_t* n_rot_classes,
                         int64_t* n_relax_classes, int64_t* n_onthefly_intervals);

/* Per-spin class tables of the compiled program (all tabulated once per call by
 * small fp64 kernels before the integrator): progression classes (arithmetic
 * series of interval moments), chirp classes (reused trapezoid ramps under the
 * ADC), train classes (reused RF trains, composed into one affine propagator per
 * spin) and the RF-train ops that use them; planes (the distinct per-spin class
 * quantities, 16 B per spin each).  Any pointer may be NULL. */
int bloch_program_classes(const bloch_ctx* ctx, int64_t* n_prog_classes, int64_t* n_chirp_classes,
                          int64_t* n_train_classes, int64_t* n_train_class_ops, int64_t* n_planes);

/*
 * Evolve one spin block through the uploaded tables — compute_block.
 *
 *   n        spins in the block (SpinBlock.n, engine.py:187-189); n >= 0
 *   pos      n*3 float64, row-major (SpinBlock.pos)
 *   mx,my,mz,t1,t2,m0,domega   n float64 each (SpinBlock fields)
 *   weight   complex128 interleaved (re, im): n_coils*n*2 doubles laid out
 *            [coil][spin]; NULL means the uniform weight 1+0j (n_coils = 1)
 *   echoes_out  n_coils * n_acq * max_samples complex128 (interleaved),
 *            un-normalised partial sums exactly as compute_block returns them
 *            (the caller divides by the global spin count, engine.py:507)
 *   snaps_out   n_snap * n * 3 float64, or NULL
 *   snap_present n_snap bytes set to 1 where the snapshot was taken, or NULL
 *   flags    BLOCH_IN_DEVICE / BLOCH_OUT_DEVICE / BLOCH_NO_SYNC
 */
int bloch_compute_block(bloch_ctx* ctx, int64_t n, const double* pos, const double* mx,
                        const double* my, const double* mz, const double* t1,
                        const double* t2, const double* m0, const double* domega,
                        const double* weight, int32_t n_coils, double* echoes_out,
                        double* snaps_out, uint8_t* snap_present, uint32_t flags);

/*
 * Device-side object model — replaces the host
 * rasterisation feeding compute_block: phantom.rasterize (phantom.py:98-142),
 * the per-spin fold of engine.build_spin_arrays (engine.py:192-226) with
 * system.spin_off_resonance (system.py:123-132) and complex_weight
 * (system.py:203-211).  Spins are produced directly in device memory in the
 * reference's order (box, then z, y, x with x fastest; sites whose M0 is zero
 * emit no spin), ready for bloch_compute_block(..., BLOCH_IN_DEVICE).
 *
 * Tissue of a box: the constants m0/t1/t2/dw, overridden inside each of its
 * shapes [shape_begin, shape_begin+shape_count) — later shapes win (label
 * maps; the seeded ellipse phantoms of the benchmark configs).  A shape is an
 * ellipse (ax[2] <= 0: z ignored) or ellipsoid rotated by angle a in the
 * x-y plane; a site is inside when u^2 + v^2 (+ w^2) <= 1 with
 * u = (dx cos a + dy sin a)/ax[0], v = (-dx sin a + dy cos a)/ax[1], w = dz/ax[2].
 */
typedef struct {
  double base[3];    /* first lattice site per axis: origin + (size - (n-1)*spacing)/2 */
  double step[3];    /* lattice spacing per axis (m); site k sits at base + step*k */
  int64_t count[3];  /* lattice sites per axis (phantom._lattice) */
  double m0, t1, t2, dw; /* background tissue of the box */
  int32_t shape_begin, shape_count;
} bloch_box_t;

typedef struct {
  double c[3], ax[3];  /* centre and semi-axes (m) */
  double cos_a, sin_a; /* in-plane rotation */
  double m0, t1, t2, dw;
} bloch_shape_t;

/* Off-resonance map added to the tissue dw (rad/s), evaluated per spin:
 *   dw += const_dw
 *       + poly_scale * sum_k coef_k * (x/s)^px_k * (y/s)^py_k * (z/s)^pz_k
 *       + sum_j amp_j * exp(-|r - c_j|^2 / (2 sigma_j^2))     (bumps; 2-D when c_j[2] is NaN)
 * poly_peak > 0 rescales the polynomial so its peak |value| over the emitted
 * spins equals poly_peak (poly_scale is then ignored). */
typedef struct {
  double const_dw;
  int32_t n_poly, n_bumps;
  const double* poly;  /* n_poly x 4: coef, px, py, pz */
  double poly_len;     /* s */
  double poly_scale, poly_peak;
  const double* bumps; /* n_bumps x 5: cx, cy, cz, sigma, amp */
} bloch_field_t;

/* Receive coils: n_coils Gaussian coils (centre, sigma, azimuth phase), or
 * n_coils = 0 for the uniform sensitivity S (weight S + 0j). */
typedef struct {
  double c[3], sigma, cos_p, sin_p;
} bloch_coil_t;

/*
 * Rasterise onto `ctx`'s device and stream.  Outputs are device pointers with
 * room for `capacity` spins (the lattice site total bounds the spin count):
 * pos capacity*3, mx/my/mz/t1/t2/m0/domega capacity each, weight
 * max(n_coils,1)*capacity*2 doubles.  The first *n_out entries are written,
 * weight as [coil][spin] interleaved complex with coil stride *n_out — the
 * layout bloch_compute_block reads.  Host pointers (poly, bumps, boxes,
 * shapes, coils) are read during the call only.  The call synchronises the
 * stream once (to learn the spin count).  BLOCH_E_INVALID when the sites
 * exceed `capacity` or an emitted tissue value is invalid (m0 < 0,
 * T1/T2 <= 0), as phantom.rasterize / RelaxationParams reject them.
 */
int bloch_rasterize(bloch_ctx* ctx, const bloch_box_t* boxes, int32_t n_boxes,
                    const bloch_shape_t* shapes, int32_t n_shapes, const bloch_field_t* field,
                    const bloch_coil_t* coils, int32_t n_coils, double uniform_s, int64_t capacity,
                    double* pos, double* mx, double* my, double* mz, double* t1, double* t2,
                    double* m0, double* domega, double* weight, int64_t* n_out);

/* Wait for all work of this context (e.g. a BLOCH_NO_SYNC call's host outputs). */
int bloch_synchronize(bloch_ctx* ctx);

/* Order this context's integrator after another context's (pipelined callers): before its
 * integrator kernel the context waits on `wait_event` (a cudaEvent_t, or NULL), after it it records
 * `signal_event` (or NULL).  Uploads and downloads stay free to overlap; the kernels serialise. */
int bloch_set_kernel_gate(bloch_ctx* ctx, void* wait_event, void* signal_event);

/* Device time (ms, CUDA events on the context stream) of the last
 * bloch_compute_block: kernel_ms = from the first integrator launch to the end of the
 * last main kernel (the integrator; with the window contraction, through the last
 * contraction fold; with a segmented program it also spans the folds and state
 * hand-overs between the segments' launches), and device_ms = all device work of the
 * call (staging kernels + integrator + contraction + reduction).  bloch_last_phases
 * splits kernel_ms into the integrator and the contraction. */
int bloch_last_timing(const bloch_ctx* ctx, float* kernel_ms, float* device_ms,
                      int32_t* kernel_launches);

/* Shape of the last integrator launch (all 0 before the first): arithmetic precision (32 / 64 bits),
 * spins per thread, coil-group width, grid (CTAs) and threads per CTA.  Chosen per call from the block
 * size, the coil count and the program (>= 16 warps per SM when the block allows). */
int bloch_last_launch(const bloch_ctx* ctx, int32_t* prec, int32_t* spins_per_thread, int32_t* coils,
                      int32_t* grid, int32_t* threads);

/* Program segments of the last call.  The integrator keeps one partial-sum row per warp and
 * recorded sample; when that would exceed BLOCH_PARTIAL_BUDGET_MB (default 24 GiB) the op stream
 * runs as several launches over contiguous op ranges, the fp64 state handed over through global
 * memory and each range's samples folded before the next: the results are bit-identical. */
int bloch_last_segments(const bloch_ctx* ctx, int32_t* segments);

/* Window contraction (fp32 mode, one receive coil; replaces the per-sample weighted sum of
 * engine.py:303-305 for long tabulated windows).  The uniform ADC windows of one rotation class
 * share the per-sample factor z of every spin, so their samples are one complex product over the
 * spins, S[w][k] = sum_s U[w][s] z_s^k: the integrator stores each window's entry magnetisation U
 * and the product runs on the tensor cores (tcgen05, TMEM accumulators; three bf16 passes).
 * `enable` = 0 keeps every window in the integrator (per-warp sums).  Default: enabled. */
int bloch_set_contraction(bloch_ctx* ctx, int32_t enable);

/* Resident-table integrator (fp32 mode, every window contracted, RF trains tabulated): the per-spin
 * class tables of a CTA's spins stay in shared memory for the whole launch, one spin per thread, so
 * each table value crosses L2 once per call instead of once per op (the reference's relax cache,
 * engine.py:292-299, generalised and held on chip).  `enable` = 0 keeps integrate_kernel, which reads
 * the tables through L2 at every op.  Default: enabled; programs it does not cover (on-the-fly
 * chirps, generic sampled events, in-kernel windows, tables beyond 227 KB per 128 spins) fall back. */
int bloch_set_resident(bloch_ctx* ctx, int32_t enable);

/* Whether the last bloch_compute_block ran the resident-table integrator, and the bytes of class
 * tables per spin of the current program's resident plan (0: the program is not covered). */
int bloch_last_resident(const bloch_ctx* ctx, int32_t* resident, int32_t* bytes_per_spin);

/* The compiled program's window groups (one contraction each), the samples they produce and the
 * samples the integrator still sums itself when the contraction runs (host-only contexts too). */
int bloch_program_groups(const bloch_ctx* ctx, int32_t* n_groups, int64_t* contracted_samples,
                         int64_t* integrator_samples);

/* The compiled op stream (diagnostics): for op i < min(n_ops, capacity) of the plain (deferred = 0) or
 * deferred-window (deferred = 1) program, its kind (program.h OpKind), sample count / flags, rotation /
 * chirp / train class, progression class, fused pulse and its four plane ids (pl: 4 per op).  Any
 * output may be NULL; *n_ops receives the op count. */
int bloch_program_ops(const bloch_ctx* ctx, int32_t deferred, int32_t capacity, int32_t* n_ops, int32_t* kind,
                      int32_t* count, int32_t* rot, int32_t* prg, int32_t* pre, int32_t* pl);

/* Phases of the last bloch_compute_block (ms, CUDA events): the integrator launches with their
 * fold, and the window contractions with theirs; the window groups contracted and the samples they
 * produced (0 when the call ran without the contraction). */
int bloch_last_phases(const bloch_ctx* ctx, float* integrate_ms, float* contract_ms, int32_t* n_groups,
                      int64_t* contracted_samples);


#ifdef __cplusplus
}
#endif

#endif /* BLOCH_B200_H */
