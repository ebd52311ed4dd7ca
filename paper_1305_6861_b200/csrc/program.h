// Device program of the Bloch event-stream engine (shared by the host
// compiler, program.cpp, and the kernels, bloch_kernels.cu).
//
// The reference walks OperatorTables.entries in Python (engine.py:276-308):
// per elementary sequence an optional 3x3 pulse (277-283), then per event an
// optional precession+relaxation (288-302), an optional ADC sample (303-305)
// and an optional snapshot (306-308).  The compiler flattens that walk into a
// linear op stream whose control flow is uniform across a CTA:
//
//   OP_ROT     hard pulse, 3x3 rotation                    (engine.py:277-283)
//   OP_EVENT   one interval: precession (+ relaxation when dt != 0), then an
//              optional snapshot                            (engine.py:286-302, 306-308)
//   OP_GSAMP   1..8 consecutive intervals each followed by an ADC sample, with
//              per-event (dt, dmom) from the side table     (engine.py:286-305)
//   OP_WINDOW  a uniform ADC window: an optional leading no-op sample followed
//              by `count - lead` identical (dt, dmom) intervals each followed
//              by a sample — the ES-level hoisting the reference's relax cache
//              (engine.py:292-299) only does for the exponentials
//   OP_CHIRP   `count` sampled intervals of equal dt whose moment increments
//              grow linearly (dmom_k = dmom_0 + k*dd): trapezoid ramps under
//              the ADC (sequence.py:106-116); the per-event rotation factors
//              form a geometric progression
//   OP_RFTRAIN `count` consecutive elementary sequences each made of a hard
//              pulse (or none) and one identical interval: a discretised
//              shaped pulse under a constant gradient (sequence.py:650-674);
//              matrices in the side table at `aux`
//
// The per-spin state is fp64 in every precision mode; in the fp32 mode only
// the ADC sample recurrence of OP_WINDOW runs in fp32.
//
// Relaxation factors are looked up, not evaluated: every distinct interval
// length T (an event's dt, or a whole window's nrot*dt) is a "relax class";
// a prep kernel tabulates exp(-T/T1), exp(-T/T2) per (class, spin) once per
// call — the reference's relax_cache keyed on dt (engine.py:272, 292-299).
#pragma once
#include <stdint.h>

namespace bloch {

enum OpKind : int32_t {
  OP_ROT = 1, OP_EVENT = 2, OP_GSAMP = 3, OP_WINDOW = 4, OP_CHIRP = 5, OP_RFTRAIN = 6, OP_UWIN = 7, OP_UCHIRP = 8
};
// OP_UCHIRP (deferred-window program): a tabulated OP_CHIRP whose samples u r0^(k+1) q^(k(k+1)/2) are formed
// by the contraction; the integrator stores u = w m in U row `s0` and applies the run's closed form (pl[2],
// pl[3]).  A generic sampled interval of one sample (OP_GSAMP, count 1) becomes a one-sample OP_UWIN.
// OP_UWIN (the deferred-window program, Program::dops): a tabulated OP_WINDOW whose samples are formed
// afterwards by the tensor-core contraction (contract.h).  The integrator stores the window's entry
// magnetisation u = Cpre m (times z without a leading no-op sample) as bf16 hi/lo words in U row `s0`
// and applies the window's exit propagator (C, (A, B)); `aux`, `pre`, `tmode`, `rot`, `pl` as OP_WINDOW.

// flags of an interval (OP_EVENT.count, GEv.flags)
enum : int32_t { EV_MOVE = 1, EV_RELAX = 2 };

struct alignas(16) DevOp {
  int32_t kind;
  int32_t count;  // WINDOW/CHIRP: samples; GSAMP: events (1..8); RFTRAIN: pairs; EVENT: EV_* flags
  int32_t s0;     // WINDOW/GSAMP/CHIRP: compact index of the first recorded sample
  int32_t aux;    // WINDOW: lead flag; GSAMP: first GEv; RFTRAIN: first matrix; EVENT: snapshot or -1
  double p[9];    // ROT: row-major matrix; EVENT/WINDOW/RFTRAIN: dt, dmx, dmy, dmz;
                  // CHIRP: dt, dmom_0 (3), dd (3)
  int32_t flags;  // RFTRAIN: EV_* flags of the shared interval
  int32_t cls;    // relax class of dt (EVENT/CHIRP/RFTRAIN on-the-fly path), -1 = no relaxation
  int32_t rot;    // rotation class (EVENT: repeated interval; WINDOW: reused run), chirp class (CHIRP),
                  // train class (RFTRAIN), -1 = none
  int32_t prg;    // EVENT: progression class (interval of an arithmetic series of moments), -1 = none
  int32_t pre;    // EVENT/WINDOW: hard pulse applied first (matrix index into mats, fused OP_ROT), -1 = none
  int32_t tmode;  // RFTRAIN: 1 = every sub-pulse rotates about x (real envelope); EVENT/WINDOW: axis of `pre` (1 x, 2 y, 0 general);
                  // CHIRP: 1 = the q plane holds conj(q)
  int32_t pl[4];  // per-spin planes (PlaneDesc) of the op's class, see assign_planes() in program.cpp:
                  //   EVENT rot: C, AB; EVENT prg: running factor, q, q^2, AB;
                  //   WINDOW rot: Cpre, z, C, AB; CHIRP: r0, q, C_total, AB_total
};

// A rotation class: pre, then `mult` times main, then post (intervals (dt,
// dmom)).  The prep kernel tabulates per spin the closed-form propagators
//   Cpre = e2(pre) exp(-i theta_pre)                 (state at the first sample)
//   C    = exp(-T/T2) exp(-i (theta_pre + mult theta + theta_post)),
//   mz -> A mz + B, A = exp(-T/T1), B = m0 (1 - A),  T = total duration
//   z    = e2(main) exp(-i theta)                    (per-sample factor)
struct alignas(16) RotClass {
  double pre[4];   // (dt, dmx, dmy, dmz) applied once before the run (WINDOW: before the samples)
  double main[4];  // the repeated interval
  double mult;     // repetitions of `main`
  double post[4];  // applied once after the run
  double pad[3];
};
static_assert(sizeof(RotClass) == 128, "RotClass must be 128 bytes");
static_assert(sizeof(DevOp) == 128, "DevOp must be 128 bytes");

// A progression class: intervals of equal dt whose moments form an arithmetic
// series in op order, dmom_j = d0 + j*step (phase-encode lobes, blips).  Per
// spin the factor of occurrence j is C0 q^j: one complex multiply per
// occurrence instead of a sincos.
struct alignas(16) ProgClass {
  double dt, d0[3], step[3];
  double pad;
};
static_assert(sizeof(ProgClass) == 64, "ProgClass must be 64 bytes");

// A chirp class: a reused OP_CHIRP run (trapezoid ramp under the ADC): dt and
// the increments dmom_k = d0 + k*dd.  Per spin the table holds
//   r0 = e2 exp(-i th_0), q = exp(-i th_dd), q^8 (one chunk ahead), A = e1, B = m0 (1 - e1).
struct alignas(16) ChirpClass {
  double dt, d0[3], dd[3];
  double pad;
};
static_assert(sizeof(ChirpClass) == 64, "ChirpClass must be 64 bytes");

// A train class: a reused OP_RFTRAIN run (the same shaped pulse under the same
// gradient, e.g. every line's slice-selective excitation).  Per spin the table
// holds the whole train's affine propagator m -> A m + b (A row-major 3x3, then
// b): 12 doubles, composed in fp64 by train_table_kernel from the same sub-pulse
// matrices and interval the on-the-fly path applies one by one.
struct alignas(16) TrainClass {
  int32_t aux;    // first matrix of the run in the side table
  int32_t count;  // sub-pulse + interval pairs
  int32_t flags;  // EV_* flags of the shared interval
  int32_t pad0;
  double p[4];    // dt, dmx, dmy, dmz of the shared interval
  double pad[2];
};
static_assert(sizeof(TrainClass) == 64, "TrainClass must be 64 bytes");
constexpr int kTrainRow = 12;  // doubles per (train class, spin)

// A plane: one complex (double2) value per spin, tabulated once per call by
// plane_kernel.  Every class quantity above (a rotation class's Cpre, C, z and
// (A, B); a progression's running factor, q, q^2, (A, B); a chirp's r0, q,
// whole-run propagator and (A, B)) is a plane, and identical planes are stored
// once: e.g. the (A, B) of every interval of the same length, the q of ramps of
// opposite slope (conjugates), the Cpre of every window without a pre-interval.
// Each op reads exactly the planes it needs, coalesced (consecutive spins,
// consecutive 16 B), and the shared planes stay in L2.
//   PL_PHASE: exp(-T/T2) exp(-i (pos . d + dw tw))  (x w, the single-coil receive weight, if PL_WEIGHT)
//   PL_AB:    (exp(-T/T1), m0 (1 - exp(-T/T1)))
enum : int32_t { PL_PHASE = 1, PL_AB = 2 };
// PL_SAMPLE: the plane only feeds fp32 ADC samples (a window's Cpre and z, a chirp's r0 and q); in
// the fp32 mode it is stored as float2 (the kernel converts it to fp32 anyway): half the bytes.
enum : int32_t { PL_WEIGHT = 1, PL_MUTABLE = 2, PL_SAMPLE = 4 };
struct alignas(16) PlaneDesc {
  int32_t kind, flags;
  double T, d[3], tw;
  double pad[2];
};
static_assert(sizeof(PlaneDesc) == 64, "PlaneDesc must be 64 bytes");

struct alignas(16) GEv {  // one generic sampled interval
  double dt, dmx, dmy, dmz;
  int32_t flags;
  int32_t cls;  // relax class of dt, -1 = none
  int32_t pad[2];
};
static_assert(sizeof(GEv) == 48, "GEv must be 48 bytes");

constexpr int kChunkSlots = 8;   // ADC slots reduced per warp transpose (samples x coils)
constexpr int kMinWindow = 4;    // shortest uniform run compiled as OP_WINDOW
constexpr int kMinChirp = 3;     // shortest linear-increment run compiled as OP_CHIRP
constexpr int kMinTrain = 4;     // shortest pulse+interval run compiled as OP_RFTRAIN
constexpr int kMmaMinWindow = 32;  // fp32 windows this long run on the tensor cores (shorter: the recurrence)
constexpr int kMinDeferWindow = 16;    // tabulated windows this long are deferred to the contraction (OP_UWIN)
constexpr int kMaxDeferWindow = 4096;  // ... up to this long (contract.h kContractMaxSamples)

// The windows of one rotation class (same z plane, same sample count) contracted as one product
// (contract.h): U rows [row0, row0 + n_windows) in op order.
struct WinGroup {
  int32_t zplane;     // plane id of the per-sample factor z (a chirp's r0)
  int32_t count;      // samples per window
  int32_t row0;       // first U row
  int32_t n_windows;  // windows (U rows)
  int32_t chirp;      // 1: chirp group, sample k = u r0^(k+1) q^(k(k+1)/2)
  int32_t qplane;     // chirp: plane of q (pure gradient phase, canonical sign)
  int32_t qconj;      // chirp: q is the conjugate of the plane
};
constexpr int kMaxDeferChirp = 64;  // chirps this long at most (k(k+1)/2 times a 12-bit phase head stays exact)
constexpr int kMinDeferGroup = 16;  // short runs (chirps, single samples) are deferred in groups this large

}  // namespace bloch
