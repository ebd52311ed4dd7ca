// C-ABI of libbloch_b200.so — see include/bloch_b200.h for the contract and the
// reference interfaces each entry point replaces.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <cmath>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/bloch_b200.h"
#include "resident.h"
#include "contract.h"
#include "kernels.h"
#include "program_host.h"
#include "raster.h"

#ifndef BLOCH_VERSION_STRING
#define BLOCH_VERSION_STRING "bloch_b200 0.1.0 (sm_100a)"
#endif

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArg : std::runtime_error {
  explicit InvalidArg(const std::string& m) : std::runtime_error(m) {}
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// bumped whenever any device buffer is (re)allocated: a captured CUDA graph holds raw pointers into
// the context's scratch buffers, so a graph recorded before a reallocation must never be replayed
std::atomic<uint64_t> g_alloc_gen{0};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes <= cap) return p;
    g_alloc_gen.fetch_add(1);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (bytes == 0) return nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      p = nullptr;
      throw CudaError(std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
    cap = bytes;
    return p;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct bloch_ctx {
  int device = 0;
  int precision = BLOCH_PREC_F32;
  int n_sm = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // call start, kernels start/end, call end, integrator end
  bloch::Program prog;
  bool has_prog = false;
  std::vector<uint8_t> snap_present;
  DevBuf d_ops, d_gev, d_mats, d_sample_g, d_relax_t, d_planes, d_train_cls;
  DevBuf in_pos, in_mx, in_my, in_mz, in_t1, in_t2, in_m0, in_dw, in_w;
  DevBuf sc, wpad, w32;
  DevBuf partial, echo, snaps, relax, planetab, planetab32, traintab;
  // window contraction (contract.h): deferred-window program, U rows, split-K partials
  DevBuf d_dops, d_dsample_g, d_urow_out0, uhi, ulo, cpart, ztab, zqtab;
  bool contraction = true;
  // resident-table integrator (resident.h): the deferred program with the class tables in shared memory
  bloch::ResidentPlan rplan;
  DevBuf d_rops, d_rloads, d_rmats, d_rmats4;
  bool resident = true;
  int32_t last_resident = 0;  // the last call ran resident_integrate_kernel
  float integrate_ms = 0.f, contract_ms = 0.f;
  int32_t last_groups = 0;
  int64_t last_csamples = 0;

  DevBuf raster_scratch;
  std::vector<unsigned char> raster_staging;
  float kernel_ms = 0.f, device_ms = 0.f;
  int launches = 0;
  int last_launch[5] = {0, 0, 0, 0, 0};  // prec, spins per thread, coils, grid, threads of the last integrator
  int32_t last_segments = 0;               // program segments of the last call (bounded partial rows)
  DevBuf state;                            // segment hand-over state, two (mx, my, mz) sets
  // CUDA graph of the device work of a device-resident call (prep, tables, integrator, fold),
  // captured on the second identical call and replayed while the arguments stay the same
  uint64_t prog_gen = 0;
  struct GraphKey {
    int64_t n = -1;
    const void* p[12] = {};
    int32_t n_coils = 0;
    uint32_t flags = 0;
    uint64_t gen = 0;
    uint64_t alloc = 0;  // g_alloc_gen: no buffer reallocated since
    cudaStream_t st = nullptr;
    bool operator==(const GraphKey& o) const {
      if (n != o.n || n_coils != o.n_coils || flags != o.flags || gen != o.gen || alloc != o.alloc || st != o.st)
        return false;
      for (int i = 0; i < 12; ++i)
        if (p[i] != o.p[i]) return false;
      return true;
    }
  } last_key, graph_key;
  cudaGraphExec_t graph_exec = nullptr;
  int graph_launches = 0;
  cudaEvent_t gate_wait = nullptr, gate_signal = nullptr;  // bloch_set_kernel_gate
  // device-set context (bloch_create_multi): one sub-context per device, in rank order; this context's
  // own device / stream (the first device's) runs the cross-device reduction
  std::vector<bloch_ctx*> subs;
  std::vector<DevBuf> sub_echo, sub_snap;  // each sub-context's partial echoes / snapshots, on its device
  std::vector<cudaEvent_t> sub_done;       // recorded on each sub-context's stream after its work
  DevBuf gather;                           // [n_sub][len] partial echoes on the first device
  std::vector<float> sub_kernel_ms, sub_device_ms;
  void drop_graph() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
    graph_key = GraphKey{};
    last_key = GraphKey{};
  }
};

namespace {

struct Variant {
  int prec, S, NC;
  bool full = true;  // program uses RF trains / chirps / generic sampled events
  bool win = true;   // program has (non-deferred) OP_WINDOW ops
};

// a contiguous op range and the contiguous compact samples it records
struct Segment {
  int32_t op_begin, op_end;
  int64_t sample_begin, n_samples;
};

int64_t op_samples(const bloch::DevOp& op) {
  switch (op.kind) {
    case bloch::OP_WINDOW:
    case bloch::OP_CHIRP:
    case bloch::OP_GSAMP:
      return op.count;
    default:
      return 0;
  }
}

int64_t partial_budget_bytes() {
  static const int64_t budget = [] {
    const char* e = getenv("BLOCH_PARTIAL_BUDGET_MB");
    const double mb = e ? atof(e) : 24.0 * 1024.0;
    return std::max<int64_t>(1, static_cast<int64_t>(mb * 1048576.0));
  }();
  return budget;
}

// integrator / contraction split of the last call's kernel time (events 1 -> 4 -> 2)
void phase_times(bloch_ctx* c) {
  float a = 0.f, b = 0.f;
  if (cudaEventElapsedTime(&a, c->ev[1], c->ev[4]) != cudaSuccess) a = 0.f;
  if (cudaEventElapsedTime(&b, c->ev[4], c->ev[2]) != cudaSuccess) b = 0.f;
  cudaGetLastError();
  c->integrate_ms = a;
  c->contract_ms = c->last_groups > 0 ? b : 0.f;
}

// Cut the program so that each segment's partial rows (bytes_per_sample per recorded sample) stay
// within the budget: BLOCH_PARTIAL_BUDGET_MB, default 24 GiB.  Samples are contiguous in op order
// (compact ids follow the walk), so a segment is an op range plus a sample range.  An op is never
// split; one op larger than the budget gets a segment of its own.
std::vector<Segment> plan_segments(const std::vector<bloch::DevOp>& ops, int64_t bytes_per_sample) {
  const int64_t budget = partial_budget_bytes();
  const int64_t cap = std::max<int64_t>(1, budget / std::max<int64_t>(1, bytes_per_sample));
  std::vector<Segment> segs;
  Segment cur{0, 0, 0, 0};
  int64_t next_sample = 0;
  for (int32_t o = 0; o < static_cast<int32_t>(ops.size()); ++o) {
    const int64_t k = op_samples(ops[o]);
    if (k > 0 && cur.n_samples > 0 && cur.n_samples + k > cap) {
      cur.op_end = o;
      segs.push_back(cur);
      cur = Segment{o, o, next_sample, 0};
    }
    if (k > 0 && cur.n_samples == 0) cur.sample_begin = ops[o].s0;
    cur.n_samples += k;
    next_sample = cur.sample_begin + cur.n_samples;
  }
  cur.op_end = static_cast<int32_t>(ops.size());
  segs.push_back(cur);
  return segs;
}

// pick (S, NC) for a block of n spins with ncp (power-of-two) coils.  win: the program keeps windows (or
// chirps / generic samples) in the integrator; plane_bytes: the per-spin class tables (planes) of the call.
Variant pick_variant(int prec, int64_t n, int ncp, int n_sm, bool win, int64_t plane_bytes) {
  if (prec == BLOCH_PREC_F32) {
    static const int force_s = [] {  // experiment hook: BLOCH_F32_SPINS=1|2|4|8
      const char* e = getenv("BLOCH_F32_SPINS");
      return e ? atoi(e) : 0;
    }();
    if (ncp == 1) {
      if (force_s == 1 || force_s == 2 || force_s == 4 || force_s == 8) return {32, force_s, 1};
      // One wave of 2 CTAs x 320 threads per SM at the smallest S that holds the block, then one step
      // down when the planes overflow L2: two waves of S = 4 keep each wave's planes in L2.  Measured
      // with the contraction (kernel ms, profiles/r2t_spins_sweep.txt), S = 8 / 4 / 2 / 1:
      //   config 2 (749k, 204 MB of planes)   11.52 / 10.40 / 12.86 / 12.81
      //   config 1 (698k,  89 MB)              3.27 /  3.56 /  4.14 /  4.00
      //   config 2 / 4 (187k)                  4.57 /  3.41 /  2.93 /  4.04;  / 8: 3.53 / 2.60 / 2.14 / 2.01
      //   config 1 / 4 (174k)                  1.67 /  1.20 /  1.05 /  1.43;  / 8: 1.33 / 0.99 / 0.83 / 0.76
      // A program that keeps windows / chirps in the integrator (config 3) carries the window stage
      // (less L1): one step more spins per thread, config 3 / 4 S = 4 1.94 vs S = 2 2.40, / 8 S = 2 1.26.
      const int64_t wave = int64_t(n_sm) * 2 * 320;
      int s = 1;
      while (s < 8 && n > wave * s) s <<= 1;
      if (win && s < 8) s <<= 1;
      if (s == 8 && n * plane_bytes > (int64_t(100) << 20)) s = 4;
      return {32, s, 1};
    }
    if (ncp == 8) {
      // eight coils carry 4x the accumulators per spin, so fewer warps already saturate: measured
      // (contraction on) config 4 (274k) S=4 7.87 vs S=2 8.14 ms; / 2 S=2 4.15 vs S=4 4.52;
      // / 4 S=1 2.37 vs S=2 2.57; / 8 S=1 1.56 vs S=2 1.66
      if (force_s == 1 || force_s == 2 || force_s == 4) return {32, force_s, 8};
      if (n < int64_t(n_sm) * 16 * 32) return {32, 1, 8};
      return {32, n >= int64_t(n_sm) * 8 * 32 * 4 ? 4 : 2, 8};
    }
    return {32, 4, ncp};
  }
  switch (ncp) {
    case 1: return {64, n >= int64_t(n_sm) * 4 * 64 ? 4 : 1, 1};
    case 2: return {64, 2, 2};
    case 4: return {64, 2, 4};
    default: return {64, 1, 8};
  }
}

template <typename R, int S, int NC>
void shape_one(const Variant& v, int* max_t, int* min_b) {
  if (v.prec == int(8 * sizeof(R)) && v.S == S && v.NC == NC) {
    *max_t = v.win ? bloch::KernelTraits<R, S, NC>::kMaxThreads : bloch::KernelTraits<R, S, NC>::kMaxThreadsNoWin;
    *min_b = v.win ? bloch::KernelTraits<R, S, NC>::kMinBlocks : bloch::KernelTraits<R, S, NC>::kMinBlocksNoWin;
  }
}

// max threads per CTA and resident CTAs per SM of a variant
void variant_shape(const Variant& v, int* max_t, int* min_b) {
  *max_t = 512;
  *min_b = 1;
#define BLOCH_SHAPE(R, S, NC) shape_one<R, S, NC>(v, max_t, min_b);
  BLOCH_FOR_EACH_VARIANT(BLOCH_SHAPE)
#undef BLOCH_SHAPE
}

template <typename R, int S, int NC>
cudaError_t dispatch_one(const Variant& v, const bloch::KParams& kp, int grid, int threads,
                         cudaStream_t st, bool* matched) {
  if (v.prec == int(8 * sizeof(R)) && v.S == S && v.NC == NC) {
    *matched = true;
    return bloch::launch_integrate<R, S, NC>(kp, grid, threads, st, v.full, v.win);
  }
  return cudaSuccess;
}

cudaError_t dispatch(const Variant& v, const bloch::KParams& kp, int grid, int threads,
                     cudaStream_t st) {
  bool matched = false;
  cudaError_t e = cudaSuccess;
#define BLOCH_DISPATCH(R, S, NC) \
  if (!matched && e == cudaSuccess) e = dispatch_one<R, S, NC>(v, kp, grid, threads, st, &matched);
  BLOCH_FOR_EACH_VARIANT(BLOCH_DISPATCH)
#undef BLOCH_DISPATCH
  if (!matched) throw InvalidArg("no kernel variant for the requested precision/coils");
  return e;
}

void upload(DevBuf& b, const void* src, size_t bytes, cudaStream_t st) {
  b.ensure(bytes);
  if (bytes) ck(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, st), "H2D");
}

}  // namespace

namespace {
// an error during capture: end it (discarding the partial graph) so the stream is usable again
void abandon_capture(bloch_ctx* c) {
  cudaGraph_t g = nullptr;
  cudaStreamEndCapture(c->stream, &g);
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  c->drop_graph();
}
}  // namespace

extern "C" {

const char* bloch_version(void) { return BLOCH_VERSION_STRING; }
int bloch_abi_version(void) { return BLOCH_ABI_VERSION; }
const char* bloch_last_error(void) { return g_err.c_str(); }

int bloch_device_count(int* out) {
  if (!out) return fail(BLOCH_E_INVALID, "out is NULL");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    *out = 0;
    return BLOCH_OK;
  }
  if (e != cudaSuccess) return fail(BLOCH_E_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  *out = n;
  return BLOCH_OK;
}

int bloch_create(int device, int precision, bloch_ctx** out) {
  if (!out) return fail(BLOCH_E_INVALID, "out is NULL");
  *out = nullptr;
  if (precision != BLOCH_PREC_F32 && precision != BLOCH_PREC_F64)
    return fail(BLOCH_E_INVALID, "precision must be 32 or 64");
  if (device == BLOCH_HOST_ONLY) {  // compile-only context: no CUDA calls at all
    bloch_ctx* c = new bloch_ctx();
    c->device = BLOCH_HOST_ONLY;
    c->precision = precision;
    *out = c;
    return BLOCH_OK;
  }
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(BLOCH_E_CUDA, "no CUDA device available (the Bloch engine has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(BLOCH_E_INVALID, "device index out of range");
  bloch_ctx* c = new bloch_ctx();
  try {
    c->device = device;
    c->precision = precision;
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10)
      throw CudaError("device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                      "; this library is built for sm_100a only");
    c->n_sm = prop.multiProcessorCount;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->own_stream = true;
    for (auto& ev : c->ev) ck(cudaEventCreate(&ev), "cudaEventCreate");
  } catch (const std::exception& ex) {
    bloch_destroy(c);
    return fail(BLOCH_E_CUDA, ex.what());
  }
  *out = c;
  return BLOCH_OK;
}

int bloch_destroy(bloch_ctx* c) {
  if (!c) return BLOCH_OK;
  if (c->device == BLOCH_HOST_ONLY) {
    delete c;
    return BLOCH_OK;
  }
  for (size_t i = 0; i < c->subs.size(); ++i) {
    cudaSetDevice(c->subs[i]->device);
    if (i < c->sub_echo.size()) c->sub_echo[i].release();
    if (i < c->sub_snap.size()) c->sub_snap[i].release();
    if (i < c->sub_done.size() && c->sub_done[i]) cudaEventDestroy(c->sub_done[i]);
    bloch_destroy(c->subs[i]);
  }
  c->subs.clear();
  cudaSetDevice(c->device);
  c->gather.release();
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  c->drop_graph();
  for (DevBuf* b : {&c->d_ops, &c->d_gev, &c->d_mats, &c->d_sample_g, &c->d_relax_t, &c->relax, &c->d_planes, &c->planetab, &c->planetab32, &c->in_pos, &c->in_mx, &c->in_my, &c->in_mz,
                    &c->in_t1, &c->in_t2, &c->in_m0, &c->in_dw, &c->in_w, &c->sc, &c->wpad, &c->w32, &c->partial,
                    &c->echo, &c->snaps, &c->d_train_cls, &c->traintab, &c->state, &c->d_dops, &c->d_dsample_g,
                    &c->d_urow_out0, &c->uhi, &c->ulo, &c->cpart, &c->ztab, &c->zqtab, &c->d_rops, &c->d_rloads, &c->d_rmats, &c->d_rmats4,
                    &c->raster_scratch})
    b->release();
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return BLOCH_OK;
}

int bloch_set_stream(bloch_ctx* c, void* stream) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->subs.empty()) return fail(BLOCH_E_STATE, "a device-set context owns one stream per device");
  if (c->device == BLOCH_HOST_ONLY) return fail(BLOCH_E_STATE, "host-only context has no stream");
  cudaSetDevice(c->device);
  c->drop_graph();
  if (c->own_stream && c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(BLOCH_E_CUDA, cudaGetErrorString(e));
    c->own_stream = true;
  }
  return BLOCH_OK;
}

int bloch_set_tables(bloch_ctx* c, int32_t n_es, const int64_t* es_ev_offset,
                     const uint8_t* es_has_pulse, const double* es_pulse_mat, const int32_t* es_acq,
                     const double* ev_dt, const double* ev_dmom, const uint8_t* ev_sample,
                     const int32_t* ev_snap, int32_t n_acq, int32_t max_samples, int32_t n_snap) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (n_es < 0) return fail(BLOCH_E_INVALID, "n_es < 0");
  if (n_es > 0 && (!es_ev_offset || !es_has_pulse || !es_pulse_mat || !es_acq))
    return fail(BLOCH_E_INVALID, "NULL elementary-sequence array");
  const int64_t E = n_es > 0 ? es_ev_offset[n_es] : 0;
  if (E > 0 && (!ev_dt || !ev_dmom || !ev_sample || !ev_snap))
    return fail(BLOCH_E_INVALID, "NULL event array");
  for (bloch_ctx* sub : c->subs) {  // a device-set context: every device gets the program
    const int st = bloch_set_tables(sub, n_es, es_ev_offset, es_has_pulse, es_pulse_mat, es_acq, ev_dt, ev_dmom,
                                    ev_sample, ev_snap, n_acq, max_samples, n_snap);
    if (st != BLOCH_OK) {
      c->has_prog = false;
      return st;
    }
  }
  bloch::TablesView tv{n_es, es_ev_offset, es_has_pulse, es_pulse_mat, es_acq, ev_dt,
                       ev_dmom, ev_sample, ev_snap, n_acq, max_samples, n_snap};
  try {
    bloch::Program prog;
    bloch::compile_program(tv, prog);
    if (c->device != BLOCH_HOST_ONLY) {
      ck(cudaSetDevice(c->device), "cudaSetDevice");
      upload(c->d_ops, prog.ops.data(), prog.ops.size() * sizeof(bloch::DevOp), c->stream);
      upload(c->d_gev, prog.gev.data(), prog.gev.size() * sizeof(bloch::GEv), c->stream);
      upload(c->d_mats, prog.mats.data(), prog.mats.size() * sizeof(double), c->stream);
      upload(c->d_relax_t, prog.relax_t.data(), prog.relax_t.size() * sizeof(double), c->stream);
      upload(c->d_planes, prog.planes.data(), prog.planes.size() * sizeof(bloch::PlaneDesc), c->stream);
      upload(c->d_train_cls, prog.train_classes.data(), prog.train_classes.size() * sizeof(bloch::TrainClass),
             c->stream);
      upload(c->d_sample_g, prog.sample_g.data(), prog.sample_g.size() * sizeof(int64_t), c->stream);
      upload(c->d_dops, prog.dops.data(), prog.dops.size() * sizeof(bloch::DevOp), c->stream);
      upload(c->d_dsample_g, prog.dsample_g.data(), prog.dsample_g.size() * sizeof(int64_t), c->stream);
      upload(c->d_urow_out0, prog.urow_out0.data(), prog.urow_out0.size() * sizeof(int64_t), c->stream);
    }
    bloch::resident_compile(prog, c->rplan);
    if (getenv("BLOCH_RESIDENT_DEBUG"))
      for (const bloch::WinGroup& g : prog.groups)
        fprintf(stderr, "group: chirp %d samples %d windows %d row0 %d\n", g.chirp, g.count, g.n_windows, g.row0);
    if (c->device != BLOCH_HOST_ONLY) {
      if (c->rplan.ok) {
        upload(c->d_rops, c->rplan.rops.data(), c->rplan.rops.size() * sizeof(bloch::ROp), c->stream);
        upload(c->d_rloads, c->rplan.loads.data(), c->rplan.loads.size() * sizeof(bloch::RLoad), c->stream);
        upload(c->d_rmats, c->rplan.mats.data(), c->rplan.mats.size() * sizeof(double), c->stream);
        upload(c->d_rmats4, c->rplan.mats4.data(), c->rplan.mats4.size() * sizeof(double), c->stream);
      }
      ck(cudaStreamSynchronize(c->stream), "set_tables sync");
    }
    c->snap_present.assign(static_cast<size_t>(n_snap), 0);
    for (const auto& op : prog.ops)
      if (op.kind == bloch::OP_EVENT && op.aux >= 0) c->snap_present[op.aux] = 1;
    c->prog = std::move(prog);
    c->has_prog = true;
    c->prog_gen++;
  } catch (const std::invalid_argument& ex) {
    c->has_prog = false;
    return fail(BLOCH_E_INVALID, std::string("invalid tables: ") + ex.what());
  } catch (const std::exception& ex) {
    c->has_prog = false;
    return fail(BLOCH_E_CUDA, ex.what());
  }
  return BLOCH_OK;
}

int bloch_program_stats(const bloch_ctx* c, int64_t* n_events, int64_t* n_samples, int64_t* n_rot,
                        int64_t* n_interval, int64_t* n_window_ops, int64_t* n_window_samples,
                        int64_t* n_chirp_samples, int64_t* n_train_pairs) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->has_prog) return fail(BLOCH_E_STATE, "no tables uploaded");
  if (n_events) *n_events = c->prog.n_events;
  if (n_samples) *n_samples = c->prog.n_samples;
  if (n_rot) *n_rot = c->prog.n_rot;
  if (n_interval) *n_interval = c->prog.n_interval + c->prog.n_gsamp_events;  // generic intervals
  if (n_window_ops) *n_window_ops = c->prog.n_window_ops;
  if (n_window_samples) *n_window_samples = c->prog.n_window_samples;
  if (n_chirp_samples) *n_chirp_samples = c->prog.n_chirp_samples;
  if (n_train_pairs) *n_train_pairs = c->prog.n_train_pairs;
  return BLOCH_OK;
}

int bloch_program_layout(const bloch_ctx* c, int64_t* n_ops, int64_t* n_rot_classes, int64_t* n_relax_classes,
                         int64_t* n_onthefly_intervals) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->has_prog) return fail(BLOCH_E_STATE, "no tables uploaded");
  int64_t otf = 0;
  for (const auto& op : c->prog.ops)
    if (op.kind == bloch::OP_EVENT && op.rot < 0 && op.prg < 0 && (op.count & bloch::EV_MOVE)) otf++;
  if (n_ops) *n_ops = static_cast<int64_t>(c->prog.ops.size());
  if (n_rot_classes) *n_rot_classes = static_cast<int64_t>(c->prog.rot_classes.size());
  if (n_relax_classes) *n_relax_classes = static_cast<int64_t>(c->prog.relax_t.size());
  if (n_onthefly_intervals) *n_onthefly_intervals = otf;
  return BLOCH_OK;
}

int bloch_program_classes(const bloch_ctx* c, int64_t* n_prog_classes, int64_t* n_chirp_classes,
                          int64_t* n_train_classes, int64_t* n_train_class_ops, int64_t* n_planes) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->has_prog) return fail(BLOCH_E_STATE, "no tables uploaded");
  if (n_prog_classes) *n_prog_classes = static_cast<int64_t>(c->prog.prog_classes.size());
  if (n_chirp_classes) *n_chirp_classes = static_cast<int64_t>(c->prog.chirp_classes.size());
  if (n_train_classes) *n_train_classes = static_cast<int64_t>(c->prog.train_classes.size());
  if (n_train_class_ops) *n_train_class_ops = c->prog.n_train_class_ops;
  if (n_planes) *n_planes = static_cast<int64_t>(c->prog.planes.size());
  return BLOCH_OK;
}

namespace {
// spin shard [b[r], b[r+1]) of rank r among k: np.linspace(0, n, k + 1).astype(int), as
// partition_blocks (engine.py:229-251) and parallel.shard_bounds compute it
std::vector<int64_t> linspace_bounds(int64_t n, int k) {
  std::vector<int64_t> b(static_cast<size_t>(k) + 1);
  const double step = static_cast<double>(n) / static_cast<double>(k);
  for (int i = 0; i < k; ++i) b[i] = static_cast<int64_t>(static_cast<double>(i) * step);
  b[k] = n;
  return b;
}

// bloch_compute_block on a device-set context: contiguous shards, one per device, computed
// concurrently (each sub-context on its own device and stream); the partial k-spaces are pulled
// to the first device (peer copies over NVLink) and summed there in rank order.
int compute_multi(bloch_ctx* c, int64_t n, const double* pos, const double* mx, const double* my, const double* mz,
                  const double* t1, const double* t2, const double* m0, const double* domega, const double* weight,
                  int32_t n_coils, double* echoes_out, double* snaps_out, uint8_t* snap_present, uint32_t flags) {
  if (flags & BLOCH_IN_DEVICE) return fail(BLOCH_E_INVALID, "a device-set context takes host spin arrays");
  const bloch::Program& P = c->prog;
  const int k = static_cast<int>(c->subs.size());
  const int64_t G = static_cast<int64_t>(P.n_acq) * P.max_samples;
  const int64_t len = G * n_coils * 2;  // doubles of one partial k-space
  const int64_t n_snap = snaps_out ? P.n_snap : 0;
  const bool out_dev = flags & BLOCH_OUT_DEVICE;
  const std::vector<int64_t> b = linspace_bounds(n, k);
  try {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    ck(cudaEventRecord(c->ev[0], c->stream), "event");
    c->sub_echo.resize(k);
    c->sub_snap.resize(k);
    c->sub_done.resize(k, nullptr);
    c->sub_kernel_ms.assign(k, 0.f);
    c->sub_device_ms.assign(k, 0.f);
    std::vector<double> wtmp;
    for (int r = 0; r < k; ++r) {
      bloch_ctx* sub = c->subs[r];
      const int64_t lo = b[r], nr = b[r + 1] - b[r];
      ck(cudaSetDevice(sub->device), "cudaSetDevice");
      if (!c->sub_done[r]) ck(cudaEventCreateWithFlags(&c->sub_done[r], cudaEventDisableTiming), "event");
      double* e = static_cast<double*>(c->sub_echo[r].ensure(static_cast<size_t>(std::max<int64_t>(1, len)) * 8));
      double* sn = n_snap ? static_cast<double*>(c->sub_snap[r].ensure(static_cast<size_t>(std::max<int64_t>(
                                1, n_snap * nr * 3)) * 8))
                          : nullptr;
      const double* w = nullptr;
      if (weight && n_coils == 1) {
        w = weight + 2 * lo;
      } else if (weight) {  // [coil][spin] -> this shard's [coil][spin]
        wtmp.assign(static_cast<size_t>(n_coils * nr * 2), 0.0);
        for (int cc = 0; cc < n_coils; ++cc)
          memcpy(wtmp.data() + cc * nr * 2, weight + (cc * n + lo) * 2, static_cast<size_t>(nr) * 16);
        w = wtmp.data();
      }
      const int st = bloch_compute_block(sub, nr, pos + 3 * lo, mx + lo, my + lo, mz + lo, t1 + lo, t2 + lo,
                                         m0 + lo, domega + lo, w, n_coils, e, sn, r == 0 ? snap_present : nullptr,
                                         BLOCH_OUT_DEVICE | BLOCH_NO_SYNC);
      if (st != BLOCH_OK) return fail(st, "device " + std::to_string(sub->device) + " (rank " + std::to_string(r) +
                                              "): " + g_err);
      if (n_snap && nr > 0)  // this shard's rows of every snapshot, in place (rank order = block order)
        ck(cudaMemcpy2DAsync(snaps_out + lo * 3, static_cast<size_t>(n) * 24, sn, static_cast<size_t>(nr) * 24,
                             static_cast<size_t>(nr) * 24, static_cast<size_t>(n_snap), cudaMemcpyDefault,
                             sub->stream),
           "snapshot copy");
      ck(cudaEventRecord(c->sub_done[r], sub->stream), "event");
    }
    // the one exchange: partial k-spaces to the first device, summed in rank order
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    double* gath = static_cast<double*>(c->gather.ensure(static_cast<size_t>(std::max<int64_t>(1, len * k)) * 8));
    for (int r = 0; r < k; ++r) {
      ck(cudaStreamWaitEvent(c->stream, c->sub_done[r], 0), "wait");
      if (len)
        ck(cudaMemcpyPeerAsync(gath + r * len, c->device, c->sub_echo[r].p, c->subs[r]->device,
                               static_cast<size_t>(len) * 8, c->stream),
           "peer copy");
    }
    double* d_out = out_dev ? echoes_out : static_cast<double*>(c->echo.ensure(static_cast<size_t>(std::max<int64_t>(1, len)) * 8));
    if (len) ck(bloch::launch_sum_rows(gath, k, len, d_out, c->stream), "sum kernel");
    if (!out_dev && len)
      ck(cudaMemcpyAsync(echoes_out, d_out, static_cast<size_t>(len) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaEventRecord(c->ev[3], c->stream), "event");
    c->launches = 1;
    if (!(flags & BLOCH_NO_SYNC)) {
      ck(cudaStreamSynchronize(c->stream), "sync");
      float mk = 0.f;
      for (int r = 0; r < k; ++r) {
        float km = 0.f, dm = 0.f;
        int32_t l = 0;
        bloch_last_timing(c->subs[r], &km, &dm, &l);
        c->sub_kernel_ms[r] = km;
        c->sub_device_ms[r] = dm;
        mk = std::max(mk, km);
        c->launches += l;
      }
      c->kernel_ms = mk;
      ck(cudaEventElapsedTime(&c->device_ms, c->ev[0], c->ev[3]), "elapsed");
    }
    for (int i = 0; snap_present && i < P.n_snap; ++i) snap_present[i] = c->snap_present[i];
    c->last_launch[0] = c->subs[0]->last_launch[0];
    for (int i = 1; i < 5; ++i) c->last_launch[i] = c->subs[0]->last_launch[i];
  } catch (const std::exception& ex) {
    return fail(BLOCH_E_CUDA, ex.what());
  }
  return BLOCH_OK;
}
}  // namespace

int bloch_create_multi(const int32_t* devices, int32_t n_devices, int precision, bloch_ctx** out) {
  if (!out) return fail(BLOCH_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!devices || n_devices < 1 || n_devices > bloch::kMaxDevices) return fail(BLOCH_E_INVALID, "need 1..64 devices");
  bloch_ctx* c = nullptr;
  int st = bloch_create(devices[0], precision, &c);
  if (st != BLOCH_OK) return st;
  for (int32_t r = 0; r < n_devices; ++r) {
    bloch_ctx* sub = nullptr;
    st = bloch_create(devices[r], precision, &sub);
    if (st != BLOCH_OK) {
      const std::string msg = g_err;
      bloch_destroy(c);
      return fail(st, "device " + std::to_string(devices[r]) + ": " + msg);
    }
    c->subs.push_back(sub);
    if (devices[r] != devices[0]) {  // NVLink peer access for the reduction's copies (they work without it)
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[0], devices[r]);
      if (can) {
        cudaSetDevice(devices[0]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[r], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          bloch_destroy(c);
          return fail(BLOCH_E_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
        }
        cudaGetLastError();
      }
    }
  }
  *out = c;
  return BLOCH_OK;
}

int bloch_device_count_of(const bloch_ctx* c, int32_t* n_devices, int32_t* devices) {
  if (!c || !n_devices) return fail(BLOCH_E_INVALID, "NULL argument");
  *n_devices = c->subs.empty() ? 1 : static_cast<int32_t>(c->subs.size());
  if (devices) {
    if (c->subs.empty())
      devices[0] = c->device;
    else
      for (size_t i = 0; i < c->subs.size(); ++i) devices[i] = c->subs[i]->device;
  }
  return BLOCH_OK;
}

int bloch_last_device_times(const bloch_ctx* c, int32_t capacity, float* kernel_ms, float* device_ms) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (c->subs.empty()) {
    float k = 0.f, d = 0.f;
    int32_t l = 0;
    bloch_last_timing(c, &k, &d, &l);
    if (capacity >= 1) {
      if (kernel_ms) kernel_ms[0] = k;
      if (device_ms) device_ms[0] = d;
    }
    return BLOCH_OK;
  }
  for (int32_t i = 0; i < capacity && i < static_cast<int32_t>(c->sub_kernel_ms.size()); ++i) {
    if (kernel_ms) kernel_ms[i] = c->sub_kernel_ms[i];
    if (device_ms) device_ms[i] = c->sub_device_ms[i];
  }
  return BLOCH_OK;
}

int bloch_compute_block(bloch_ctx* c, int64_t n, const double* pos, const double* mx,
                        const double* my, const double* mz, const double* t1, const double* t2,
                        const double* m0, const double* domega, const double* weight,
                        int32_t n_coils, double* echoes_out, double* snaps_out,
                        uint8_t* snap_present, uint32_t flags) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->subs.empty()) {
    if (!c->has_prog) return fail(BLOCH_E_STATE, "bloch_set_tables must be called first");
    if (n < 0) return fail(BLOCH_E_INVALID, "n < 0");
    if (n_coils < 1 || n_coils > 8) return fail(BLOCH_E_INVALID, "n_coils must be in [1, 8]");
    if (n_coils > 1 && !weight) return fail(BLOCH_E_INVALID, "n_coils > 1 requires a weight array");
    if (n > 0 && (!pos || !mx || !my || !mz || !t1 || !t2 || !m0 || !domega))
      return fail(BLOCH_E_INVALID, "NULL spin array");
    if (static_cast<int64_t>(c->prog.n_acq) * c->prog.max_samples > 0 && !echoes_out)
      return fail(BLOCH_E_INVALID, "echoes_out is NULL");
    return compute_multi(c, n, pos, mx, my, mz, t1, t2, m0, domega, weight, n_coils, echoes_out, snaps_out,
                         snap_present, flags);
  }
  if (!c->has_prog) return fail(BLOCH_E_STATE, "bloch_set_tables must be called first");
  if (c->device == BLOCH_HOST_ONLY) return fail(BLOCH_E_STATE, "host-only context cannot compute");
  if (n < 0) return fail(BLOCH_E_INVALID, "n < 0");
  if (n_coils < 1 || n_coils > 8) return fail(BLOCH_E_INVALID, "n_coils must be in [1, 8]");
  if (n_coils > 1 && !weight) return fail(BLOCH_E_INVALID, "n_coils > 1 requires a weight array");
  if (n > 0 && (!pos || !mx || !my || !mz || !t1 || !t2 || !m0 || !domega))
    return fail(BLOCH_E_INVALID, "NULL spin array");
  const bloch::Program& P = c->prog;
  const int64_t G = static_cast<int64_t>(P.n_acq) * P.max_samples;
  if (G > 0 && !echoes_out) return fail(BLOCH_E_INVALID, "echoes_out is NULL");
  const bool in_dev = flags & BLOCH_IN_DEVICE, out_dev = flags & BLOCH_OUT_DEVICE;
  static const bool no_graph = getenv("BLOCH_NO_GRAPH") != nullptr;
  const bool graphable = in_dev && out_dev && !no_graph && !c->gate_wait && !c->gate_signal;
  bloch_ctx::GraphKey key;
  if (graphable) {
    const void* ptrs[12] = {pos, mx, my, mz, t1, t2, m0, domega, weight, echoes_out, snaps_out, nullptr};
    key.n = n;
    for (int i = 0; i < 12; ++i) key.p[i] = ptrs[i];
    key.n_coils = n_coils;
    key.flags = flags & ~BLOCH_NO_SYNC;
    key.gen = c->prog_gen;
    key.alloc = g_alloc_gen.load();
    key.st = c->stream;
  }
  bool capturing = false;
  try {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    cudaStream_t st = c->stream;
    if (graphable && c->graph_exec && key == c->graph_key) {  // replay the captured device work
      ck(cudaGraphLaunch(c->graph_exec, st), "graph launch");
      c->launches = c->graph_launches;
      if (!(flags & BLOCH_NO_SYNC)) {
        ck(cudaStreamSynchronize(st), "stream sync");
        ck(cudaEventElapsedTime(&c->kernel_ms, c->ev[1], c->ev[2]), "elapsed");
        ck(cudaEventElapsedTime(&c->device_ms, c->ev[0], c->ev[3]), "elapsed");
        phase_times(c);
      }
      if (snap_present)
        for (int32_t i = 0; i < P.n_snap; ++i) snap_present[i] = c->snap_present[i];
      return BLOCH_OK;
    }
    // the second identical call is captured (the first sized every buffer: no allocation below)
    if (graphable && key == c->last_key) {
      ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
      capturing = true;
    }
    c->launches = 0;
    ck(cudaEventRecordWithFlags(c->ev[0], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
    const int ncp = n_coils <= 1 ? 1 : n_coils <= 2 ? 2 : n_coils <= 4 ? 4 : 8;
    const size_t nd = static_cast<size_t>(n) * sizeof(double);

    // 1. inputs on the device
    const double *d_pos = pos, *d_mx = mx, *d_my = my, *d_mz = mz, *d_t1 = t1, *d_t2 = t2,
                 *d_m0 = m0, *d_dw = domega, *d_w = weight;
    if (!in_dev && n > 0) {
      upload(c->in_pos, pos, 3 * nd, st);
      upload(c->in_mx, mx, nd, st);
      upload(c->in_my, my, nd, st);
      upload(c->in_mz, mz, nd, st);
      upload(c->in_t1, t1, nd, st);
      upload(c->in_t2, t2, nd, st);
      upload(c->in_m0, m0, nd, st);
      upload(c->in_dw, domega, nd, st);
      d_pos = c->in_pos.as<double>();
      d_mx = c->in_mx.as<double>();
      d_my = c->in_my.as<double>();
      d_mz = c->in_mz.as<double>();
      d_t1 = c->in_t1.as<double>();
      d_t2 = c->in_t2.as<double>();
      d_m0 = c->in_m0.as<double>();
      d_dw = c->in_dw.as<double>();
      if (weight) {
        upload(c->in_w, weight, 2 * nd * n_coils, st);
        d_w = c->in_w.as<double>();
      }
    }
    // 2. staging: per-spin constant records, relax / rotation / progression class tables
    if (n > 0) {
      c->sc.ensure(static_cast<size_t>(n) * sizeof(bloch::SpinConst));
      bloch::SpinConst* d_sc = c->sc.as<bloch::SpinConst>();
      ck(bloch::launch_prep(n, d_pos, d_dw, d_m0, d_t1, d_t2, d_sc, st), "prep kernel");
      c->launches++;
      const int n_cls = static_cast<int>(P.relax_t.size());
      if (n_cls > 0) {
        c->relax.ensure(2 * nd * n_cls);
        ck(bloch::launch_relax_table(n, n_cls, c->d_relax_t.as<double>(), d_sc, c->relax.as<double>(), st),
           "relax table kernel");
        c->launches++;
      }
      const int n_planes = static_cast<int>(P.planes.size());
      if (n_planes > 0) {
        c->planetab.ensure(2 * nd * n_planes);
        float2* p32 = nullptr;  // fp32 mode: the PL_SAMPLE planes as float2
        if (c->precision == BLOCH_PREC_F32) p32 = static_cast<float2*>(c->planetab32.ensure(nd * n_planes));
        ck(bloch::launch_planes(n, n_planes, c->d_planes.as<bloch::PlaneDesc>(), d_sc, n_coils == 1 ? d_w : nullptr,
                                c->planetab.as<double>(), p32, st),
           "plane kernel");
        c->launches++;
      }
      const int n_train = static_cast<int>(P.train_classes.size());
      if (n_train > 0) {
        c->traintab.ensure(bloch::kTrainRow * nd * n_train);
        ck(bloch::launch_train_table(n, n_train, c->d_train_cls.as<bloch::TrainClass>(), c->d_mats.as<double>(), d_sc,
                                     c->traintab.as<double>(), st),
           "train table kernel");
        c->launches++;
      }
      if (d_w && ncp != n_coils) {
        c->wpad.ensure(2 * nd * ncp);
        ck(bloch::launch_pad_weights(n, n_coils, ncp, d_w, c->wpad.as<double>(), st), "pad kernel");
        c->launches++;
        d_w = c->wpad.as<double>();
      }
      if (d_w && ncp >= 2 && c->precision == BLOCH_PREC_F32) {  // fp32 weights for the tensor-core windows
        c->w32.ensure(static_cast<size_t>(n) * ncp * sizeof(float2));
        ck(bloch::launch_weights_f32(n, ncp, d_w, c->w32.as<float2>(), st), "weights kernel");
        c->launches++;
      }
    }
    // 3. outputs
    const size_t echo_bytes = static_cast<size_t>(G) * n_coils * 2 * sizeof(double);
    double* d_echo = out_dev ? echoes_out : static_cast<double*>(c->echo.ensure(echo_bytes));
    if (echo_bytes) ck(cudaMemsetAsync(d_echo, 0, echo_bytes, st), "memset echoes");
    const size_t snap_bytes = static_cast<size_t>(P.n_snap) * n * 3 * sizeof(double);
    double* d_snap = nullptr;
    if (snaps_out && snap_bytes) {
      d_snap = out_dev ? snaps_out : static_cast<double*>(c->snaps.ensure(snap_bytes));
      ck(cudaMemsetAsync(d_snap, 0, snap_bytes, st), "memset snapshots");
    }
    // 4. integrator + ordered fold
    float kms = 0.f;
    c->last_groups = 0;
    c->last_csamples = 0;
    if (n > 0) {
      // the window contraction: fp32 mode, one receive coil, U rows within the partial budget
      const int64_t urows = static_cast<int64_t>(P.urow_out0.size());
      const int64_t uwords = bloch::contract_u_words(urows, n);
      const bool defer = c->contraction && c->precision == BLOCH_PREC_F32 && !P.groups.empty() &&
                         2 * uwords * 4 <= partial_budget_bytes();
      const std::vector<bloch::DevOp>& OPS = defer ? P.dops : P.ops;
      bool full = false, win = c->precision != BLOCH_PREC_F32;
      for (const bloch::DevOp& op : OPS) {  // tabulated RF trains (train classes) run in every variant
        if ((op.kind == bloch::OP_RFTRAIN && op.rot < 0) || op.kind == bloch::OP_CHIRP || op.kind == bloch::OP_GSAMP)
          full = true;
        if (op.kind == bloch::OP_WINDOW) win = true;
      }
      win = win || full;
      // the L2 working set of the stream: planes read by at least 4 ops (a snapshot at the end, for one,
      // splits the last window's class off: those planes are read once)
      std::vector<int32_t> refs(P.planes.size(), 0);
      for (const bloch::DevOp& op : OPS)
        for (int k = 0; k < 4; ++k)
          if (op.pl[k] >= 0 && op.pl[k] < static_cast<int32_t>(refs.size())) refs[op.pl[k]]++;
      int64_t hot = 0;
      for (int32_t r : refs) hot += r >= 4;
      Variant v = pick_variant(c->precision, n, ncp, c->n_sm, win, hot * 16);
      v.full = full;
      v.win = win;
      // the resident-table integrator: fully deferred fp32 programs whose tables fit a CTA's shared memory
      static const bool no_resident = getenv("BLOCH_NO_RESIDENT") != nullptr;  // A/B hook
      int res_s = 1;
      const int res_threads = (defer && !full && !win && c->resident && !no_resident && c->rplan.ok)
                                  ? bloch::resident_threads(c->rplan, n, c->n_sm, &res_s) : 0;
      c->last_resident = res_threads > 0;
      if (res_threads > 0) v.S = res_s;
      int max_t = 512, min_b = 1;
      variant_shape(v, &max_t, &min_b);
      const int64_t slots = int64_t(c->n_sm) * min_b;  // resident CTAs per wave
      const int64_t per_wave = slots * v.S * max_t;
      const int64_t waves = (n + per_wave - 1) / per_wave;
      int64_t threads = (n + slots * waves * v.S - 1) / (slots * waves * v.S);
      threads = ((threads + 31) / 32) * 32;
      threads = std::max<int64_t>(32, std::min<int64_t>(max_t, threads));
      if (res_threads > 0) threads = res_threads;
      const int64_t spc = threads * v.S;
      int64_t grid = (n + spc - 1) / spc;
      bloch::ResidentShape rshape{};
      if (res_threads > 0) {  // two-spin launches: spins dealt evenly over full waves of CTAs
        bloch::resident_grid(n, c->n_sm, res_threads, v.S, &rshape);
        grid = rshape.grid;
        threads = rshape.block;
      }
      c->last_launch[0] = v.prec;
      c->last_launch[1] = v.S;
      c->last_launch[2] = v.NC;
      c->last_launch[3] = static_cast<int>(grid);
      c->last_launch[4] = static_cast<int>(threads);
      const size_t rsz = v.prec == 32 ? sizeof(float) : sizeof(double);
      const int64_t rows = grid * (threads / 32);  // one partial row per warp
      // Program segments: the partial rows hold one slot per (warp, sample, coil), so a long
      // acquisition on a large block can exceed the device.  The op stream is cut into segments
      // whose samples fit the budget; each runs as its own launch (state handed over in fp64
      // through global memory, bit-identical to one launch) followed by the fold of its samples.
      const std::vector<Segment> segs = plan_segments(OPS, rows * ncp * 2 * static_cast<int64_t>(rsz));
      int64_t max_seg_slots = 1;
      for (const Segment& g : segs) max_seg_slots = std::max<int64_t>(max_seg_slots, g.n_samples * ncp);
      c->partial.ensure(static_cast<size_t>(rows * max_seg_slots * 2) * rsz);
      c->last_segments = static_cast<int32_t>(segs.size());
      if (segs.size() > 1) {
        c->state.ensure(static_cast<size_t>(6) * nd);  // two ping-pong (mx, my, mz) sets
      }
      // contraction buffers (sized before any capture: the first call of a shape allocates)
      std::vector<bloch::ContractPlan> cplans;
      if (defer) {
        c->uhi.ensure(static_cast<size_t>(uwords) * 4);
        c->ulo.ensure(static_cast<size_t>(uwords) * 4);
        size_t cb = 0;
        for (const bloch::WinGroup& g : P.groups) {
          cplans.push_back(bloch::contract_plan(g.count, g.n_windows, n, c->n_sm, n_coils));
          bloch::ContractJob j0{};
          j0.W = g.n_windows;
          j0.K = g.count;
          j0.C = n_coils;
          cb = std::max(cb, bloch::contract_part_bytes(cplans.back(), j0));
        }
        c->cpart.ensure(cb);
        c->ztab.ensure(static_cast<size_t>(n) * sizeof(float4));
        c->zqtab.ensure(static_cast<size_t>(n) * sizeof(float2));
      }
      bloch::KParams kp{};
      kp.ops = defer ? c->d_dops.as<bloch::DevOp>() : c->d_ops.as<bloch::DevOp>();
      kp.n_ops = static_cast<int32_t>(OPS.size());
      kp.uhi = defer ? c->uhi.as<uint32_t>() : nullptr;
      kp.ulo = defer ? c->ulo.as<uint32_t>() : nullptr;
      kp.urows = urows;
      if (defer && (n & 15)) {  // the last 16-spin block's padding words: zero (the product reads them)
        const size_t off = static_cast<size_t>(n / 16) * urows * 16 * 4, len = static_cast<size_t>(urows) * 16 * 4;
        ck(cudaMemsetAsync(c->uhi.as<char>() + off, 0, len, st), "memset U");
        ck(cudaMemsetAsync(c->ulo.as<char>() + off, 0, len, st), "memset U");
      }
      kp.spins_per_cta = static_cast<int32_t>(spc);
      kp.gev = c->d_gev.as<bloch::GEv>();
      kp.mats = c->d_mats.as<double>();
      {
        static const bool no_smem_mats = getenv("BLOCH_NO_SMEM_MATS") != nullptr;  // A/B hook
        const int64_t nm = static_cast<int64_t>(P.mats.size() / 9);
        kp.n_mats_smem = (!no_smem_mats && !v.full && !v.win && v.S <= 2 && nm <= bloch::kMatsSmemMax)
                             ? static_cast<int32_t>(nm) : 0;
        // progression running factors in shared memory (register-state kernels, up to 64 KB per CTA)
        static const bool no_smem_prog = getenv("BLOCH_NO_SMEM_PROG") != nullptr;  // A/B hook
        kp.n_prog_smem = 0;
        const int np = static_cast<int>(P.prog_classes.size());
        if (!no_smem_prog && !v.full && !v.win && v.S <= 4 && np > 0 && np <= 32 &&
            static_cast<int64_t>(np) * v.S * threads * 16 <= 64 * 1024) {
          for (int pc = 0; pc < np; ++pc) kp.prog_plane[pc] = -1;
          for (const bloch::DevOp& op : OPS)
            if (op.kind == bloch::OP_EVENT && op.prg >= 0 && op.prg < np) kp.prog_plane[op.prg] = op.pl[0];
          bool ok = true;
          for (int pc = 0; pc < np; ++pc) ok = ok && kp.prog_plane[pc] >= 0;
          if (ok) kp.n_prog_smem = np;
        }
      }
      kp.n = n;
      kp.sc = c->sc.as<bloch::SpinConst>();
      kp.mx0 = d_mx;
      kp.my0 = d_my;
      kp.mz0 = d_mz;
      kp.w = d_w;
      kp.w32 = (d_w && ncp >= 2 && c->precision == BLOCH_PREC_F32) ? c->w32.as<float2>() : nullptr;
      kp.partial = c->partial.p;
      kp.snaps = d_snap;
      kp.relax = c->relax.as<double>();
      kp.planes = c->planetab.as<double2>();
      kp.planes32 = c->precision == BLOCH_PREC_F32 ? c->planetab32.as<float2>() : nullptr;
      kp.train = c->traintab.as<double>();
      if (c->gate_wait) ck(cudaStreamWaitEvent(st, c->gate_wait, 0), "gate wait");
      ck(cudaEventRecordWithFlags(c->ev[1], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
      double* state = c->state.as<double>();
      for (size_t k = 0; k < segs.size(); ++k) {
        const Segment& g = segs[k];
        const int64_t seg_slots = g.n_samples * ncp;
        kp.op_begin = g.op_begin;
        kp.n_ops = g.op_end;
        kp.sample_base = static_cast<int32_t>(g.sample_begin);
        kp.part_stride = seg_slots * 2;
        kp.mx0 = k == 0 ? d_mx : state + ((k - 1) & 1) * 3 * n;
        kp.my0 = k == 0 ? d_my : state + ((k - 1) & 1) * 3 * n + n;
        kp.mz0 = k == 0 ? d_mz : state + ((k - 1) & 1) * 3 * n + 2 * n;
        const bool hand_over = k + 1 < segs.size();
        kp.mx1 = hand_over ? state + (k & 1) * 3 * n : nullptr;
        kp.my1 = hand_over ? state + (k & 1) * 3 * n + n : nullptr;
        kp.mz1 = hand_over ? state + (k & 1) * 3 * n + 2 * n : nullptr;
        if (res_threads > 0) {
          bloch::RParams rp{};
          rp.rops = c->d_rops.as<bloch::ROp>();
          rp.n_rops = static_cast<int32_t>(c->rplan.rops.size());
          rp.loads = c->d_rloads.as<bloch::RLoad>();
          rp.n_loads = static_cast<int32_t>(c->rplan.loads.size());
          rp.mats = c->d_rmats.as<double>();
          rp.n_mats = static_cast<int32_t>(c->rplan.mats.size() / 9);
          rp.mats4 = c->d_rmats4.as<double>();
          rp.n_mats4 = static_cast<int32_t>(c->rplan.mats4.size() / 4);
          rp.ops = kp.ops;
          rp.n = n;
          rp.mx0 = kp.mx0;
          rp.my0 = kp.my0;
          rp.mz0 = kp.mz0;
          rp.planes = kp.planes;
          rp.planes32 = kp.planes32;
          rp.train = kp.train;
          rp.sc = kp.sc;
          rp.relax = kp.relax;
          rp.w1 = n_coils == 1 ? reinterpret_cast<const double2*>(d_w) : nullptr;
          rp.snaps = kp.snaps;
          rp.uhi = kp.uhi;
          rp.ulo = kp.ulo;
          rp.urows = kp.urows;
          rp.n_big = rshape.n_big;
          rp.bd_big = rshape.bd_big;
          rp.bd_small = rshape.bd_small;
          ck(bloch::launch_resident(rp, c->rplan, v.S, static_cast<int>(grid), static_cast<int>(threads), st),
             "resident integrate kernel");
        } else {
          ck(dispatch(v, kp, static_cast<int>(grid), static_cast<int>(threads), st), "integrate kernel");
        }
        c->launches++;
        if (!hand_over && !defer) {  // after the last integrator launch (the fold of its samples follows)
          if (c->gate_signal) ck(cudaEventRecord(c->gate_signal, st), "gate signal");
          ck(cudaEventRecordWithFlags(c->ev[2], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault),
             "event");
        }
        if (seg_slots > 0) {
          const int64_t* sg = (defer ? c->d_dsample_g : c->d_sample_g).as<int64_t>() + g.sample_begin;
          const int fold_rows = static_cast<int>(rows);  // every warp's row, in a fixed order
          const int64_t row_stride = seg_slots * 2;
          if (v.prec == 32)
            ck(bloch::launch_reduce<float>(c->partial.as<float>(), fold_rows, row_stride, seg_slots, n_coils, ncp,
                                           sg, G, d_echo, st),
               "reduce kernel");
          else
            ck(bloch::launch_reduce<double>(c->partial.as<double>(), fold_rows, row_stride, seg_slots, n_coils,
                                            ncp, sg, G, d_echo, st),
               "reduce kernel");
          c->launches++;
        }
      }
      ck(cudaEventRecordWithFlags(c->ev[4], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
      if (defer) {  // 5. the window groups on the tensor cores (every U row is written: the last segment ran)
        for (size_t gi = 0; gi < P.groups.size(); ++gi) {
          const bloch::WinGroup& g = P.groups[gi];
          const bloch::PlaneDesc& zd = P.planes[g.zplane];
          bloch::ContractJob j{};
          j.sc = c->sc.as<bloch::SpinConst>();
          j.n = n;
          j.T = zd.T;
          j.d[0] = zd.d[0];
          j.d[1] = zd.d[1];
          j.d[2] = zd.d[2];
          j.tw = zd.tw;
          j.K = g.count;
          j.W = g.n_windows;
          j.row0 = g.row0;
          j.uhi = c->uhi.as<uint32_t>();
          j.ulo = c->ulo.as<uint32_t>();
          j.rows = urows;
          j.part = c->cpart.as<float>();
          j.out0 = c->d_urow_out0.as<int64_t>() + g.row0;
          j.echo = d_echo;
          j.chirp = g.chirp;
          j.qconj = g.qconj;
          if (g.chirp) {
            const bloch::PlaneDesc& qdsc = P.planes[g.qplane];
            j.qd[0] = qdsc.d[0];
            j.qd[1] = qdsc.d[1];
            j.qd[2] = qdsc.d[2];
          }
          j.C = n_coils;
          j.ncp = ncp;
          j.w32 = n_coils > 1 ? c->w32.as<float2>() : nullptr;
          j.G = G;
          j.zt = c->ztab.as<float4>();
          j.zq = c->zqtab.as<float2>();
          ck(bloch::launch_contract(j, cplans[gi], st), "contraction kernel");
          c->launches += 3;
        }
        c->last_groups = static_cast<int32_t>(P.groups.size());
        c->last_csamples = P.n_deferred_samples;
        if (c->gate_signal) ck(cudaEventRecord(c->gate_signal, st), "gate signal");
        ck(cudaEventRecordWithFlags(c->ev[2], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault),
           "event");
      }
    } else {
      ck(cudaEventRecordWithFlags(c->ev[1], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
      ck(cudaEventRecordWithFlags(c->ev[2], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
      ck(cudaEventRecordWithFlags(c->ev[4], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
    }
    // 6. outputs to the host
    if (!out_dev) {
      if (echo_bytes) ck(cudaMemcpyAsync(echoes_out, d_echo, echo_bytes, cudaMemcpyDeviceToHost, st), "D2H echoes");
      if (d_snap) ck(cudaMemcpyAsync(snaps_out, d_snap, snap_bytes, cudaMemcpyDeviceToHost, st), "D2H snapshots");
    }
    ck(cudaEventRecordWithFlags(c->ev[3], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault), "event");
    if (capturing) {
      cudaGraph_t g = nullptr;
      capturing = false;
      ck(cudaStreamEndCapture(st, &g), "end capture");
      if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
      c->graph_exec = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&c->graph_exec, g, 0);
      cudaGraphDestroy(g);
      ck(e, "graph instantiate");
      c->graph_key = key;
      c->graph_launches = c->launches;
      ck(cudaGraphLaunch(c->graph_exec, st), "graph launch");
    }
    if (graphable) {
      c->last_key = key;
      c->last_key.alloc = g_alloc_gen.load();  // the buffers this call sized: the next identical call captures
    }
    if (!(flags & BLOCH_NO_SYNC)) {
      ck(cudaStreamSynchronize(st), "stream sync");
      ck(cudaEventElapsedTime(&kms, c->ev[1], c->ev[2]), "elapsed");
      c->kernel_ms = kms;
      ck(cudaEventElapsedTime(&c->device_ms, c->ev[0], c->ev[3]), "elapsed");
      phase_times(c);
    }
    if (snap_present)
      for (int32_t i = 0; i < P.n_snap; ++i) snap_present[i] = c->snap_present[i];
  } catch (const InvalidArg& ex) {
    if (capturing) abandon_capture(c);
    return fail(BLOCH_E_INVALID, ex.what());
  } catch (const std::exception& ex) {
    if (capturing) abandon_capture(c);
    return fail(BLOCH_E_CUDA, ex.what());
  }
  return BLOCH_OK;
}

int bloch_set_resident(bloch_ctx* c, int32_t enable) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  c->resident = enable != 0;
  for (bloch_ctx* sub : c->subs) sub->resident = enable != 0;
  c->drop_graph();
  return BLOCH_OK;
}

int bloch_last_resident(const bloch_ctx* c, int32_t* resident, int32_t* bytes_per_spin) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  const bloch_ctx* q = c->subs.empty() ? c : c->subs[0];
  if (resident) *resident = q->last_resident;
  if (bytes_per_spin) *bytes_per_spin = q->rplan.ok ? q->rplan.bytes_per_spin : 0;
  return BLOCH_OK;
}

int bloch_set_contraction(bloch_ctx* c, int32_t enable) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  c->contraction = enable != 0;
  for (bloch_ctx* sub : c->subs) sub->contraction = enable != 0;
  c->drop_graph();
  return BLOCH_OK;
}

int bloch_program_groups(const bloch_ctx* c, int32_t* n_groups, int64_t* contracted_samples,
                         int64_t* integrator_samples) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->has_prog) return fail(BLOCH_E_STATE, "no tables uploaded");
  if (n_groups) *n_groups = static_cast<int32_t>(c->prog.groups.size());
  if (contracted_samples) *contracted_samples = c->prog.n_deferred_samples;
  if (integrator_samples) *integrator_samples = static_cast<int64_t>(c->prog.dsample_g.size());
  return BLOCH_OK;
}

int bloch_program_ops(const bloch_ctx* c, int32_t deferred, int32_t capacity, int32_t* n_ops, int32_t* kind,
                      int32_t* count, int32_t* rot, int32_t* prg, int32_t* pre, int32_t* pl) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->has_prog) return fail(BLOCH_E_STATE, "no tables uploaded");
  const std::vector<bloch::DevOp>& ops = deferred ? c->prog.dops : c->prog.ops;
  if (n_ops) *n_ops = static_cast<int32_t>(ops.size());
  for (int32_t i = 0; i < capacity && i < static_cast<int32_t>(ops.size()); ++i) {
    const bloch::DevOp& o = ops[i];
    if (kind) kind[i] = o.kind;
    if (count) count[i] = o.count;
    if (rot) rot[i] = o.rot;
    if (prg) prg[i] = o.prg;
    if (pre) pre[i] = o.pre;
    if (pl)
      for (int k = 0; k < 4; ++k) pl[4 * i + k] = o.pl[k];
  }
  return BLOCH_OK;
}

int bloch_last_phases(const bloch_ctx* c, float* integrate_ms, float* contract_ms, int32_t* n_groups,
                      int64_t* contracted_samples) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  const bloch_ctx* s = c->subs.empty() ? c : c->subs[0];
  if (s->device != BLOCH_HOST_ONLY && s->ev[3]) {  // asynchronous calls: wait for the call's last event
    cudaSetDevice(s->device);
    if (cudaEventSynchronize(s->ev[3]) == cudaSuccess) phase_times(const_cast<bloch_ctx*>(s));
    cudaGetLastError();
  }
  if (integrate_ms) *integrate_ms = s->integrate_ms;
  if (contract_ms) *contract_ms = s->contract_ms;
  if (n_groups) *n_groups = s->last_groups;
  if (contracted_samples) *contracted_samples = s->last_csamples;
  return BLOCH_OK;
}

int bloch_rasterize(bloch_ctx* c, const bloch_box_t* boxes, int32_t n_boxes, const bloch_shape_t* shapes,
                    int32_t n_shapes, const bloch_field_t* field, const bloch_coil_t* coils, int32_t n_coils,
                    double uniform_s, int64_t capacity, double* pos, double* mx, double* my, double* mz,
                    double* t1, double* t2, double* m0, double* domega, double* weight, int64_t* n_out) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (c->device == BLOCH_HOST_ONLY) return fail(BLOCH_E_STATE, "host-only context cannot rasterize");
  if (!n_out) return fail(BLOCH_E_INVALID, "n_out is NULL");
  *n_out = 0;
  if (n_boxes < 1 || n_boxes > bloch::kMaxRasterBoxes || !boxes)
    return fail(BLOCH_E_INVALID, "need 1.." + std::to_string(bloch::kMaxRasterBoxes) + " boxes");
  if (n_shapes < 0 || n_shapes > bloch::kMaxShapes || (n_shapes && !shapes))
    return fail(BLOCH_E_INVALID, "shape count out of range");
  if (n_coils < 0 || n_coils > 8 || (n_coils && !coils)) return fail(BLOCH_E_INVALID, "n_coils must be in [0, 8]");
  bloch_field_t f{};
  if (field) f = *field;
  if (f.n_poly < 0 || f.n_poly > bloch::kMaxPoly || (f.n_poly && !f.poly) || f.n_bumps < 0 ||
      f.n_bumps > bloch::kMaxBumps || (f.n_bumps && !f.bumps))
    return fail(BLOCH_E_INVALID, "field model out of range");
  if (f.n_poly && !(f.poly_len > 0.0)) return fail(BLOCH_E_INVALID, "poly_len must be > 0");
  for (int k = 0; k < f.n_poly; ++k)
    for (int j = 1; j < 4; ++j) {
      const double e = f.poly[4 * k + j];
      if (!(e >= 0.0 && e <= 16.0 && e == (double)(int)e))
        return fail(BLOCH_E_INVALID, "polynomial exponents must be integers in [0, 16]");
    }
  int64_t sites = 0;
  for (int b = 0; b < n_boxes; ++b) {
    const bloch_box_t& bx = boxes[b];
    if (bx.shape_count < 0 || bx.shape_begin < 0 || bx.shape_begin + bx.shape_count > n_shapes)
      return fail(BLOCH_E_INVALID, "box " + std::to_string(b) + " shape range outside the shape table");
    int64_t cnt = 1;
    for (int a = 0; a < 3; ++a) {
      if (bx.count[a] < 1) return fail(BLOCH_E_INVALID, "box lattice counts must be >= 1");
      cnt *= bx.count[a];
    }
    sites += cnt;
  }
  if (sites > capacity)
    return fail(BLOCH_E_INVALID, std::to_string(sites) + " lattice sites exceed the capacity of " +
                                     std::to_string(capacity));
  if (sites >= (int64_t)INT32_MAX) return fail(BLOCH_E_INVALID, "more than 2^31 lattice sites");
  if (sites > 0 && (!pos || !mx || !my || !mz || !t1 || !t2 || !m0 || !domega || !weight))
    return fail(BLOCH_E_INVALID, "NULL output array");
  try {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t need = bloch::raster_scratch_bytes(sites);
    c->raster_scratch.ensure(need);
    c->raster_staging.resize(bloch::raster_staging_bytes());
    bloch::RasterArgs a{};
    a.boxes = boxes;
    a.n_boxes = n_boxes;
    a.shapes = shapes;
    a.n_shapes = n_shapes;
    a.field = f;
    a.coils = coils;
    a.n_coils = n_coils;
    a.uniform_s = uniform_s;
    a.capacity = capacity;
    a.out = bloch::RasterOut{pos, mx, my, mz, t1, t2, m0, domega, weight};
    int64_t n = 0;
    int bad = 0;
    ck(bloch::raster_run(a, c->raster_scratch.p, c->raster_scratch.cap, c->raster_staging.data(), c->n_sm,
                         c->stream, &n, &bad),
       "rasterize");
    *n_out = n;
    if (bad) return fail(BLOCH_E_INVALID, "rasterized tissue has m0 < 0 or T1/T2 <= 0");
  } catch (const std::exception& ex) {
    return fail(BLOCH_E_CUDA, ex.what());
  }
  return BLOCH_OK;
}

int bloch_set_kernel_gate(bloch_ctx* c, void* wait_event, void* signal_event) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (!c->subs.empty()) return fail(BLOCH_E_STATE, "not available on a device-set context");
  c->gate_wait = static_cast<cudaEvent_t>(wait_event);
  c->gate_signal = static_cast<cudaEvent_t>(signal_event);
  c->drop_graph();
  return BLOCH_OK;
}

int bloch_synchronize(bloch_ctx* c) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (c->device == BLOCH_HOST_ONLY) return BLOCH_OK;
  for (bloch_ctx* sub : c->subs) {
    const int st = bloch_synchronize(sub);
    if (st != BLOCH_OK) return st;
  }
  cudaSetDevice(c->device);
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return fail(BLOCH_E_CUDA, std::string("stream sync: ") + cudaGetErrorString(e));
  return BLOCH_OK;
}

int bloch_last_timing(const bloch_ctx* c, float* kernel_ms, float* device_ms, int32_t* launches) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (c->device != BLOCH_HOST_ONLY && c->ev[3]) {  // asynchronous calls: wait for the call's last event
    cudaSetDevice(c->device);
    if (cudaEventSynchronize(c->ev[3]) == cudaSuccess) {
      float k = 0.f, d = 0.f;
      if (cudaEventElapsedTime(&k, c->ev[1], c->ev[2]) == cudaSuccess) const_cast<bloch_ctx*>(c)->kernel_ms = k;
      if (cudaEventElapsedTime(&d, c->ev[0], c->ev[3]) == cudaSuccess) const_cast<bloch_ctx*>(c)->device_ms = d;
      phase_times(const_cast<bloch_ctx*>(c));
    }
    cudaGetLastError();
  }
  if (kernel_ms) *kernel_ms = c->kernel_ms;
  if (device_ms) *device_ms = c->device_ms;
  if (launches) *launches = c->launches;
  return BLOCH_OK;
}

int bloch_last_launch(const bloch_ctx* c, int32_t* prec, int32_t* spins_per_thread, int32_t* coils,
                      int32_t* grid, int32_t* threads) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  int32_t* out[5] = {prec, spins_per_thread, coils, grid, threads};
  for (int i = 0; i < 5; ++i)
    if (out[i]) *out[i] = c->last_launch[i];
  return BLOCH_OK;
}

int bloch_last_segments(const bloch_ctx* c, int32_t* segments) {
  if (!c) return fail(BLOCH_E_INVALID, "ctx is NULL");
  if (segments) *segments = c->last_segments;
  return BLOCH_OK;
}

}  // extern "C"
