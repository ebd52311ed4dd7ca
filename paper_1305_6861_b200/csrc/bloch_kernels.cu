// sm_100a kernels of the Bloch event-stream engine.
//
// integrate_kernel<R, S, NC>  — the hot path: restates engine.compute_block
//   (engine.py:259-310) for S spins per thread.  The op stream (program.h) is
//   identical for every thread, so all control flow is CTA-uniform and op
//   fields are broadcast loads.  ADC samples are reduced without atomics and
//   without CTA barriers: per-thread sum over its S spins -> warp
//   transpose-reduction of 8 slots (sample x coil) -> the warp's own row of the
//   partial buffer; reduce_partials_kernel folds the rows in a fixed order in
//   fp64 (deterministic, like the reference's ordered fold, engine.py:594-595).
//
// Precision: the per-spin state (mx, my, mz) is fp64 in every mode and lives in
// shared memory between ops (it only changes at pulses, intervals, RF trains,
// chirps and window exits).  R is the type of the ADC sample recurrence inside
// uniform windows, the dominant work: fp32 (BLOCH_PREC_F32, packed
// FFMA2/FMUL2/FADD2 over spin pairs) or fp64.
//
// Uniform ADC windows (OP_WINDOW): per spin the sample factor
// z = e2 * exp(-i*theta) and the closed-form propagators of the whole
// (pre, samples, post) run come from the per-spin planes of its rotation
// class (plane_kernel, fp64, once per call); the receive-weighted transverse
// magnetisation u = w * (Cpre m) is advanced by one complex multiply per sample
// (engine.py:289-305 for every sample of the window: same theta, same e2 from
// the relax cache).  The state leaving the window is C m, mz -> A mz + B in
// fp64, so per-sample rounding never feeds back into the spin state.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "contract.h"
#include "kernels.h"
#include "program.h"

namespace bloch {

// ---------------------------------------------------------------------------
// math helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ double reduce_2pi(double th) {
  const double kInv2Pi = 0.15915494309189535;
  const double kHi = 6.283185307179586;       // 2*pi rounded to double
  const double kLo = 2.4492935982947064e-16;  // 2*pi - kHi
  const double k = rint(th * kInv2Pi);
  return fma(-k, kLo, fma(-k, kHi, th));
}

// exp(-i*theta) = (c, -s), fp64
__device__ __forceinline__ void phase_factor(double th, double& c, double& ms) {
  double s;
  sincos(reduce_2pi(th), &s, &c);
  ms = -s;
}

template <typename R>
__device__ __forceinline__ R shfl_x(R v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Transpose-reduce 8 per-lane slots across the warp.  Afterwards v[0] of lane
// l holds the warp total of slot ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1)
// (identical on the 4 lanes l, l^1, l^2, l^3).  9 shuffles for 8 slots
// instead of 40 for eight butterflies.
template <typename R>
__device__ __forceinline__ void transpose_reduce8(R (&v)[kChunkSlots], int lane) {
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const R send = hi ? v[j] : v[j + 4];
      const R keep = hi ? v[j + 4] : v[j];
      v[j] = keep + shfl_x(send, 16);
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const R send = hi ? v[j] : v[j + 2];
      const R keep = hi ? v[j + 2] : v[j];
      v[j] = keep + shfl_x(send, 8);
    }
  }
  {
    const bool hi = lane & 4;
    const R send = hi ? v[0] : v[1];
    const R keep = hi ? v[1] : v[0];
    v[0] = keep + shfl_x(send, 4);
  }
  v[0] += shfl_x(v[0], 2);
  v[0] += shfl_x(v[0], 1);
}

// Each warp owns one row of the partial buffer: after the transpose-reduction
// the 8 lanes holding a slot total write it straight to global memory (64 B per
// chunk, coalesced).  No shared-memory staging, no CTA barrier.
template <typename R>
struct Strip {
  R* row;  // this warp's partial row: [n_slots][2]
  int lane;

  __device__ __forceinline__ void push(R (&re)[kChunkSlots], R (&im)[kChunkSlots], int cnt, int32_t first_id) {
    transpose_reduce8(re, lane);
    transpose_reduce8(im, lane);
    const int j = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && j < cnt) {
      R* p = row + static_cast<int64_t>(first_id + j) * 2;
      __stcs(p, re[0]);  // streaming: the partial rows must not evict the class tables from L2
      __stcs(p + 1, im[0]);
    }
  }
};

// L2 priority of the progression running factors (read, advanced and rewritten at every occurrence
// of the class, ~1000 times per spin on config 2): evict_last keeps the RMW in L2 while the streamed
// partial rows (evict_first) and the read-only planes pass through; without it the factors were
// evicted between occurrences and re-fetched from DRAM (ncu: 26 GB of DRAM traffic per launch)
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double2 ld_keep(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------------------
// spin state (shared memory, [3][S][blockDim] fp64) and per-spin constants
// ---------------------------------------------------------------------------

// kReg: the state lives in registers (every access indexed by an unrolled slot loop); the kernels
// without window / chirp / train code use it, the others keep it in shared memory
template <int S, bool kReg = false>
struct Spins {
  static constexpr int kS = S;
  double* sm;
  int64_t base;  // spin index of slot 0 of this thread
  int bd;
  int64_t n;
  int nact;      // active slots: idx(s) < n exactly for s < nact (idx grows with s)
  double v[kReg ? 3 : 1][kReg ? S : 1];
  __device__ __forceinline__ int64_t idx(int s) const { return base + static_cast<int64_t>(s) * bd; }
  __device__ __forceinline__ bool act(int s) const { return s < nact; }
  __device__ __forceinline__ void init_active() {
    const int64_t left = n - base;
    nact = left <= 0 ? 0 : static_cast<int>(left >= static_cast<int64_t>(S) * bd ? S : (left + bd - 1) / bd);
  }
  __device__ __forceinline__ double& mx(int s) {
    if constexpr (kReg) return v[0][s]; else return sm[(0 * S + s) * bd + threadIdx.x];
  }
  __device__ __forceinline__ double& my(int s) {
    if constexpr (kReg) return v[1][s]; else return sm[(1 * S + s) * bd + threadIdx.x];
  }
  __device__ __forceinline__ double& mz(int s) {
    if constexpr (kReg) return v[2][s]; else return sm[(2 * S + s) * bd + threadIdx.x];
  }
};

// SpinConst (kernels.h): one 64-byte record per spin, 4 x 16-byte loads
struct SC {
  double x, y, z, dw, m0;
};
__device__ __forceinline__ SC load_sc(const KParams& kp, int64_t i) {
  const double2* p = reinterpret_cast<const double2*>(kp.sc + i);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  return SC{a.x, a.y, b.x, b.y, c.x};
}
// engine.py:289 — theta = pos @ dmom + domega * dt
__device__ __forceinline__ double theta_of(const SC& c, double dt, double dmx, double dmy, double dmz) {
  return fma(c.z, dmz, fma(c.y, dmy, c.x * dmx)) + c.dw * dt;
}
// relax-class table: (e1, e2) = (exp(-T_c/T1_i), exp(-T_c/T2_i)) at [c][i]
__device__ __forceinline__ double2 relax_pair(const KParams& kp, int c, int64_t i) {
  return __ldg(reinterpret_cast<const double2*>(kp.relax) + static_cast<int64_t>(c) * kp.n + i);
}
// plane `id` of the op (program.h PlaneDesc): [n] double2, one value per spin
__device__ __forceinline__ const double2* plane(const KParams& kp, const DevOp* op, int k) {
  return kp.planes + static_cast<int64_t>(__ldg(&op->pl[k])) * kp.n;
}
__device__ __forceinline__ const double2* plane_at(const KParams& kp, int id, int64_t i) {
  return kp.planes + (static_cast<int64_t>(id) * kp.n + i);
}
// fp32 mode: a PL_SAMPLE plane (window Cpre / z, chirp r0 / q) as float2
__device__ __forceinline__ const float2* plane32_at(const KParams& kp, int id, int64_t i) {
  return kp.planes32 + (static_cast<int64_t>(id) * kp.n + i);
}
__device__ __forceinline__ double2 ab_at(const KParams& kp, const DevOp* op, int k, int64_t i) {
  return __ldg(plane_at(kp, __ldg(&op->pl[k]), i));
}
// rotation-class quantities of a window: Cpre, C, (A, B), z
struct RotCoef {
  double pr, pi, cr, ci, a, b, zr, zi;
};
template <typename R>
__device__ __forceinline__ RotCoef load_rot(const KParams& kp, const DevOp* op, int64_t i) {
  const double2 b = __ldg(plane(kp, op, 2) + i), d = __ldg(plane(kp, op, 3) + i);
  double2 a, e;
  if constexpr (sizeof(R) == 4) {  // Cpre and z only form fp32 samples: float2 planes
    const float2 af = __ldg(kp.planes32 + (static_cast<int64_t>(__ldg(&op->pl[0])) * kp.n + i));
    const float2 ef = __ldg(kp.planes32 + (static_cast<int64_t>(__ldg(&op->pl[1])) * kp.n + i));
    a = make_double2(af.x, af.y);
    e = make_double2(ef.x, ef.y);
  } else {
    a = __ldg(plane(kp, op, 0) + i);
    e = __ldg(plane(kp, op, 1) + i);
  }
  return RotCoef{a.x, a.y, b.x, b.y, d.x, d.y, e.x, e.y};
}

// a hard pulse fused into the following op (DevOp.pre): 9 uniform matrix entries, bloch.py:124-139
struct Mat3 {
  double r[9];
};
__device__ __forceinline__ Mat3 load_mat(const double* mats, int pre) {
  Mat3 m;
  const double* q = mats + static_cast<int64_t>(pre) * 9;
#pragma unroll
  for (int k = 0; k < 9; ++k) m.r[k] = q[k];  // shared memory (staged) or global through L1
  return m;
}
__device__ __forceinline__ void rotate(const Mat3& m, double& x, double& y, double& z) {
  const double nx = m.r[0] * x + m.r[1] * y + m.r[2] * z;
  const double ny = m.r[3] * x + m.r[4] * y + m.r[5] * z;
  const double nz = m.r[6] * x + m.r[7] * y + m.r[8] * z;
  x = nx;
  y = ny;
  z = nz;
}

// one interval on spin s (on the fly): precession (+ relaxation), fp64 — engine.py:288-302
template <int S, class SP>
__device__ __forceinline__ void interval(const KParams& kp, SP& sp, int s, int flags, int cls, double dt,
                                         double dmx, double dmy, double dmz) {
  if (!(flags & EV_MOVE) || !sp.act(s)) return;
  const int64_t i = sp.idx(s);
  const SC c = load_sc(kp, i);
  const double2 e = cls >= 0 ? relax_pair(kp, cls, i) : make_double2(1.0, 1.0);
  double cs, ms;
  phase_factor(theta_of(c, dt, dmx, dmy, dmz), cs, ms);
  const double x = sp.mx(s), y = sp.my(s);
  sp.mx(s) = e.y * (cs * x - ms * y);  // clockwise: (c - i s)(x + i y), bloch.py:10-17
  sp.my(s) = e.y * (cs * y + ms * x);
  if (cls >= 0) sp.mz(s) = fma(sp.mz(s), e.x, c.m0 * (1.0 - e.x));
}

// the fused pulse on its own pass over the state (paths that do not load the state anyway)
template <int S, class SP>
__device__ __forceinline__ void apply_pre(const double* mats, SP& sp, int pre, int mode) {
  const Mat3 m = load_mat(mats, pre);
  if (mode == 1) {  // about x: (x, r4 y + r5 z, r7 y + r8 z)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double y = sp.my(s), z = sp.mz(s);
      sp.my(s) = m.r[4] * y + m.r[5] * z;
      sp.mz(s) = m.r[7] * y + m.r[8] * z;
    }
    return;
  }
  if (mode == 2) {  // about y: (r0 x + r2 z, y, r6 x + r8 z)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double x = sp.mx(s), z = sp.mz(s);
      sp.mx(s) = m.r[0] * x + m.r[2] * z;
      sp.mz(s) = m.r[6] * x + m.r[8] * z;
    }
    return;
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    double x = sp.mx(s), y = sp.my(s), z = sp.mz(s);
    rotate(m, x, y, z);
    sp.mx(s) = x;
    sp.my(s) = y;
    sp.mz(s) = z;
  }
}

// receive-weighted transverse magnetisation of the (fp64) state summed over the
// thread's spins into slots [base, base+NC) — engine.py:303-305
template <typename R, int S, int NC>
__device__ __forceinline__ void record_state(const KParams& kp, Spins<S>& sp, R (&ar)[kChunkSlots],
                                             R (&ai)[kChunkSlots], int base) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (!sp.act(s)) continue;
      double2 w = make_double2(1.0, 0.0);
      if (kp.w != nullptr) w = __ldg(reinterpret_cast<const double2*>(kp.w) + static_cast<int64_t>(c) * kp.n + sp.idx(s));
      const double x = sp.mx(s), y = sp.my(s);
      re += w.x * x - w.y * y;
      im += w.x * y + w.y * x;
    }
    ar[base + c] = static_cast<R>(re);
    ai[base + c] = static_cast<R>(im);
  }
}

// ---------------------------------------------------------------------------
// ADC window sample recurrence
// ---------------------------------------------------------------------------

// generic (any R, any NC): u_s <- u_s * z_s before every sample but a leading one
template <typename R, int S, int NC, bool FULL, bool LEAD>
__device__ __forceinline__ void window_chunk(R (&ur)[S], R (&ui)[S], const R (&zr)[S], const R (&zi)[S],
                                             const R (&wr)[NC][S], const R (&wi)[NC][S], R (&ar)[kChunkSlots],
                                             R (&ai)[kChunkSlots], int ck) {
  constexpr int kSamp = kChunkSlots / NC;
#pragma unroll
  for (int j = 0; j < kSamp; ++j) {
    if (!FULL && j >= ck) {
#pragma unroll
      for (int c = 0; c < NC; ++c) ar[j * NC + c] = ai[j * NC + c] = R(0);
      continue;
    }
    if (!(LEAD && j == 0)) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const R x = ur[s], y = ui[s];
        ur[s] = x * zr[s] - y * zi[s];
        ui[s] = x * zi[s] + y * zr[s];
      }
    }
    if (NC == 1) {
      R re = ur[0], im = ui[0];
#pragma unroll
      for (int s = 1; s < S; ++s) {
        re += ur[s];
        im += ui[s];
      }
      ar[j] = re;
      ai[j] = im;
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        R re = R(0), im = R(0);
#pragma unroll
        for (int s = 0; s < S; ++s) {
          re += wr[c][s] * ur[s] - wi[c][s] * ui[s];
          im += wr[c][s] * ui[s] + wi[c][s] * ur[s];
        }
        ar[j * NC + c] = re;
        ai[j * NC + c] = im;
      }
    }
  }
}

// fp32, single coil: spins packed in pairs, one FMUL2+FMUL2+FFMA2+FFMA2 per
// pair-sample (sm_100 f32x2 datapath), FADD2 for the per-thread spin sum.
template <int P, bool FULL, bool LEAD>
__device__ __forceinline__ void window_chunk_f2(float2 (&U)[P], float2 (&V)[P], const float2 (&ZR)[P],
                                                const float2 (&ZI)[P], float (&ar)[kChunkSlots],
                                                float (&ai)[kChunkSlots], int ck) {
#pragma unroll
  for (int j = 0; j < kChunkSlots; ++j) {
    if (!FULL && j >= ck) {
      ar[j] = ai[j] = 0.f;
      continue;
    }
    if (!(LEAD && j == 0)) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float2 a = U[p];
        const float2 nzi = make_float2(-ZI[p].x, -ZI[p].y);  // folded into FMUL2's negate modifier
        const float2 t1 = __fmul2_rn(V[p], nzi);              // -v*zi
        const float2 t2 = __fmul2_rn(V[p], ZR[p]);            //  v*zr
        U[p] = __ffma2_rn(a, ZR[p], t1);                      // u*zr - v*zi
        V[p] = __ffma2_rn(a, ZI[p], t2);                      // u*zi + v*zr
      }
    }
    float2 sr = U[0], si = V[0];
#pragma unroll
    for (int p = 1; p < P; ++p) {
      sr = __fadd2_rn(sr, U[p]);
      si = __fadd2_rn(si, V[p]);
    }
    ar[j] = sr.x + sr.y;
    ai[j] = si.x + si.y;
  }
}

// fp32, NC coils (even): track m per spin (scalar complex multiply) and
// multiply-accumulate the coil weights packed two coils per FFMA2:
//   (re_c, re_c+1) += (wr_c, wr_c+1) ur - (wi_c, wi_c+1) ui
//   (im_c, im_c+1) += (wr_c, wr_c+1) ui + (wi_c, wi_c+1) ur
template <int S, int NC, bool FULL, bool LEAD>
__device__ __forceinline__ void window_chunk_mc2(float (&ur)[S], float (&ui)[S], const float (&zr)[S],
                                                 const float (&zi)[S], const float2 (&WR)[NC / 2][S],
                                                 const float2 (&WI)[NC / 2][S], float (&ar)[kChunkSlots],
                                                 float (&ai)[kChunkSlots], int ck) {
  constexpr int kSamp = kChunkSlots / NC;
  constexpr int PC = NC / 2;
#pragma unroll
  for (int j = 0; j < kSamp; ++j) {
    if (!FULL && j >= ck) {
#pragma unroll
      for (int c = 0; c < NC; ++c) ar[j * NC + c] = ai[j * NC + c] = 0.f;
      continue;
    }
    if (!(LEAD && j == 0)) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const float x = ur[s], y = ui[s];
        ur[s] = x * zr[s] - y * zi[s];
        ui[s] = x * zi[s] + y * zr[s];
      }
    }
    float2 re[PC], im[PC];
#pragma unroll
    for (int p = 0; p < PC; ++p) re[p] = im[p] = make_float2(0.f, 0.f);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const float2 u2 = make_float2(ur[s], ur[s]), v2 = make_float2(ui[s], ui[s]);
      const float2 nv2 = make_float2(-ui[s], -ui[s]);
#pragma unroll
      for (int p = 0; p < PC; ++p) {
        re[p] = __ffma2_rn(WR[p][s], u2, re[p]);
        re[p] = __ffma2_rn(WI[p][s], nv2, re[p]);
        im[p] = __ffma2_rn(WR[p][s], v2, im[p]);
        im[p] = __ffma2_rn(WI[p][s], u2, im[p]);
      }
    }
#pragma unroll
    for (int p = 0; p < PC; ++p) {
      ar[j * NC + 2 * p] = re[p].x;
      ar[j * NC + 2 * p + 1] = re[p].y;
      ai[j * NC + 2 * p] = im[p].x;
      ai[j * NC + 2 * p + 1] = im[p].y;
    }
  }
}


// ---------------------------------------------------------------------------
// ADC windows on the tensor cores (fp32 mode, one receive weight)
// ---------------------------------------------------------------------------
//
// The window's samples are S_k = sum_s u_s z_s^k (k = 0..cnt-1, u_s the
// weighted transverse magnetisation at the first sample, z_s the per-sample
// factor).  Split k = 64 j + 8 a + b: S_k = sum_s z_s^b * (u_s z_s^(64 j + 8 a)),
// a complex (8 x spins) x (spins x 8) product per 64-sample tile — a GEMM whose
// contraction runs over the spins.  Embedded as a real m16n8k8 product:
//   A[(b, re)][(s, re)] = Re z^b   A[(b, re)][(s, im)] = -Im z^b
//   A[(b, im)][(s, re)] = Im z^b   A[(b, im)][(s, im)] =  Re z^b
//   B[(s, re)][a] = Re V           B[(s, im)][a] = Im V,  V = u z^(64 j + 8 a)
// so D[(b, re/im)][a] = Re/Im S_(64 j + 8 a + b).  One warp contracts its own
// 32*S spins, 4 per mma (k = 8 = 4 spins x re/im), accumulating in fp32
// registers; the per-sample spin sum never touches the CUDA cores.
//
// Precision: each operand is split x = hi + lo with both parts exact tf32
// values (low 13 mantissa bits zero) and the product formed as
// hi*hi + hi*lo + lo*hi (3 mma) — ~2^-20 relative per product, below the
// fp32 recurrence it replaces.  Lane (g = lane/4, t = lane%4) needs z^g and
// u z^(8 g) of spin t; it forms them from z by squarings.


struct cf {
  float r, i;
};
__device__ __forceinline__ cf cmul(cf a, cf b) { return cf{a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ cf csq(cf a) { return cf{a.r * a.r - a.i * a.i, 2.f * a.r * a.i}; }
__device__ __forceinline__ cf csel(bool c, cf a) { return c ? a : cf{1.f, 0.f}; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Window products: x = hi + lo with hi exact in tf32.  BLOCH_MMA_SPLIT 3: three tf32
// passes (hi hi + hi lo + lo hi, lo masked to tf32).  BLOCH_MMA_SPLIT 2 (default): the
// hi hi pass in tf32, and both cross terms in ONE bf16 m16n8k16 whose K concatenates
// (A_hi | A_lo) against (B_lo ; B_hi).  The bf16 operands are the top 16 bits of the
// fp32 words (one PRMT per pair, no F2FP conversion): the cross terms are ~2^-11 of
// the product and carry 2^-8 relative truncation, ~2^-19 overall — the same order as
// the fp32 recurrence.  The bf16 pipe runs twice the tf32 MAC rate, so the two cross
// terms cost one tf32 pass: 2 instead of 3 tensor-pipe units per product.
#ifndef BLOCH_MMA_SPLIT
#define BLOCH_MMA_SPLIT 2
#endif
#ifndef BLOCH_PACKED_ADVANCE
#define BLOCH_PACKED_ADVANCE 1
#endif
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
#if BLOCH_MMA_SPLIT == 3
  lo = __float_as_uint(x - __uint_as_float(hi)) & 0xffffe000u;
#else
  lo = __float_as_uint(x - __uint_as_float(hi));  // exact; the bf16 pack keeps its top 16 bits
#endif
}

#ifndef BLOCH_KB_UNROLL
#define BLOCH_KB_UNROLL 2
#endif
constexpr int kKbUnroll = BLOCH_KB_UNROLL;  // k-block loop unroll of the single-coil window rounds

// {x, y} -> bf16x2 (x in the low half) by truncation: the high halves of the fp32 words
__device__ __forceinline__ uint32_t pack_bf16(uint32_t x, uint32_t y) { return __byte_perm(x, y, 0x7632); }

__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Per-warp stage of one round (one spin per lane): for lane-spin q and power g,
// (Re z^g, Im z^g, Re V_g, Im V_g) with V_g = u z^(8 g) at [g][q ^ 4 (g & 1)]
// (the swizzle makes both the staging stores and the k-block loads
// conflict-free), then z^64 per spin.
constexpr int kStageFloat4 = 8 * 32;
constexpr int kStageBytes = kStageFloat4 * 16 + 32 * 8 + 32 * 16;  // + z^64 per lane + cp.async slot (Cpre, z) per lane
__device__ __forceinline__ int stage_idx(int g, int q) { return g * 32 + (q ^ ((g & 1) << 2)); }

// One lane's spin into the stage: its 8 powers z^g and 8 values u z^(8g).
__device__ __forceinline__ void stage_spin(float4* __restrict__ st, float2* __restrict__ z64s, int lane, cf u, cf z) {
  cf zg{1.f, 0.f};
  const cf z2 = csq(z), z4 = csq(z2), z8 = csq(z4);
  cf v = u;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    st[stage_idx(g, lane)] = make_float4(zg.r, zg.i, v.r, v.i);
    zg = cmul(zg, z);
    v = cmul(v, z8);
  }
  const cf z64 = csq(csq(csq(z8)));
  z64s[lane] = make_float2(z64.r, z64.i);
}

// The 8 k-blocks (4 spins each) of one staged round into the NT tile
// accumulators.  The three split products are issued pass-major across the NT
// independent accumulators so consecutive mma never wait on each other.
template <int NT, int MT>
__device__ __forceinline__ void mma_round_t(const float4* __restrict__ st, const float2* __restrict__ z64s, int lane,
                                            float (&acc)[MT][4]) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll kKbUnroll
  for (int kb = 0; kb < 8; ++kb) {
    const int q = 4 * kb + t;
    const float4 e = st[stage_idx(g, q)];
    const float2 w = z64s[q];
    const cf z64{w.x, w.y};
    uint32_t arh, arl, aih, ail;
    split_tf32(e.x, arh, arl);
    split_tf32(e.y, aih, ail);
    const uint32_t naih = aih ^ 0x80000000u, nail = ail ^ 0x80000000u;
    uint32_t brh[NT], brl[NT], bih[NT], bil[NT];
#if BLOCH_MMA_SPLIT == 3 || !BLOCH_PACKED_ADVANCE
    cf v{e.z, e.w};
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      split_tf32(v.r, brh[j], brl[j]);
      split_tf32(v.i, bih[j], bil[j]);
      if (j + 1 < NT) v = cmul(v, z64);
    }
#else
    // packed (FFMA2/FMUL2) tile advance v <- v z^64 and residuals lo = v - hi: half the issue slots
    float2 v = make_float2(e.z, e.w);
    const float2 nz = make_float2(-z64.i, z64.r), zz = make_float2(z64.r, z64.i), m1 = make_float2(-1.f, -1.f);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      brh[j] = __float_as_uint(v.x) & 0xffffe000u;
      bih[j] = __float_as_uint(v.y) & 0xffffe000u;
      const float2 lo = __ffma2_rn(make_float2(__uint_as_float(brh[j]), __uint_as_float(bih[j])), m1, v);
      brl[j] = __float_as_uint(lo.x);
      bil[j] = __float_as_uint(lo.y);
      if (j + 1 < NT) v = __ffma2_rn(make_float2(v.y, v.y), nz, __fmul2_rn(make_float2(v.x, v.x), zz));
    }
#endif
#pragma unroll
    for (int j = 0; j < NT; ++j) mma_tf32(acc[j], arh, aih, naih, arh, brh[j], bih[j]);
#if BLOCH_MMA_SPLIT == 3
#pragma unroll
    for (int j = 0; j < NT; ++j) mma_tf32(acc[j], arh, aih, naih, arh, brl[j], bil[j]);
#pragma unroll
    for (int j = 0; j < NT; ++j) mma_tf32(acc[j], arl, ail, nail, arl, brh[j], bih[j]);
#else
    // k16 slots of lane t: 2t, 2t+1 = (re, im) of its spin against (A_hi, B_lo); 2t+8, 2t+9 against (A_lo, B_hi)
    const uint32_t c0 = pack_bf16(arh, naih), c1 = pack_bf16(aih, arh), c2 = pack_bf16(arl, nail),
                   c3 = pack_bf16(ail, arl);
#pragma unroll
    for (int j = 0; j < NT; ++j) mma_bf16(acc[j], c0, c1, c2, c3, pack_bf16(brl[j], bil[j]), pack_bf16(brh[j], bih[j]));
#endif
  }
}

// MT: tiles per pass (accumulator rows), 8 in the basic kernel, 4 in the full one
template <int MT>
__device__ __forceinline__ void mma_round(const float4* __restrict__ st, const float2* __restrict__ z64s, int lane,
                                          int ntile, float (&acc)[MT][4]) {
  switch (ntile) {
    case 8: if constexpr (MT >= 8) mma_round_t<8, MT>(st, z64s, lane, acc); break;
    case 7: if constexpr (MT >= 7) mma_round_t<7, MT>(st, z64s, lane, acc); break;
    case 6: if constexpr (MT >= 6) mma_round_t<6, MT>(st, z64s, lane, acc); break;
    case 5: if constexpr (MT >= 5) mma_round_t<5, MT>(st, z64s, lane, acc); break;
    case 4: mma_round_t<4, MT>(st, z64s, lane, acc); break;
    case 3: mma_round_t<3, MT>(st, z64s, lane, acc); break;
    case 2: mma_round_t<2, MT>(st, z64s, lane, acc); break;
    default: mma_round_t<1, MT>(st, z64s, lane, acc); break;
  }
}

// Multi-coil windows: S_(k,c) = sum_s z_s^b * (w_(c,s) u_s z_s^(64 j + 8 a)).  The
// A operand (z^b) is shared by the coils; each coil has its own B = w_c V.  One
// 64-sample tile at a time (NC x 4 accumulators), rounds of one spin per lane
// inside; the coil weights (fp32, spin-major) arrive by cp.async one round
// ahead, double-buffered.
template <int NC>
struct McStage {
  static constexpr int kW = 32 * NC * 8;                            // one weight buffer: [lane spin][coil] float2
  static constexpr int kBytes = kStageFloat4 * 16 + 2 * kW + 32 * 16;  // + cp.async slot (Cpre, z) per lane
};

__device__ __forceinline__ void stage_spin_mc(float4* __restrict__ st, int lane, cf u, cf z) {
  const cf z8 = csq(csq(csq(z)));
  cf zg{1.f, 0.f}, v = u;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    st[stage_idx(g, lane)] = make_float4(zg.r, zg.i, v.r, v.i);
    zg = cmul(zg, z);
    v = cmul(v, z8);
  }
}

template <int NC>
__device__ __forceinline__ void mma_round_mc(const float4* __restrict__ st, const float2* __restrict__ wst, int lane,
                                             float (&acc)[NC][4]) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll 1
  for (int kb = 0; kb < 8; ++kb) {
    const int q = 4 * kb + t;
    const float4 e = st[stage_idx(g, q)];
    uint32_t arh, arl, aih, ail;
    split_tf32(e.x, arh, arl);
    split_tf32(e.y, aih, ail);
    const uint32_t naih = aih ^ 0x80000000u, nail = ail ^ 0x80000000u;
    const cf v{e.z, e.w};
    uint32_t brh[NC], brl[NC], bih[NC], bil[NC];
    const float4* wq = reinterpret_cast<const float4*>(wst + q * NC);
#pragma unroll
    for (int c2 = 0; c2 < NC / 2; ++c2) {
      const float4 w2 = wq[c2];
      const cf b0 = cmul(cf{w2.x, w2.y}, v), b1 = cmul(cf{w2.z, w2.w}, v);
      split_tf32(b0.r, brh[2 * c2], brl[2 * c2]);
      split_tf32(b0.i, bih[2 * c2], bil[2 * c2]);
      split_tf32(b1.r, brh[2 * c2 + 1], brl[2 * c2 + 1]);
      split_tf32(b1.i, bih[2 * c2 + 1], bil[2 * c2 + 1]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) mma_tf32(acc[c], arh, aih, naih, arh, brh[c], bih[c]);
#if BLOCH_MMA_SPLIT == 3
#pragma unroll
    for (int c = 0; c < NC; ++c) mma_tf32(acc[c], arh, aih, naih, arh, brl[c], bil[c]);
#pragma unroll
    for (int c = 0; c < NC; ++c) mma_tf32(acc[c], arl, ail, nail, arl, brh[c], bih[c]);
#else
    const uint32_t c0 = pack_bf16(arh, naih), c1 = pack_bf16(aih, arh), c2 = pack_bf16(arl, nail),
                   c3 = pack_bf16(ail, arl);
#pragma unroll
    for (int c = 0; c < NC; ++c) mma_bf16(acc[c], c0, c1, c2, c3, pack_bf16(brl[c], bil[c]), pack_bf16(brh[c], bih[c]));
#endif
  }
}

// Eight coils: the coils go into the MMA's M dimension instead.  For the 8 samples n of MMA m
// (k = 64 j + 8 m + n) and a k-block of 4 spins,
//   D[(c, re/im)][n] += sum_s [[Re w_cs, -Im w_cs], [Im w_cs, Re w_cs]] (Re v_sn, Im v_sn),  v_sn = u_s z_s^k
// so A is the spin's coil weights (prepared once per k-block, shared by the tile's 8 MMAs) and B the
// per-sample value u z^k, shared by all coils and advanced by z^8 from one MMA to the next — instead
// of forming and splitting w_c V for every coil of every k-block.  The stage holds (u z^(64 j + g), z^8)
// per (g, spin): lane (g, t) feeds sample n = g of spin 4 kb + t, and holds coil g of samples 2t, 2t + 1.
__device__ __forceinline__ void stage_spin_mc8(float4* __restrict__ st, int lane, cf u, cf z) {
  const cf z8 = csq(csq(csq(z)));
  cf v = u;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    st[stage_idx(g, lane)] = make_float4(v.r, v.i, z8.r, z8.i);
    v = cmul(v, z);
  }
}

__device__ __forceinline__ void mma_round_mc8(const float4* __restrict__ st, const float2* __restrict__ wst, int lane,
                                              float (&acc)[8][4]) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll 1
  for (int kb = 0; kb < 8; ++kb) {
    const int q = 4 * kb + t;
    const float4 e = st[stage_idx(g, q)];  // u z^(64 j + g) of spin q, z^8
    const float2 w = wst[q * 8 + g];        // receive weight of coil g for spin q
    uint32_t arh, arl, aih, ail;
    split_tf32(w.x, arh, arl);
    split_tf32(w.y, aih, ail);
    const uint32_t naih = aih ^ 0x80000000u, nail = ail ^ 0x80000000u;
    const uint32_t c0 = pack_bf16(arh, naih), c1 = pack_bf16(aih, arh), c2 = pack_bf16(arl, nail),
                   c3 = pack_bf16(ail, arl);
    float2 v = make_float2(e.x, e.y);
    const float2 nz = make_float2(-e.w, e.z), zz = make_float2(e.z, e.w), m1 = make_float2(-1.f, -1.f);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const uint32_t brh = __float_as_uint(v.x) & 0xffffe000u, bih = __float_as_uint(v.y) & 0xffffe000u;
      const float2 lo = __ffma2_rn(make_float2(__uint_as_float(brh), __uint_as_float(bih)), m1, v);
      mma_tf32(acc[m], arh, aih, naih, arh, brh, bih);
      mma_bf16(acc[m], c0, c1, c2, c3, pack_bf16(__float_as_uint(lo.x), __float_as_uint(lo.y)), pack_bf16(brh, bih));
      if (m < 7) v = __ffma2_rn(make_float2(v.y, v.y), nz, __fmul2_rn(make_float2(v.x, v.x), zz));
    }
  }
}

// ---------------------------------------------------------------------------
// tabulated chirps in the fp32 mode
// ---------------------------------------------------------------------------

// A chirp (OP_CHIRP: K sampled intervals whose moments grow linearly) applies
// r_k = r0 q^k to the transverse magnetisation before sample k.  The fp64 state
// leaves the run through its closed form: m -> C_total m (C_total = prod r_k, the
// plane of the whole run's (K dt, K d0 + K(K-1)/2 dd)) and mz -> A mz + B, applied
// at the first block.  The samples only feed the fp32 ADC sums, so they run as an
// fp32 recurrence u <- u r, r <- r q from u = w m: 8 FP32 multiply-adds per
// sample instead of ~10 fp64 operations and two F2F conversions.  Blocks of
// kBlk samples are spin-outer; between blocks each spin's (u, r) waits in this
// warp's window stage (free outside windows).
template <int S, int NC>
__device__ __forceinline__ void chirp_f32(const KParams& kp, const DevOp* op, Spins<S>& sp, Strip<float>& strip,
                                          unsigned char* smem_raw, int cnt, int s0) {
  constexpr int kSampPerChunk = kChunkSlots / NC;
  constexpr int kBlk = 2 * kSampPerChunk;
  constexpr int G = S < 4 ? S : 4;
  const int lane = threadIdx.x & 31;
  constexpr size_t kStage = NC == 1 ? kStageBytes : McStage<NC>::kBytes;
  static_assert(S * 32 * 16 <= kStageFloat4 * 16, "chirp stash exceeds the window stage");
  float4* stash = reinterpret_cast<float4*>(smem_raw + static_cast<size_t>(3 * S) * sp.bd * sizeof(double) +
                                            static_cast<size_t>(threadIdx.x >> 5) * kStage);
  const float2 *pr0 = plane32_at(kp, __ldg(&op->pl[0]), 0), *pq = plane32_at(kp, __ldg(&op->pl[1]), 0);
  const double2* pct = plane(kp, op, 2);
  const float qsgn = (__ldg(&op->tmode) & 1) ? -1.f : 1.f;
  // entry: u = w m into the stash, then the state leaves through the closed form (loads of a group of
  // spins issued together, as in the interval handler)
#pragma unroll
  for (int s = 0; s < S; ++s) {
    double2 w = make_double2(1.0, 0.0);
    if (NC == 1 && kp.w != nullptr && sp.act(s)) w = __ldg(reinterpret_cast<const double2*>(kp.w) + sp.idx(s));
    const double x = sp.mx(s), y = sp.my(s);
    stash[s * 32 + lane] =
        make_float4(static_cast<float>(w.x * x - w.y * y), static_cast<float>(w.x * y + w.y * x), 0.f, 0.f);
  }
#pragma unroll
  for (int g0 = 0; g0 < S; g0 += G) {
    double2 ct[G], ab[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t i = sp.act(g0 + g) ? sp.idx(g0 + g) : 0;
      ct[g] = __ldg(pct + i);
      ab[g] = ab_at(kp, op, 3, i);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int s = g0 + g;
      const double x = sp.mx(s), y = sp.my(s);
      sp.mx(s) = ct[g].x * x - ct[g].y * y;
      sp.my(s) = ct[g].x * y + ct[g].y * x;
      sp.mz(s) = fma(sp.mz(s), ab[g].x, ab[g].y);
    }
  }
  // samples: spin-outer per block; the next spin's (r0, q) loads are in flight while this spin runs
  for (int k0 = 0; k0 < cnt; k0 += kBlk) {
    const int cb = min(kBlk, cnt - k0);
    float ar[2][kChunkSlots], ai[2][kChunkSlots];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < kChunkSlots; ++j) ar[h][j] = ai[h][j] = 0.f;
    float2 nq = __ldg(pq + (sp.act(0) ? sp.idx(0) : 0)), nr = k0 == 0 ? __ldg(pr0 + (sp.act(0) ? sp.idx(0) : 0))
                                                                      : make_float2(0.f, 0.f);
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      const float2 qd = nq, r0 = nr;
      if (s + 1 < S) {
        const int64_t in = sp.act(s + 1) ? sp.idx(s + 1) : 0;
        nq = __ldg(pq + in);
        if (k0 == 0) nr = __ldg(pr0 + in);
      }
      if (!sp.act(s)) continue;
      const int64_t i = sp.idx(s);
      const cf q{qd.x, qsgn * qd.y};
      const float4 v = stash[s * 32 + lane];
      cf u{v.x, v.y}, r{v.z, v.w};
      if (k0 == 0) r = cf{r0.x, r0.y};
      cf w[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        w[c] = cf{1.f, 0.f};
        if (NC > 1 && kp.w32 != nullptr) {
          const float2 wf = __ldg(kp.w32 + i * NC + c);
          w[c] = cf{wf.x, wf.y};
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int j = 0; j < kSampPerChunk; ++j) {
          if (h * kSampPerChunk + j < cb) {
            u = cmul(u, r);
            r = cmul(r, q);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              if (NC == 1) {
                ar[h][j] += u.r;
                ai[h][j] += u.i;
              } else {
                ar[h][j * NC + c] += w[c].r * u.r - w[c].i * u.i;
                ai[h][j * NC + c] += w[c].r * u.i + w[c].i * u.r;
              }
            }
          }
        }
      }
      if (k0 + kBlk < cnt) stash[s * 32 + lane] = make_float4(u.r, u.i, r.r, r.i);
    }
    strip.push(ar[0], ai[0], min(kSampPerChunk, cb) * NC, (s0 + k0) * NC);
    if (cb > kSampPerChunk) strip.push(ar[1], ai[1], (cb - kSampPerChunk) * NC, (s0 + k0 + kSampPerChunk) * NC);
  }
}

// ---------------------------------------------------------------------------
// the integrator
// ---------------------------------------------------------------------------

// kFull: the program uses RF trains, chirps or generic sampled events.  Programs
// made only of pulses, intervals and uniform windows (spin/turbo-spin echoes) run
// a kernel without those handlers: less register pressure in the hot loop.
// BD: the block size as a compile-time constant (0: blockDim.x).  The spin state
// [3][S][bd] is addressed (component, slot) x bd + thread on every access; with a
// constant bd those offsets are immediates.
template <typename R, int S, int NC, bool kFull, int BD, bool kWin>
__global__ void __launch_bounds__(kWin ? KernelTraits<R, S, NC>::kMaxThreads : KernelTraits<R, S, NC>::kMaxThreadsNoWin,
                                  kWin ? KernelTraits<R, S, NC>::kMinBlocks : KernelTraits<R, S, NC>::kMinBlocksNoWin)
    integrate_kernel(const KParams kp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kSampPerChunk = kChunkSlots / NC;
  constexpr bool kPacked = sizeof(R) == 4 && NC == 1 && (S % 2 == 0);  // FFMA2 recurrence over spin pairs
  constexpr bool kMma1 = sizeof(R) == 4 && NC == 1;                     // single-coil tensor-core windows
  const int bd = BD ? BD : static_cast<int>(blockDim.x);
  const int nw = bd >> 5;
  // registers hold the state of up to 4 spins per thread; 8 spill (measured: config 1 S=8 3.94 vs 3.26 ms
  // in shared memory; S <= 4 3-10% faster in registers, profiles/r2v_register_state_ab.txt)
  constexpr bool kRegState = !kFull && !kWin && S <= 4;
  Spins<S, kRegState> sp;
  sp.sm = reinterpret_cast<double*>(smem_raw);
  sp.base = static_cast<int64_t>(blockIdx.x) * kp.spins_per_cta + threadIdx.x;
  sp.bd = bd;
  sp.n = kp.n;
  sp.init_active();
  // the fused pulse matrices: staged in shared memory by the register-state kernels (their shared memory
  // is otherwise unused; each matrix is read once per op by every warp, an L2 round trip from global)
  const double* mats = kp.mats;
  // ... and the progression running factors of this thread's spins, [class][S][bd] after the matrices: an
  // L2 read-modify-write per member otherwise (config 2: the kernel's top stall)
  double2* progs = nullptr;
  if constexpr (kRegState) {
    if (kp.n_mats_smem > 0) {
      double* sm = reinterpret_cast<double*>(smem_raw);
      for (int k = threadIdx.x; k < 9 * kp.n_mats_smem; k += blockDim.x) sm[k] = __ldg(kp.mats + k);
      __syncthreads();
      mats = sm;
    }
    if (kp.n_prog_smem > 0) {
      progs = reinterpret_cast<double2*>(smem_raw + ((static_cast<size_t>(kp.n_mats_smem) * 72 + 15) & ~size_t(15)));
      for (int pc = 0; pc < kp.n_prog_smem; ++pc) {
        const double2* src = kp.planes + static_cast<int64_t>(kp.prog_plane[pc]) * kp.n;
#pragma unroll
        for (int s = 0; s < S; ++s)
          progs[(pc * S + s) * bd + threadIdx.x] = sp.act(s) ? src[sp.idx(s)] : make_double2(1.0, 0.0);
      }
    }
  }
  Strip<R> strip;  // one partial row per warp of the grid
  strip.lane = threadIdx.x & 31;
  strip.row = reinterpret_cast<R*>(kp.partial) +
              (static_cast<int64_t>(blockIdx.x) * nw + (threadIdx.x >> 5)) * kp.part_stride;

#pragma unroll
  for (int s = 0; s < S; ++s) {
    const bool a = sp.act(s);
    const int64_t i = a ? sp.idx(s) : 0;
    sp.mx(s) = a ? kp.mx0[i] : 0.0;
    sp.my(s) = a ? kp.my0[i] : 0.0;
    sp.mz(s) = a ? kp.mz0[i] : 0.0;
  }

  for (int o = kp.op_begin; o < kp.n_ops; ++o) {
    const DevOp* op = kp.ops + o;
    const int kind = __ldg(&op->kind);

    if (kind == OP_ROT) {  // engine.py:277-283
      double r[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) r[k] = __ldg(&op->p[k]);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double x = sp.mx(s), y = sp.my(s), z = sp.mz(s);
        sp.mx(s) = r[0] * x + r[1] * y + r[2] * z;
        sp.my(s) = r[3] * x + r[4] * y + r[5] * z;
        sp.mz(s) = r[6] * x + r[7] * y + r[8] * z;
      }
      continue;
    }

    if (kind == OP_EVENT) {
      const int flags = __ldg(&op->count), snap = __ldg(&op->aux), cls = __ldg(&op->cls), rc = __ldg(&op->rot),
                pg = __ldg(&op->prg), pre = __ldg(&op->pre);
      if constexpr (!kFull) {  // a fused pulse (basic programs only): its own pass over the state
        if (pre >= 0) apply_pre<S>(mats, sp, pre, __ldg(&op->tmode));
      }
      // Two-phase per group of G spins: issue every table load of the group
      // before any store, so the L2 round trips overlap instead of serialising
      // behind possibly-aliasing shared/global stores.
      constexpr int G = S < 4 ? S : 4;
      if (rc >= 0) {  // repeated interval: tabulated propagator
        const double2 *pc = plane(kp, op, 0), *pab = plane(kp, op, 1);
#pragma unroll
        for (int g0 = 0; g0 < S; g0 += G) {
          double2 c[G], ab[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int64_t i = sp.act(g0 + g) ? sp.idx(g0 + g) : 0;
            c[g] = __ldg(pc + i);
            ab[g] = __ldg(pab + i);
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int s = g0 + g;
            const double x = sp.mx(s), y = sp.my(s);
            sp.mx(s) = c[g].x * x - c[g].y * y;
            sp.my(s) = c[g].x * y + c[g].y * x;
            sp.mz(s) = fma(sp.mz(s), ab[g].x, ab[g].y);
          }
        }
      } else if (kRegState && pg >= 0 && progs != nullptr) {  // progression member, running factor in smem
        const int adv = __ldg(&op->flags);  // 0 (last member), 1 or 2
        const double2 *pq = plane(kp, op, adv == 2 ? 2 : 1), *pab = plane(kp, op, 3);  // q or q^2
        double2 c[S], ab[S], q[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int64_t i = sp.act(s) ? sp.idx(s) : 0;
          c[s] = progs[(pg * S + s) * bd + threadIdx.x];
          ab[s] = __ldg(pab + i);
          q[s] = adv ? __ldg(pq + i) : make_double2(1.0, 0.0);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double x = sp.mx(s), y = sp.my(s);
          sp.mx(s) = c[s].x * x - c[s].y * y;
          sp.my(s) = c[s].x * y + c[s].y * x;
          sp.mz(s) = fma(sp.mz(s), ab[s].x, ab[s].y);
          if (adv)
            progs[(pg * S + s) * bd + threadIdx.x] = make_double2(c[s].x * q[s].x - c[s].y * q[s].y,
                                                                  c[s].x * q[s].y + c[s].y * q[s].x);
        }
      } else if (pg >= 0) {  // one member of an interval progression: C, then C *= q^adv
        const int adv = __ldg(&op->flags);  // 0 (last member), 1 or 2
        double2* prun = kp.planes + static_cast<int64_t>(__ldg(&op->pl[0])) * kp.n;
        const uint64_t l2pol = l2_evict_last();
        const double2 *pq = plane(kp, op, adv == 2 ? 2 : 1), *pab = plane(kp, op, 3);  // q or q^2
#pragma unroll
        for (int g0 = 0; g0 < S; g0 += G) {
          double2 c[G], ab[G], q[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int64_t i = sp.act(g0 + g) ? sp.idx(g0 + g) : 0;
            c[g] = ld_keep(prun + i, l2pol);  // running factor: L2-coherent (rewritten below), kept in L2
            ab[g] = __ldg(pab + i);
            q[g] = adv ? __ldg(pq + i) : make_double2(1.0, 0.0);
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int s = g0 + g;
            const double x = sp.mx(s), y = sp.my(s);
            sp.mx(s) = c[g].x * x - c[g].y * y;
            sp.my(s) = c[g].x * y + c[g].y * x;
            sp.mz(s) = fma(sp.mz(s), ab[g].x, ab[g].y);
            if (adv && sp.act(s))
              st_keep(prun + sp.idx(s), make_double2(c[g].x * q[g].x - c[g].y * q[g].y,
                                                       c[g].x * q[g].y + c[g].y * q[g].x), l2pol);
          }
        }
      } else {
        const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]), dmz = __ldg(&op->p[3]);
#pragma unroll
        for (int s = 0; s < S; ++s) interval<S>(kp, sp, s, flags, cls, dt, dmx, dmy, dmz);
      }
      if (snap >= 0 && kp.snaps != nullptr) {  // engine.py:306-308
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!sp.act(s)) continue;
          double* q = kp.snaps + (static_cast<int64_t>(snap) * kp.n + sp.idx(s)) * 3;
          q[0] = sp.mx(s);
          q[1] = sp.my(s);
          q[2] = sp.mz(s);
        }
      }
      continue;
    }

    if (kind == OP_UWIN || kind == OP_UCHIRP) {  // deferred window / chirp (contract.h): store u, apply the exit
      // window: u = Cpre m (times z without a leading no-op sample); chirp: u = w m (one coil), the samples
      // u r0^(k+1) q^(k(k+1)/2) are the contraction's
      const bool chirp = kind == OP_UCHIRP;
      const int lead = chirp ? 1 : __ldg(&op->aux), pre = __ldg(&op->pre);
      if constexpr (!kFull) {
        if (pre >= 0) apply_pre<S>(mats, sp, pre, __ldg(&op->tmode));
      }
      const int64_t row = __ldg(&op->s0);
      const double2 *pc = plane(kp, op, 2), *pab = plane(kp, op, 3);
      const int pcp = __ldg(&op->pl[0]), pz = __ldg(&op->pl[1]);
      constexpr int G = S < 4 ? S : 4;
#pragma unroll
      for (int g0 = 0; g0 < S; g0 += G) {
        double2 c[G], ab[G];
        float2 cp[G], zz[G];  // Cpre and z only form U (bf16 hi + lo, ~2^-16): fp32 suffices
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int64_t i = sp.act(g0 + g) ? sp.idx(g0 + g) : 0;
          c[g] = __ldg(pc + i);
          ab[g] = __ldg(pab + i);
          if (chirp) {  // the single-coil receive weight (several coils: applied by the contraction)
            const double2 w = (NC == 1 && kp.w != nullptr) ? __ldg(reinterpret_cast<const double2*>(kp.w) + i)
                                                           : make_double2(1.0, 0.0);
            cp[g] = make_float2(static_cast<float>(w.x), static_cast<float>(w.y));
            zz[g] = make_float2(1.f, 0.f);
          } else if constexpr (sizeof(R) == 4) {  // Cpre and z are PL_SAMPLE planes: float2 in the fp32 mode
            cp[g] = __ldg(plane32_at(kp, pcp, i));
            zz[g] = __ldg(plane32_at(kp, pz, i));
          } else {
            const double2 a = __ldg(plane_at(kp, pcp, i)), b = __ldg(plane_at(kp, pz, i));
            cp[g] = make_float2(static_cast<float>(a.x), static_cast<float>(a.y));
            zz[g] = make_float2(static_cast<float>(b.x), static_cast<float>(b.y));
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int s = g0 + g;
          const double x = sp.mx(s), y = sp.my(s);
          if (sp.act(s)) {
            uint32_t hi, lo;
            // u in fp32 (two conversions of the state) or in fp64 (split with fp64 residuals): equal to
            // ~2^-24, well inside the bf16 hi + lo split; the faster one per variant, measured same-box:
            // S = 8 fp32 3.23 vs 3.34 ms (config 1), S = 1 1.39 vs 1.41 (config 2 / 8), S = 4 fp64 8.65 vs
            // 8.80 (config 2) and 2.38 vs 2.63 (config 2 / 2), profiles/r2z_u_split_ab.txt
            constexpr bool kU32 = S == 8 || S == 1;
            if constexpr (kU32) {
              const float fx = static_cast<float>(x), fy = static_cast<float>(y);
              float ur = cp[g].x * fx - cp[g].y * fy, ui = cp[g].x * fy + cp[g].y * fx;
              if (!lead) {  // the first sample follows one interval
                const float t = ur * zz[g].x - ui * zz[g].y;
                ui = ur * zz[g].y + ui * zz[g].x;
                ur = t;
              }
              contract_split_f(ur, ui, hi, lo);
            } else {
              const double cr = cp[g].x, ci = cp[g].y, zr = zz[g].x, zi = zz[g].y;
              double ur = cr * x - ci * y, ui = cr * y + ci * x;
              if (!lead) {
                const double t = ur * zr - ui * zi;
                ui = ur * zi + ui * zr;
                ur = t;
              }
              contract_split(ur, ui, hi, lo);
            }
            const int64_t q = contract_u_index(kp.urows, row, sp.idx(s));
            __stcs(kp.uhi + q, hi);  // streamed: read back by the contraction
            __stcs(kp.ulo + q, lo);
          }
          sp.mx(s) = c[g].x * x - c[g].y * y;
          sp.my(s) = c[g].x * y + c[g].y * x;
          sp.mz(s) = fma(sp.mz(s), ab[g].x, ab[g].y);
        }
      }
      continue;
    }

    if (kind == OP_RFTRAIN && __ldg(&op->rot) >= 0) {
      // a reused RF train (train class): its tabulated affine propagator m -> A m + b (train_table_kernel);
      // every variant has it (a program whose trains are all classes needs no on-the-fly train code)
      const int tcl = __ldg(&op->rot);
      constexpr int G = S < 4 ? S : 4;
      const double2* tb = reinterpret_cast<const double2*>(kp.train) + static_cast<int64_t>(tcl) * kp.n * 6;
#pragma unroll
      for (int g0 = 0; g0 < S; g0 += G) {
        double2 a[G][6];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int64_t i = sp.act(g0 + g) ? sp.idx(g0 + g) : 0;
#pragma unroll
          for (int k = 0; k < 6; ++k) a[g][k] = __ldg(tb + i * 6 + k);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int s = g0 + g;
          const double x = sp.mx(s), y = sp.my(s), z = sp.mz(s);
          sp.mx(s) = fma(a[g][0].x, x, fma(a[g][0].y, y, fma(a[g][1].x, z, a[g][4].y)));
          sp.my(s) = fma(a[g][1].y, x, fma(a[g][2].x, y, fma(a[g][2].y, z, a[g][5].x)));
          sp.mz(s) = fma(a[g][3].x, x, fma(a[g][3].y, y, fma(a[g][4].x, z, a[g][5].y)));
        }
      }
      continue;
    }

    if constexpr (kFull) {
    if (kind == OP_RFTRAIN) {  // discretised shaped pulse: (pulse_j, identical interval) x count, on the fly
      const int cnt = __ldg(&op->count), m0i = __ldg(&op->aux), flags = __ldg(&op->flags), cls = __ldg(&op->cls);
      const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]), dmz = __ldg(&op->p[3]);
      const double* mats = kp.mats + static_cast<int64_t>(m0i) * 9;
      constexpr int G = S < 4 ? S : 4;  // spins per register group
#pragma unroll 1
      for (int g0 = 0; g0 < S; g0 += G) {
        double x[G], y[G], z[G], zr[G], zi[G], e1[G], rg[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int s = g0 + g;
          x[g] = sp.mx(s);
          y[g] = sp.my(s);
          z[g] = sp.mz(s);
          zr[g] = 1.0;
          zi[g] = 0.0;
          e1[g] = 1.0;
          rg[g] = 0.0;
          if (!sp.act(s) || !(flags & EV_MOVE)) continue;
          const int64_t i = sp.idx(s);
          const SC c = load_sc(kp, i);
          const double2 e = cls >= 0 ? relax_pair(kp, cls, i) : make_double2(1.0, 1.0);
          phase_factor(theta_of(c, dt, dmx, dmy, dmz), zr[g], zi[g]);
          zr[g] *= e.y;
          zi[g] *= e.y;
          e1[g] = e.x;
          rg[g] = c.m0 * (1.0 - e.x);
        }
        if (__ldg(&op->tmode) == 1) {  // x-axis sub-pulses: (x, y, z) -> (x, r4 y + r5 z, r7 y + r8 z)
          double a4 = __ldg(mats + 4), a5 = __ldg(mats + 5), a7 = __ldg(mats + 7), a8 = __ldg(mats + 8);
          for (int j = 0; j < cnt; ++j) {
            const double* mn = mats + 9 * (j + 1 < cnt ? j + 1 : j);
            const double b4 = __ldg(mn + 4), b5 = __ldg(mn + 5), b7 = __ldg(mn + 7), b8 = __ldg(mn + 8);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const double ny = a4 * y[g] + a5 * z[g];
              const double nz = a7 * y[g] + a8 * z[g];
              const double nx = x[g];
              x[g] = nx * zr[g] - ny * zi[g];
              y[g] = nx * zi[g] + ny * zr[g];
              z[g] = fma(nz, e1[g], rg[g]);
            }
            a4 = b4;
            a5 = b5;
            a7 = b7;
            a8 = b8;
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            sp.mx(g0 + g) = x[g];
            sp.my(g0 + g) = y[g];
            sp.mz(g0 + g) = z[g];
          }
          continue;
        }
        // the pulse matrices are CTA-uniform: prefetch pulse j+1 while applying pulse j
        double r[9], rn[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) r[k] = __ldg(mats + k);
        for (int j = 0; j < cnt; ++j) {
          const int jn = j + 1 < cnt ? j + 1 : j;
#pragma unroll
          for (int k = 0; k < 9; ++k) rn[k] = __ldg(mats + 9 * jn + k);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const double nx = r[0] * x[g] + r[1] * y[g] + r[2] * z[g];
            const double ny = r[3] * x[g] + r[4] * y[g] + r[5] * z[g];
            const double nz = r[6] * x[g] + r[7] * y[g] + r[8] * z[g];
            x[g] = nx * zr[g] - ny * zi[g];
            y[g] = nx * zi[g] + ny * zr[g];
            z[g] = fma(nz, e1[g], rg[g]);
          }
#pragma unroll
          for (int k = 0; k < 9; ++k) r[k] = rn[k];
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          sp.mx(g0 + g) = x[g];
          sp.my(g0 + g) = y[g];
          sp.mz(g0 + g) = z[g];
        }
      }
      continue;
    }

    if (kind == OP_GSAMP) {  // generic sampled intervals
      const int cnt = __ldg(&op->count), g0 = __ldg(&op->aux), s0 = __ldg(&op->s0) - kp.sample_base;
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        R ar[kChunkSlots], ai[kChunkSlots];
#pragma unroll
        for (int j = 0; j < kSampPerChunk; ++j) {
          if (j < ck) {
            const GEv* g = kp.gev + g0 + k0 + j;
            const int flags = __ldg(&g->flags), cls = __ldg(&g->cls);
            const double dt = __ldg(&g->dt), dmx = __ldg(&g->dmx), dmy = __ldg(&g->dmy), dmz = __ldg(&g->dmz);
#pragma unroll
            for (int s = 0; s < S; ++s) interval<S>(kp, sp, s, flags, cls, dt, dmx, dmy, dmz);
            record_state<R, S, NC>(kp, sp, ar, ai, j * NC);
          } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) ar[j * NC + c] = ai[j * NC + c] = R(0);
          }
        }
        strip.push(ar, ai, ck * NC, (s0 + k0) * NC);
      }
      continue;
    }

    if (kind == OP_CHIRP) {  // linear-increment sampled run: geometric rotation factors, fp64
      // Spin-outer over blocks of two chunks: each spin's chirp-class row (or its
      // SpinConst) is read once per block, not once per 8-sample chunk.
      const int cnt = __ldg(&op->count), s0 = __ldg(&op->s0) - kp.sample_base, cls = __ldg(&op->cls), crc = __ldg(&op->rot);
      const double dt = __ldg(&op->p[0]);
      const double d0x = __ldg(&op->p[1]), d0y = __ldg(&op->p[2]), d0z = __ldg(&op->p[3]);
      const double ddx = __ldg(&op->p[4]), ddy = __ldg(&op->p[5]), ddz = __ldg(&op->p[6]);
      constexpr int kBlk = 2 * kSampPerChunk;
      if constexpr (sizeof(R) == 4) {
        if (crc >= 0) {  // tabulated chirp, fp32 samples (see chirp_f32 below)
          chirp_f32<S, NC>(kp, op, sp, strip, smem_raw, cnt, s0);
          continue;
        }
      }
      for (int k0 = 0; k0 < cnt; k0 += kBlk) {
        const int cb = min(kBlk, cnt - k0);
        R ar[2][kChunkSlots], ai[2][kChunkSlots];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < kChunkSlots; ++j) ar[h][j] = ai[h][j] = R(0);
#pragma unroll 1
        for (int s = 0; s < S; ++s) {
          if (!sp.act(s)) continue;
          const int64_t i = sp.idx(s);
          double rr, ri, qc, qs, e1, rgw;
          if (crc >= 0) {  // tabulated chirp class (fp64 mode): planes r0, q (conj if tmode), (A, B) of the run
            const double2 r0 = __ldg(plane(kp, op, 0) + i);
            double2 q = __ldg(plane(kp, op, 1) + i);
            if (__ldg(&op->tmode) & 1) q.y = -q.y;
            rr = r0.x;
            ri = r0.y;
            if (k0 > 0) {  // advance to event k0 by q^kBlk per block (chirps are a block or two long)
              double2 qb = q;
#pragma unroll
              for (int m = 1; m < kBlk; m <<= 1) qb = make_double2(qb.x * qb.x - qb.y * qb.y, 2.0 * qb.x * qb.y);
              for (int a = 0; a < k0; a += kBlk) {
                const double r0r = rr;
                rr = r0r * qb.x - ri * qb.y;
                ri = r0r * qb.y + ri * qb.x;
              }
            } else {  // mz never enters a sample: the run's longitudinal map at once
              const double2 ab = __ldg(plane(kp, op, 3) + i);
              sp.mz(s) = fma(sp.mz(s), ab.x, ab.y);
            }
            qc = q.x;
            qs = q.y;
            e1 = 1.0;
            rgw = 0.0;
          } else {
            const SC c = load_sc(kp, i);
            const double2 e = cls >= 0 ? relax_pair(kp, cls, i) : make_double2(1.0, 1.0);
            const double b = fma(c.z, ddz, fma(c.y, ddy, c.x * ddx));
            phase_factor(fma(static_cast<double>(k0), b, theta_of(c, dt, d0x, d0y, d0z)), rr, ri);
            phase_factor(b, qc, qs);  // q = exp(-i b) = (qc, qs)
            rr *= e.y;
            ri *= e.y;
            e1 = e.x;
            rgw = c.m0 * (1.0 - e.x);
          }
          double x = sp.mx(s), y = sp.my(s), z = sp.mz(s);
          double2 w[NC];
#pragma unroll
          for (int cc = 0; cc < NC; ++cc)
            w[cc] = kp.w != nullptr ? __ldg(reinterpret_cast<const double2*>(kp.w) + static_cast<int64_t>(cc) * kp.n + i)
                                    : make_double2(1.0, 0.0);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int j = 0; j < kSampPerChunk; ++j) {
              if (h * kSampPerChunk + j < cb) {
                const double nx = x * rr - y * ri;
                y = x * ri + y * rr;
                x = nx;
                z = fma(z, e1, rgw);  // e1 = 1, rgw = 0 without relaxation
                const double a = rr;
                rr = a * qc - ri * qs;  // r <- r * q
                ri = a * qs + ri * qc;
#pragma unroll
                for (int cc = 0; cc < NC; ++cc) {
                  ar[h][j * NC + cc] += static_cast<R>(w[cc].x * x - w[cc].y * y);
                  ai[h][j * NC + cc] += static_cast<R>(w[cc].x * y + w[cc].y * x);
                }
              }
            }
          }
          sp.mx(s) = x;
          sp.my(s) = y;
          sp.mz(s) = z;
        }
        strip.push(ar[0], ai[0], min(kSampPerChunk, cb) * NC, (s0 + k0) * NC);
        if (cb > kSampPerChunk) strip.push(ar[1], ai[1], (cb - kSampPerChunk) * NC, (s0 + k0 + kSampPerChunk) * NC);
      }
      continue;
    }

    }

    // OP_WINDOW (compiled out of the kernels for programs whose windows are all deferred, OP_UWIN)
    if constexpr (kWin) {
      const int cnt = __ldg(&op->count), lead = __ldg(&op->aux), s0 = __ldg(&op->s0) - kp.sample_base, rc = __ldg(&op->rot),
                pre = __ldg(&op->pre);
      if constexpr (!kFull) {
        if (pre >= 0) apply_pre<S>(mats, sp, pre, __ldg(&op->tmode));
      }
      if constexpr (sizeof(R) == 4 && NC >= 2) {
        if (cnt >= kMmaMinWindow && kp.w32 != nullptr) {  // tensor-core multi-coil window
          char* stb = reinterpret_cast<char*>(smem_raw) + static_cast<size_t>(3 * S) * bd * sizeof(double) +
                      static_cast<size_t>(threadIdx.x >> 5) * McStage<NC>::kBytes;
          float4* st = reinterpret_cast<float4*>(stb);
          float2* wbuf = reinterpret_cast<float2*>(stb + kStageFloat4 * 16);  // 2 x [32][NC]
          float2* pf = reinterpret_cast<float2*>(stb + kStageFloat4 * 16 + 2 * McStage<NC>::kW);  // [lane][Cpre, z]
          const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
          float2* out = reinterpret_cast<float2*>(strip.row);
          const bool tb = rc >= 0;  // tabulated: planes Cpre, z (float2), C, (A, B)
          const int pcp = __ldg(&op->pl[0]), pz = __ldg(&op->pl[1]);
          const int ntile = (cnt + 63) >> 6;
          for (int j = 0; j < ntile; ++j) {
            const bool last = j + 1 == ntile;
            float acc[NC][4];
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
            auto fetch = [&](int r, int buf) {  // (Cpre, z) and the coil weights of this lane's spin r
              if (!sp.act(r)) return;
              const int64_t i = sp.idx(r);
              if (tb) {
                cp_async8(pf + 2 * lane, plane32_at(kp, pcp, i));
                cp_async8(pf + 2 * lane + 1, plane32_at(kp, pz, i));
              }
              const float2* wsrc = kp.w32 + i * NC;
#pragma unroll
              for (int c2 = 0; c2 < NC / 2; ++c2)
                cp_async16(wbuf + buf * 32 * NC + lane * NC + 2 * c2, wsrc + 2 * c2);
            };
            fetch(0, 0);
            cp_async_commit();
#pragma unroll 1
            for (int r = 0; r < S; ++r) {
              cp_async_wait_all();
              const float2 cpre = pf[2 * lane], zz = pf[2 * lane + 1];
              if (!sp.act(r)) {  // inactive spin: zero weights (the buffer may hold another spin's)
#pragma unroll
                for (int c = 0; c < NC; ++c) wbuf[(r & 1) * 32 * NC + lane * NC + c] = make_float2(0.f, 0.f);
              }
              if (r + 1 < S) fetch(r + 1, (r + 1) & 1);
              cp_async_commit();
              cf u{0.f, 0.f}, z{0.f, 0.f};
              if (sp.act(r)) {
                const int64_t i = sp.idx(r);
                double pr = cpre.x, pi = cpre.y, zr0 = zz.x, zi0 = zz.y, th = 0.0;
                SC c{};
                if (!tb) {
                  const int c1 = __ldg(&op->cls);
                  c = load_sc(kp, i);
                  th = theta_of(c, __ldg(&op->p[0]), __ldg(&op->p[1]), __ldg(&op->p[2]), __ldg(&op->p[3]));
                  const double2 e = c1 >= 0 ? relax_pair(kp, c1, i) : make_double2(1.0, 1.0);
                  phase_factor(th, zr0, zi0);
                  zr0 *= e.y;
                  zi0 *= e.y;
                  pr = 1.0;
                  pi = 0.0;
                }
                const double x = sp.mx(r), y = sp.my(r);
                u = cf{static_cast<float>(pr * x - pi * y), static_cast<float>(pr * y + pi * x)};
                z = cf{static_cast<float>(zr0), static_cast<float>(zi0)};
                if (!lead) u = cmul(u, z);
                const cf z64 = csq(csq(csq(csq(csq(csq(z))))));
                for (int q = 0; q < j; ++q) u = cmul(u, z64);  // this tile starts at sample 64 j
                if (!tb && last) {
                  const int cw = __ldg(&op->flags);
                  const double2 E = cw >= 0 ? relax_pair(kp, cw, i) : make_double2(1.0, 1.0);
                  double cr, ci;
                  phase_factor(th * static_cast<double>(cnt - lead), cr, ci);
                  sp.mx(r) = E.y * (cr * x - ci * y);
                  sp.my(r) = E.y * (cr * y + ci * x);
                  sp.mz(r) = fma(sp.mz(r), E.x, c.m0 * (1.0 - E.x));
                }
              }
              if constexpr (NC == 8) {
                stage_spin_mc8(st, lane, u, z);
                __syncwarp();
                mma_round_mc8(st, wbuf + (r & 1) * 32 * NC, lane, acc);
              } else {
                stage_spin_mc(st, lane, u, z);
                __syncwarp();
                mma_round_mc<NC>(st, wbuf + (r & 1) * 32 * NC, lane, acc);
              }
              __syncwarp();
            }
            if constexpr (NC == 8) {  // acc[m]: coil g of samples 64 j + 8 m + 2 t (+1)
#pragma unroll
              for (int m = 0; m < 8; ++m) {
                const int k1 = 64 * j + 8 * m + 2 * t, k2 = k1 + 1;
                if (k1 < cnt) __stcs(out + static_cast<int64_t>(s0 + k1) * NC + g, make_float2(acc[m][0], acc[m][2]));
                if (k2 < cnt) __stcs(out + static_cast<int64_t>(s0 + k2) * NC + g, make_float2(acc[m][1], acc[m][3]));
              }
            } else {
              const int k1 = 64 * j + 16 * t + g, k2 = k1 + 8;
#pragma unroll
              for (int c = 0; c < NC; ++c) {
                if (k1 < cnt) __stcs(out + static_cast<int64_t>(s0 + k1) * NC + c, make_float2(acc[c][0], acc[c][2]));
                if (k2 < cnt) __stcs(out + static_cast<int64_t>(s0 + k2) * NC + c, make_float2(acc[c][1], acc[c][3]));
              }
            }
          }
          if (tb) {
            const double2 *pc = plane(kp, op, 2), *pab = plane(kp, op, 3);
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int64_t i = sp.act(r) ? sp.idx(r) : 0;
              const double2 c = __ldg(pc + i), ab = __ldg(pab + i);
              const double x = sp.mx(r), y = sp.my(r);
              sp.mx(r) = c.x * x - c.y * y;
              sp.my(r) = c.x * y + c.y * x;
              sp.mz(r) = fma(sp.mz(r), ab.x, ab.y);
            }
          }
          continue;
        }
      }
      if constexpr (kMma1) {
        if (cnt >= kMmaMinWindow) {  // tensor-core window (see the notes above stage_spin)
          char* stb = reinterpret_cast<char*>(smem_raw) + static_cast<size_t>(3 * S) * bd * sizeof(double) +
                      static_cast<size_t>(threadIdx.x >> 5) * kStageBytes;
          float4* st = reinterpret_cast<float4*>(stb);
          float2* z64s = reinterpret_cast<float2*>(stb + kStageFloat4 * 16);
          float2* pf = reinterpret_cast<float2*>(stb + kStageFloat4 * 16 + 32 * 8);  // [lane][Cpre, z]
          const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
          float2* out = reinterpret_cast<float2*>(strip.row) + s0;
          const bool tb = rc >= 0;  // tabulated: planes Cpre, z, C, (A, B)
          const int pcp = __ldg(&op->pl[0]), pz = __ldg(&op->pl[1]);  // plane ids (32-bit: fewer live registers)
          constexpr int kMaxTiles = kFull ? 4 : 8;  // 64-sample tiles per pass (4 accumulators each)
          for (int p0 = 0; p0 < cnt; p0 += 64 * kMaxTiles) {  // passes of up to kMaxTiles tiles of 64 samples
            const int ntile = min(kMaxTiles, (cnt - p0 + 63) >> 6);
            const bool last = p0 + 64 * kMaxTiles >= cnt;
            float acc[kMaxTiles][4];
#pragma unroll
            for (int j = 0; j < kMaxTiles; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
            if (tb && sp.act(0)) {  // (Cpre, z) of round 0 into this lane's prefetch slot
              cp_async8(pf + 2 * lane, plane32_at(kp, pcp, sp.idx(0)));
              cp_async8(pf + 2 * lane + 1, plane32_at(kp, pz, sp.idx(0)));
            }
            cp_async_commit();
#pragma unroll 1
            for (int r = 0; r < S; ++r) {
              cf u{0.f, 0.f}, z{0.f, 0.f};
              cp_async_wait_all();
              const float2 cpre = pf[2 * lane], zz = pf[2 * lane + 1];
              if (tb && r + 1 < S && sp.act(r + 1)) {  // next round's (Cpre, z) lands during this round's mma
                cp_async8(pf + 2 * lane, plane32_at(kp, pcp, sp.idx(r + 1)));
                cp_async8(pf + 2 * lane + 1, plane32_at(kp, pz, sp.idx(r + 1)));
              }
              cp_async_commit();
              if (sp.act(r)) {
                const int64_t i = sp.idx(r);
                double pr = cpre.x, pi = cpre.y, zr0 = zz.x, zi0 = zz.y;
                double th = 0.0;
                SC c{};
                if (!tb) {  // on the fly: a window whose interval is not reused
                  const int c1 = __ldg(&op->cls);
                  c = load_sc(kp, i);
                  th = theta_of(c, __ldg(&op->p[0]), __ldg(&op->p[1]), __ldg(&op->p[2]), __ldg(&op->p[3]));
                  const double2 e = c1 >= 0 ? relax_pair(kp, c1, i) : make_double2(1.0, 1.0);
                  phase_factor(th, zr0, zi0);
                  zr0 *= e.y;
                  zi0 *= e.y;
                  // no pre-interval on the fly: the entry factor is the receive weight alone
                  // (tabulated windows carry w in their Cpre plane)
                  const double2 w0 = kp.w != nullptr ? __ldg(reinterpret_cast<const double2*>(kp.w) + i)
                                                     : make_double2(1.0, 0.0);
                  pr = w0.x;
                  pi = w0.y;
                }
                const double x = sp.mx(r), y = sp.my(r);
                u = cf{static_cast<float>(pr * x - pi * y), static_cast<float>(pr * y + pi * x)};
                z = cf{static_cast<float>(zr0), static_cast<float>(zi0)};
                if (!lead) u = cmul(u, z);  // first sample after one interval
                if (p0 > 0) {               // later pass: u z^p0
                  cf zp = z;
#pragma unroll
                  for (int q = 1; q < 64 * kMaxTiles; q <<= 1) zp = csq(zp);  // z^(64 kMaxTiles)
                  for (int q = 0; q < p0; q += 64 * kMaxTiles) u = cmul(u, zp);
                }
                if (!tb && last) {  // exit propagator of the whole run, on the fly
                  const int cw = __ldg(&op->flags);
                  const double2 E = cw >= 0 ? relax_pair(kp, cw, i) : make_double2(1.0, 1.0);
                  double cr, ci;
                  phase_factor(th * static_cast<double>(cnt - lead), cr, ci);
                  sp.mx(r) = E.y * (cr * x - ci * y);
                  sp.my(r) = E.y * (cr * y + ci * x);
                  sp.mz(r) = fma(sp.mz(r), E.x, c.m0 * (1.0 - E.x));
                }
              }
              stage_spin(st, z64s, lane, u, z);
              __syncwarp();
              mma_round<kMaxTiles>(st, z64s, lane, ntile, acc);
              __syncwarp();  // the stage is rewritten by the next round
            }
#pragma unroll
            for (int j = 0; j < kMaxTiles; ++j) {
              if (j < ntile) {
                const int k1 = p0 + 64 * j + 16 * t + g, k2 = k1 + 8;
                if (k1 < cnt) __stcs(out + k1, make_float2(acc[j][0], acc[j][2]));
                if (k2 < cnt) __stcs(out + k2, make_float2(acc[j][1], acc[j][3]));
              }
            }
          }
          if (tb) {  // exit: C m, mz -> A mz + B for all spins, loads issued together
            const double2 *pc = plane(kp, op, 2), *pab = plane(kp, op, 3);
            double2 c[S], ab[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int64_t i = sp.act(r) ? sp.idx(r) : 0;
              c[r] = __ldg(pc + i);
              ab[r] = __ldg(pab + i);
            }
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const double x = sp.mx(r), y = sp.my(r);
              sp.mx(r) = c[r].x * x - c[r].y * y;
              sp.my(r) = c[r].x * y + c[r].y * x;
              sp.mz(r) = fma(sp.mz(r), ab[r].x, ab[r].y);
            }
          }
          continue;
        }
      }
      // per-spin setup: sample factor z and the exit propagator of the whole run
      R zr[S], zi[S], ur[S], ui[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        zr[s] = R(1);
        zi[s] = R(0);
        ur[s] = R(0);
        ui[s] = R(0);
        if (!sp.act(s)) continue;
        const int64_t i = sp.idx(s);
        RotCoef k;
        if (rc >= 0) {  // tabulated (pre, window, post) propagators
          k = load_rot<R>(kp, op, i);
        } else {  // on the fly: a window whose interval is not reused
          const int c1 = __ldg(&op->cls), cw = __ldg(&op->flags);
          const double dt = __ldg(&op->p[0]);
          const SC c = load_sc(kp, i);
          const double th = theta_of(c, dt, __ldg(&op->p[1]), __ldg(&op->p[2]), __ldg(&op->p[3]));
          const double2 e = c1 >= 0 ? relax_pair(kp, c1, i) : make_double2(1.0, 1.0);
          const double2 E = cw >= 0 ? relax_pair(kp, cw, i) : make_double2(1.0, 1.0);
          phase_factor(th, k.zr, k.zi);
          phase_factor(th * static_cast<double>(cnt - lead), k.cr, k.ci);
          k.zr *= e.y;
          k.zi *= e.y;
          k.cr *= E.y;
          k.ci *= E.y;
          k.a = E.x;
          k.b = c.m0 * (1.0 - E.x);
          k.pr = 1.0;
          k.pi = 0.0;
        }
        zr[s] = static_cast<R>(k.zr);
        zi[s] = static_cast<R>(k.zi);
        double2 w0 = make_double2(1.0, 0.0);  // tabulated windows carry w in Cpre
        if (kp.w != nullptr && NC == 1 && rc < 0) w0 = __ldg(reinterpret_cast<const double2*>(kp.w) + i);
        const double x = sp.mx(s), y = sp.my(s);
        // state at the first sample: the absorbed pre-interval applied
        const double x0 = k.pr * x - k.pi * y, y0 = k.pr * y + k.pi * x;
        // NC == 1: track u = w*m (the weight rides along the recurrence); else m
        ur[s] = static_cast<R>(w0.x * x0 - w0.y * y0);
        ui[s] = static_cast<R>(w0.x * y0 + w0.y * x0);
        sp.mx(s) = k.cr * x - k.ci * y;
        sp.my(s) = k.cr * y + k.ci * x;
        sp.mz(s) = fma(sp.mz(s), k.a, k.b);
      }
      if constexpr (kPacked) {
        constexpr int P = S / 2;
        float2 U[P], V[P], ZR[P], ZI[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          ZR[p] = make_float2(zr[2 * p], zr[2 * p + 1]);
          ZI[p] = make_float2(zi[2 * p], zi[2 * p + 1]);
          U[p] = make_float2(ur[2 * p], ur[2 * p + 1]);
          V[p] = make_float2(ui[2 * p], ui[2 * p + 1]);
        }
        int k0 = 0;
        if (lead && cnt >= kChunkSlots) {
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk_f2<P, true, true>(U, V, ZR, ZI, ar, ai, kChunkSlots);
          strip.push(ar, ai, kChunkSlots, s0);
          k0 = kChunkSlots;
        }
        // two chunks per trip in one basic block: the warp transpose-reduction of
        // the first (shuffle latency) overlaps the complex multiplies of the second
        for (; k0 + 2 * kChunkSlots <= cnt; k0 += 2 * kChunkSlots) {
          R ar[kChunkSlots], ai[kChunkSlots], br[kChunkSlots], bi[kChunkSlots];
          window_chunk_f2<P, true, false>(U, V, ZR, ZI, ar, ai, kChunkSlots);
          window_chunk_f2<P, true, false>(U, V, ZR, ZI, br, bi, kChunkSlots);
          strip.push(ar, ai, kChunkSlots, s0 + k0);
          strip.push(br, bi, kChunkSlots, s0 + k0 + kChunkSlots);
        }
        for (; k0 + kChunkSlots <= cnt; k0 += kChunkSlots) {
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk_f2<P, true, false>(U, V, ZR, ZI, ar, ai, kChunkSlots);
          strip.push(ar, ai, kChunkSlots, s0 + k0);
        }
        if (k0 < cnt) {
          const int ck = cnt - k0;
          R ar[kChunkSlots], ai[kChunkSlots];
          if (lead && k0 == 0)
            window_chunk_f2<P, false, true>(U, V, ZR, ZI, ar, ai, ck);
          else
            window_chunk_f2<P, false, false>(U, V, ZR, ZI, ar, ai, ck);
          strip.push(ar, ai, ck, s0 + k0);
        }
      } else if constexpr (sizeof(R) == 4 && NC >= 2) {
        constexpr int PC = NC / 2;
        float2 WR[PC][S], WI[PC][S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int p = 0; p < PC; ++p) {
            WR[p][s] = WI[p][s] = make_float2(0.f, 0.f);
            if (sp.act(s)) {
              const double2* wp = reinterpret_cast<const double2*>(kp.w) + sp.idx(s);
              const double2 a = __ldg(wp + static_cast<int64_t>(2 * p) * kp.n);
              const double2 b = __ldg(wp + static_cast<int64_t>(2 * p + 1) * kp.n);
              WR[p][s] = make_float2(static_cast<float>(a.x), static_cast<float>(b.x));
              WI[p][s] = make_float2(static_cast<float>(a.y), static_cast<float>(b.y));
            }
          }
        }
        int k0 = 0;
        if (lead && cnt >= kSampPerChunk) {
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk_mc2<S, NC, true, true>(ur, ui, zr, zi, WR, WI, ar, ai, kSampPerChunk);
          strip.push(ar, ai, kChunkSlots, s0 * NC);
          k0 = kSampPerChunk;
        }
        for (; k0 + kSampPerChunk <= cnt; k0 += kSampPerChunk) {
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk_mc2<S, NC, true, false>(ur, ui, zr, zi, WR, WI, ar, ai, kSampPerChunk);
          strip.push(ar, ai, kChunkSlots, (s0 + k0) * NC);
        }
        if (k0 < cnt) {
          const int ck = cnt - k0;
          R ar[kChunkSlots], ai[kChunkSlots];
          if (lead && k0 == 0)
            window_chunk_mc2<S, NC, false, true>(ur, ui, zr, zi, WR, WI, ar, ai, ck);
          else
            window_chunk_mc2<S, NC, false, false>(ur, ui, zr, zi, WR, WI, ar, ai, ck);
          strip.push(ar, ai, ck * NC, (s0 + k0) * NC);
        }
      } else {
        R wr[NC][S], wi[NC][S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            wr[c][s] = wi[c][s] = R(0);
            if (NC > 1 && sp.act(s)) {
              const double2 w =
                  __ldg(reinterpret_cast<const double2*>(kp.w) + static_cast<int64_t>(c) * kp.n + sp.idx(s));
              wr[c][s] = static_cast<R>(w.x);
              wi[c][s] = static_cast<R>(w.y);
            }
          }
        }
        int k0 = 0;
        if (lead && cnt >= kSampPerChunk) {
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk<R, S, NC, true, true>(ur, ui, zr, zi, wr, wi, ar, ai, kSampPerChunk);
          strip.push(ar, ai, kChunkSlots, s0 * NC);
          k0 = kSampPerChunk;
        }
        for (; k0 + kSampPerChunk <= cnt; k0 += kSampPerChunk) {
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk<R, S, NC, true, false>(ur, ui, zr, zi, wr, wi, ar, ai, kSampPerChunk);
          strip.push(ar, ai, kChunkSlots, (s0 + k0) * NC);
        }
        if (k0 < cnt) {
          const int ck = cnt - k0;
          R ar[kChunkSlots], ai[kChunkSlots];
          if (lead && k0 == 0)
            window_chunk<R, S, NC, false, true>(ur, ui, zr, zi, wr, wi, ar, ai, ck);
          else
            window_chunk<R, S, NC, false, false>(ur, ui, zr, zi, wr, wi, ar, ai, ck);
          strip.push(ar, ai, ck * NC, (s0 + k0) * NC);
        }
      }
    }
  }
  if constexpr (kRegState) {  // a segmented program: the running factors travel to the next segment's launch
    if (progs != nullptr && kp.mx1 != nullptr) {
      for (int pc = 0; pc < kp.n_prog_smem; ++pc) {
        double2* dst = kp.planes + static_cast<int64_t>(kp.prog_plane[pc]) * kp.n;
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (sp.act(s)) dst[sp.idx(s)] = progs[(pc * S + s) * bd + threadIdx.x];
      }
    }
  }
  if (kp.mx1 != nullptr) {  // a segmented program: the state travels to the next segment's launch
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (!sp.act(s)) continue;
      const int64_t i = sp.idx(s);
      kp.mx1[i] = sp.mx(s);
      kp.my1[i] = sp.my(s);
      kp.mz1[i] = sp.mz(s);
    }
  }
}

// ---------------------------------------------------------------------------
// staging, class tables, fold
// ---------------------------------------------------------------------------

__device__ __forceinline__ int64_t gtid() { return blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return static_cast<int64_t>(gridDim.x) * blockDim.x; }

// SpinConst records from the caller's SoA inputs (engine.py:192-226 fields)
__global__ void prep_kernel(int64_t n, const double* __restrict__ pos, const double* __restrict__ dw,
                            const double* __restrict__ m0, const double* __restrict__ t1,
                            const double* __restrict__ t2, SpinConst* __restrict__ sc) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    SpinConst c;
    c.x = pos[3 * i + 0];
    c.y = pos[3 * i + 1];
    c.z = pos[3 * i + 2];
    c.dw = dw[i];
    c.m0 = m0[i];
    c.r1 = 1.0 / t1[i];  // engine.py:270 (inf -> 0: no relaxation)
    c.r2 = 1.0 / t2[i];
    c.pad = 0.0;
    sc[i] = c;
  }
}

// relax_cache restated (engine.py:292-299): (e1, e2) = (exp(-T*inv_t1), exp(-T*inv_t2))
__global__ void relax_table_kernel(int64_t n, int n_cls, const double* __restrict__ T,
                                   const SpinConst* __restrict__ sc, double2* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n_cls) * n;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int64_t c = t / n, i = t - c * n;
    out[t] = make_double2(exp(-T[c] * sc[i].r1), exp(-T[c] * sc[i].r2));
  }
}

// planes (program.h PlaneDesc), fp64, one thread per (plane, spin):
//   PL_PHASE: exp(-T/T2) exp(-i (pos . d + dw tw))  (x w1[i] if PL_WEIGHT and single-coil weights are given)
//   PL_AB:    (exp(-T/T1), m0 (1 - exp(-T/T1)))
// e.g. a rotation class (pre, m x main, post) gives Cpre = PHASE(pre), z = PHASE(main),
// C = PHASE(pre + m main + post) and AB(T) with T its whole duration (relax_cache
// restated, engine.py:292-299, for every interval length the program reuses).
__global__ void plane_kernel(int64_t n, int n_planes, const PlaneDesc* __restrict__ pd,
                             const SpinConst* __restrict__ sc, const double2* __restrict__ w1,
                             double2* __restrict__ out, float2* __restrict__ out32) {
  const int64_t total = static_cast<int64_t>(n_planes) * n;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int64_t c = t / n, i = t - c * n;
    const PlaneDesc& k = pd[c];
    const SpinConst s = sc[i];
    if (k.kind == PL_AB) {
      const double e1 = exp(-k.T * s.r1);
      out[t] = make_double2(e1, s.m0 * (1.0 - e1));
      continue;
    }
    double pc, ps;
    phase_factor(fma(s.z, k.d[2], fma(s.y, k.d[1], s.x * k.d[0])) + s.dw * k.tw, pc, ps);
    const double e2 = k.T != 0.0 ? exp(-k.T * s.r2) : 1.0;
    pc *= e2;
    ps *= e2;
    if ((k.flags & PL_WEIGHT) && w1 != nullptr) {
      const double2 w = w1[i];
      const double r = w.x * pc - w.y * ps;
      ps = w.x * ps + w.y * pc;
      pc = r;
    }
    if ((k.flags & PL_SAMPLE) && out32 != nullptr)
      out32[t] = make_float2(static_cast<float>(pc), static_cast<float>(ps));
    else
      out[t] = make_double2(pc, ps);
  }
}

// train classes (program.h TrainClass): per (class, spin) the affine propagator of the
// whole run, m -> A m + b, composed in fp64 in the order the on-the-fly path applies
// it (engine.py:277-302 per elementary sequence): pulse j, then the shared interval
// (precession by th, transverse decay e2, longitudinal e1 and regrowth m0 (1 - e1)).
// The three columns of A and the vector b are pushed through the pairs together.
// Output row: A (row-major, 9), b (3).
__global__ void train_table_kernel(int64_t n, int n_cls, const TrainClass* __restrict__ tc,
                                   const double* __restrict__ mats, const SpinConst* __restrict__ sc,
                                   double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n_cls) * n;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int64_t c = t / n, i = t - c * n;
    const TrainClass& k = tc[c];
    const SpinConst s = sc[i];
    double zr = 1.0, zi = 0.0, e1 = 1.0, rg = 0.0;
    if (k.flags & EV_MOVE) {
      const double th = fma(s.z, k.p[3], fma(s.y, k.p[2], s.x * k.p[1])) + s.dw * k.p[0];
      phase_factor(th, zr, zi);
      if (k.flags & EV_RELAX) {
        const double e2 = exp(-k.p[0] * s.r2);
        e1 = exp(-k.p[0] * s.r1);
        zr *= e2;
        zi *= e2;
        rg = s.m0 * (1.0 - e1);
      }
    }
    // v[col][row]: columns 0..2 of A, column 3 = b
    double v[4][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}, {0.0, 0.0, 0.0}};
    const double* m = mats + 9 * static_cast<int64_t>(k.aux);
    for (int j = 0; j < k.count; ++j, m += 9) {
      double r[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) r[q] = __ldg(m + q);
#pragma unroll
      for (int col = 0; col < 4; ++col) {
        const double x = v[col][0], y = v[col][1], z = v[col][2];
        const double nx = r[0] * x + r[1] * y + r[2] * z;
        const double ny = r[3] * x + r[4] * y + r[5] * z;
        const double nz = r[6] * x + r[7] * y + r[8] * z;
        v[col][0] = nx * zr - ny * zi;
        v[col][1] = nx * zi + ny * zr;
        v[col][2] = col == 3 ? fma(nz, e1, rg) : nz * e1;
      }
    }
    double* o = out + t * kTrainRow;
#pragma unroll
    for (int row = 0; row < 3; ++row)
#pragma unroll
      for (int col = 0; col < 3; ++col) o[row * 3 + col] = v[col][row];
#pragma unroll
    for (int row = 0; row < 3; ++row) o[9 + row] = v[3][row];
  }
}

// pad [nc][n][2] weights to [ncp][n][2] (zero coils beyond nc)
__global__ void pad_weights_kernel(int64_t n, int nc, int ncp, const double* __restrict__ w, double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int64_t c = t / (n * 2);
    out[t] = c < nc ? w[t] : 0.0;
  }
}

// fp32 copy of the (padded) coil weights, spin-major: out[i][c] = w[c][i]
__global__ void weights_f32_kernel(int64_t n, int ncp, const double2* __restrict__ w, float2* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(ncp) * n;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int64_t i = t / ncp, c = t % ncp;
    const double2 v = w[c * n + i];
    out[t] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
}

// fixed-order fp64 fold of `rows` partial rows spaced row_stride elements apart (every warp row, or
// one folded row per CTA) into the echo layout out[c][sample_g[s]][re, im]
template <typename R>
__global__ void reduce_partials_kernel(const R* __restrict__ part, int rows, int64_t row_stride, int64_t n_slots,
                                       int nc, int ncp, const int64_t* __restrict__ sample_g, int64_t G,
                                       double* __restrict__ out) {
  const int64_t total = n_slots * 2;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int64_t sl = t >> 1;
    const int comp = static_cast<int>(t & 1);
    const int64_t s = sl / ncp;
    const int c = static_cast<int>(sl % ncp);
    if (c >= nc) continue;
    double acc = 0.0;
    for (int b = 0; b < rows; ++b) acc += static_cast<double>(part[static_cast<int64_t>(b) * row_stride + t]);
    out[(static_cast<int64_t>(c) * G + sample_g[s]) * 2 + comp] = acc;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

template <typename R, int S, int NC>
size_t integrate_smem_bytes(int threads, bool win) {
  // fp64 spin state [3][S][threads] + (fp32, programs with windows or chirps) the tensor-core window stage
  size_t stage = 0;
  if constexpr (sizeof(R) == 4 && NC == 1) stage = kStageBytes;
  if constexpr (sizeof(R) == 4 && NC >= 2) stage = McStage<NC>::kBytes;
  if (!win && S <= 4) return 0;  // the variant without window / chirp / train code: state in registers
  if (!win) stage = 0;
  return static_cast<size_t>(3 * S * threads) * sizeof(double) + static_cast<size_t>(threads / 32) * stage;
}

// the opt-in shared-memory limit is a per-device function attribute: track what was allowed per
// (kernel instance, device), under a lock (contexts on several devices or threads share the instances)
static std::mutex g_smem_mu;

template <typename R, int S, int NC, bool kFull, int BD, bool kWin>
static cudaError_t launch_bd(const KParams& kp, int grid, int threads, cudaStream_t stream) {
  size_t smem = integrate_smem_bytes<R, S, NC>(threads, kWin || kFull);
  if (!kWin && !kFull && S <= 4)  // staged pulse matrices and progression running factors (host-sized)
    smem += ((static_cast<size_t>(kp.n_mats_smem) * 72 + 15) & ~size_t(15)) +
            static_cast<size_t>(kp.n_prog_smem) * S * threads * sizeof(double2);
  static size_t smem_set[kMaxDevices] = {};  // raise the limit only when needed (not inside a graph capture)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  {
    std::lock_guard<std::mutex> lk(g_smem_mu);
    if (smem > 48 * 1024 && smem > smem_set[dev]) {
      e = cudaFuncSetAttribute(integrate_kernel<R, S, NC, kFull, BD, kWin>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      smem_set[dev] = smem;
    }
  }
  integrate_kernel<R, S, NC, kFull, BD, kWin><<<grid, threads, smem, stream>>>(kp);
  return cudaGetLastError();
}

// the basic fp32 single-coil kernel with 8 spins per thread at its full block size (config 1's
// launch) gets a constant-block-size instance: config 1 -1.0%; the kFull variant measured +2.8%
// on config 3 with it, so it keeps the runtime block size
template <typename R, int S, int NC, bool kFull, bool kWin>
static cudaError_t launch_one(const KParams& kp, int grid, int threads, cudaStream_t stream) {
#ifndef BLOCH_NO_FIXED_BD
  constexpr int kMax = kWin ? KernelTraits<R, S, NC>::kMaxThreads : KernelTraits<R, S, NC>::kMaxThreadsNoWin;
  if constexpr (sizeof(R) == 4 && NC == 1 && S == 8 && !kFull) {
    if (threads == kMax) return launch_bd<R, S, NC, kFull, kMax, kWin>(kp, grid, threads, stream);
  }
#endif
  return launch_bd<R, S, NC, kFull, 0, kWin>(kp, grid, threads, stream);
}

template <typename R, int S, int NC>
cudaError_t launch_integrate(const KParams& kp, int grid, int threads, cudaStream_t stream, bool full, bool win) {
  if constexpr (sizeof(R) == 4) {  // fp32 mode: programs of pulses, intervals and deferred windows only
    if (!full && !win) return launch_one<R, S, NC, false, false>(kp, grid, threads, stream);
  }
  return full ? launch_one<R, S, NC, true, true>(kp, grid, threads, stream)
              : launch_one<R, S, NC, false, true>(kp, grid, threads, stream);
}

static int grid_for(int64_t total, int threads) {
  const int64_t blocks = (total + threads - 1) / threads;
  return static_cast<int>(blocks < 8192 ? (blocks > 0 ? blocks : 1) : 8192);
}

cudaError_t launch_prep(int64_t n, const double* pos, const double* dw, const double* m0, const double* t1,
                        const double* t2, SpinConst* sc, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  prep_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, pos, dw, m0, t1, t2, sc);
  return cudaGetLastError();
}

cudaError_t launch_relax_table(int64_t n, int n_cls, const double* T, const SpinConst* sc, double* out,
                               cudaStream_t stream) {
  if (n == 0 || n_cls == 0) return cudaSuccess;
  relax_table_kernel<<<grid_for(static_cast<int64_t>(n_cls) * n, 256), 256, 0, stream>>>(
      n, n_cls, T, sc, reinterpret_cast<double2*>(out));
  return cudaGetLastError();
}

cudaError_t launch_planes(int64_t n, int n_planes, const PlaneDesc* pd, const SpinConst* sc, const double* w1,
                          double* out, float2* out32, cudaStream_t stream) {
  if (n == 0 || n_planes == 0) return cudaSuccess;
  plane_kernel<<<grid_for(static_cast<int64_t>(n_planes) * n, 256), 256, 0, stream>>>(
      n, n_planes, pd, sc, reinterpret_cast<const double2*>(w1), reinterpret_cast<double2*>(out), out32);
  return cudaGetLastError();
}

cudaError_t launch_train_table(int64_t n, int n_cls, const TrainClass* tc, const double* mats, const SpinConst* sc,
                               double* out, cudaStream_t stream) {
  if (n == 0 || n_cls == 0) return cudaSuccess;
  train_table_kernel<<<grid_for(static_cast<int64_t>(n_cls) * n, 128), 128, 0, stream>>>(n, n_cls, tc, mats, sc, out);
  return cudaGetLastError();
}

cudaError_t launch_pad_weights(int64_t n, int nc, int ncp, const double* w, double* out, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  if (total == 0) return cudaSuccess;
  pad_weights_kernel<<<grid_for(total, 256), 256, 0, stream>>>(n, nc, ncp, w, out);
  return cudaGetLastError();
}

cudaError_t launch_weights_f32(int64_t n, int ncp, const double* w, float2* out, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(ncp) * n;
  if (total == 0) return cudaSuccess;
  weights_f32_kernel<<<grid_for(total, 256), 256, 0, stream>>>(n, ncp, reinterpret_cast<const double2*>(w), out);
  return cudaGetLastError();
}

__global__ void sum_rows_kernel(const double* __restrict__ rows, int n_rows, int64_t len, double* __restrict__ out) {
  for (int64_t t = gtid(); t < len; t += gstride()) {
    double acc = rows[t];
    for (int r = 1; r < n_rows; ++r) acc += rows[static_cast<int64_t>(r) * len + t];
    out[t] = acc;
  }
}

cudaError_t launch_sum_rows(const double* rows, int n_rows, int64_t len, double* out, cudaStream_t stream) {
  if (len == 0) return cudaSuccess;
  sum_rows_kernel<<<grid_for(len, 256), 256, 0, stream>>>(rows, n_rows, len, out);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_reduce(const R* part, int rows, int64_t row_stride, int64_t n_slots, int nc, int ncp,
                          const int64_t* sample_g, int64_t G, double* out, cudaStream_t stream) {
  const int64_t total = n_slots * 2;
  if (total == 0) return cudaSuccess;
  const int64_t blocks = (total + 255) / 256;
  reduce_partials_kernel<R><<<static_cast<int>(blocks < 65535 ? blocks : 65535), 256, 0, stream>>>(
      part, rows, row_stride, n_slots, nc, ncp, sample_g, G, out);
  return cudaGetLastError();
}

template <typename R, int S, int NC>
cudaError_t kernel_attrs(int* max_threads, int* regs) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, integrate_kernel<R, S, NC, true, 0, true>);
  if (e != cudaSuccess) return e;
  *max_threads = a.maxThreadsPerBlock;
  *regs = a.numRegs;
  return cudaSuccess;
}

#define BLOCH_INST(R, S, NC)                                                              \
  template cudaError_t launch_integrate<R, S, NC>(const KParams&, int, int, cudaStream_t, bool, bool); \
  template cudaError_t kernel_attrs<R, S, NC>(int*, int*);                                 \
  template size_t integrate_smem_bytes<R, S, NC>(int, bool);
BLOCH_FOR_EACH_VARIANT(BLOCH_INST)
#undef BLOCH_INST

template cudaError_t launch_reduce<float>(const float*, int, int64_t, int64_t, int, int, const int64_t*, int64_t,
                                          double*, cudaStream_t);
template cudaError_t launch_reduce<double>(const double*, int, int64_t, int64_t, int, int, const int64_t*, int64_t,
                                           double*, cudaStream_t);

}  // namespace bloch
