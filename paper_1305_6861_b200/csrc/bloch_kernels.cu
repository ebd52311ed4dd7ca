// sm_100a kernels of the Bloch event-stream engine.
//
// integrate_kernel<R, S, NC>  — the hot path: restates engine.compute_block
//   (engine.py:259-310) for S spins per thread.  The op stream (program.h) is
//   identical for every thread, so all control flow is CTA-uniform and op
//   fields are broadcast loads.  ADC samples are reduced without atomics:
//   per-thread sum over its S spins -> warp transpose-reduction of 8 slots
//   (sample x coil) -> per-warp strip in shared memory -> CTA sum written to
//   this CTA's row of the partial buffer; reduce_partials() then folds the rows
//   in a fixed order in fp64 (deterministic, like the reference's ordered fold,
//   engine.py:594-595).
//
// Precision: the per-spin state (mx, my, mz) is fp64 in every mode and lives in
// shared memory between ops (it only changes at pulses, generic intervals, RF
// trains, chirps and window exits).  R is the type of the ADC sample
// recurrence inside uniform windows, the dominant work: fp32
// (BLOCH_PREC_F32, packed FFMA2/FMUL2/FADD2 over spin pairs) or fp64.
//
// Uniform ADC windows (OP_WINDOW): per spin the window rotation
// z = e2 * exp(-i*theta) is formed once (fp64 phase, reduced mod 2pi) and the
// receive-weighted transverse magnetisation u = w * (mx + i*my) is advanced by
// one complex multiply per sample (engine.py:289-305 for every sample of the
// window: same theta, same e2 from the relax cache).  The state that leaves the
// window comes from the closed form m * E2^n * exp(-i*n*theta),
// mz -> m0 + (mz - m0) * E1^n in fp64, so per-sample rounding never feeds back
// into the spin state.  Relaxation factors come from the per-(class, spin)
// table built by relax_table_kernel (the reference's relax_cache).
#include <cuda_runtime.h>
#include <stdint.h>

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

template <typename R>
__device__ __forceinline__ void phase_sincos(double th, R& s, R& c);
template <>
__device__ __forceinline__ void phase_sincos<float>(double th, float& s, float& c) {
  sincosf(static_cast<float>(reduce_2pi(th)), &s, &c);
}
template <>
__device__ __forceinline__ void phase_sincos<double>(double th, double& s, double& c) {
  sincos(reduce_2pi(th), &s, &c);
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

// ---------------------------------------------------------------------------
// per-CTA ADC strip (shared memory) and its flush to the partial buffer
// ---------------------------------------------------------------------------

// Each warp owns one row of the partial buffer: after the transpose-reduction
// the 8 lanes holding a slot total write it straight to global memory (64 B per
// chunk, coalesced).  No shared-memory staging, no CTA barrier: warps never wait
// for each other.  reduce_partials_kernel folds the warp rows in a fixed order
// in fp64, so results stay bit-reproducible (engine.py:594-595).
template <typename R>
struct Strip {
  R* row;  // this warp's partial row: [n_slots][2]
  int lane;

  // Reduce one chunk (cnt <= 8 slots) across the warp and store it.
  __device__ __forceinline__ void push(R (&re)[kChunkSlots], R (&im)[kChunkSlots], int cnt, int32_t first_id) {
    transpose_reduce8(re, lane);
    transpose_reduce8(im, lane);
    const int j = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && j < cnt) {
      R* p = row + static_cast<int64_t>(first_id + j) * 2;
      p[0] = re[0];
      p[1] = im[0];
    }
  }
  __device__ __forceinline__ void reserve(int, R*) {}
};

// ---------------------------------------------------------------------------
// spin state in shared memory: [3][S][blockDim] doubles (mx, my, mz)
// ---------------------------------------------------------------------------

template <int S>
struct Spins {
  double* sm;
  int64_t base;  // spin index of slot 0 of this thread
  int bd;
  int64_t n;
  __device__ __forceinline__ int64_t idx(int s) const { return base + static_cast<int64_t>(s) * bd; }
  __device__ __forceinline__ bool act(int s) const { return idx(s) < n; }
  __device__ __forceinline__ double& mx(int s) { return sm[(0 * S + s) * bd + threadIdx.x]; }
  __device__ __forceinline__ double& my(int s) { return sm[(1 * S + s) * bd + threadIdx.x]; }
  __device__ __forceinline__ double& mz(int s) { return sm[(2 * S + s) * bd + threadIdx.x]; }
};

__device__ __forceinline__ double spin_theta(const KParams& kp, int64_t i, double dt, double dmx, double dmy,
                                             double dmz) {
  // engine.py:289 — theta = pos @ dmom + domega * dt
  return fma(kp.z[i], dmz, fma(kp.y[i], dmy, kp.x[i] * dmx)) + kp.dw[i] * dt;
}

// relax-class table: e1 = exp(-T_c/T1_i) at [2c][i], e2 = exp(-T_c/T2_i) at [2c+1][i]
__device__ __forceinline__ double rt_e1(const KParams& kp, int c, int64_t i) {
  return kp.relax[(2 * static_cast<int64_t>(c)) * kp.n + i];
}
__device__ __forceinline__ double rt_e2(const KParams& kp, int c, int64_t i) {
  return kp.relax[(2 * static_cast<int64_t>(c) + 1) * kp.n + i];
}

// rotation-class table (program.h RotClass), SoA [class][field][spin], fp64:
//   0,1 = Cpre; 2,3 = C (whole run); 4,5 = A, B (mz affine map); 6,7 = z (per sample)
struct RotCoef {
  double cr, ci, a, b;
};
constexpr int kRotFields = 8;
__device__ __forceinline__ const double* rot_ptr(const KParams& kp, int c, int64_t i) {
  return kp.rot + static_cast<int64_t>(c) * kRotFields * kp.n + i;
}
__device__ __forceinline__ RotCoef rot_coef(const KParams& kp, int c, int64_t i) {
  const double* t = rot_ptr(kp, c, i);
  RotCoef k;  // read-only path: lets the loads of all spins issue ahead of the shared-memory state stores
  k.cr = __ldg(t + 2 * kp.n);
  k.ci = __ldg(t + 3 * kp.n);
  k.a = __ldg(t + 4 * kp.n);
  k.b = __ldg(t + 5 * kp.n);
  return k;
}

// one interval on spin s: precession (+ relaxation), fp64 — engine.py:288-302
template <int S>
__device__ __forceinline__ void interval(const KParams& kp, Spins<S>& sp, int s, int flags, int cls, double dt,
                                         double dmx, double dmy, double dmz) {
  if (!(flags & EV_MOVE) || !sp.act(s)) return;
  const int64_t i = sp.idx(s);
  double sn, cs;
  phase_sincos<double>(spin_theta(kp, i, dt, dmx, dmy, dmz), sn, cs);
  const double x = sp.mx(s), y = sp.my(s);
  double nx = cs * x + sn * y;  // clockwise, bloch.py:10-17
  double ny = cs * y - sn * x;
  if (cls >= 0) {
    const double e1 = rt_e1(kp, cls, i), e2 = rt_e2(kp, cls, i);
    nx *= e2;
    ny *= e2;
    sp.mz(s) = sp.mz(s) * e1 + kp.m0[i] * (1.0 - e1);
  }
  sp.mx(s) = nx;
  sp.my(s) = ny;
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
      double wr = 1.0, wi = 0.0;
      if (kp.w != nullptr) {
        const double* p = kp.w + (static_cast<int64_t>(c) * kp.n + sp.idx(s)) * 2;
        wr = p[0];
        wi = p[1];
      }
      const double x = sp.mx(s), y = sp.my(s);
      re += wr * x - wi * y;
      im += wr * y + wi * x;
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
                                                const float2 (&ZI)[P], const float2 (&NZI)[P],
                                                float (&ar)[kChunkSlots], float (&ai)[kChunkSlots], int ck) {
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
        const float2 t1 = __fmul2_rn(V[p], NZI[p]);  // -v*zi
        const float2 t2 = __fmul2_rn(V[p], ZR[p]);   //  v*zr
        U[p] = __ffma2_rn(a, ZR[p], t1);             // u*zr - v*zi
        V[p] = __ffma2_rn(a, ZI[p], t2);             // u*zi + v*zr
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

// ---------------------------------------------------------------------------
// the integrator
// ---------------------------------------------------------------------------

template <typename R, int S, int NC>
__global__ void __launch_bounds__(KernelTraits<R, S, NC>::kMaxThreads, KernelTraits<R, S, NC>::kMinBlocks)
    integrate_kernel(const KParams kp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kSampPerChunk = kChunkSlots / NC;
  constexpr bool kPacked = sizeof(R) == 4 && NC == 1 && (S % 2 == 0);
  const int bd = blockDim.x;
  const int nw = bd >> 5;
  Spins<S> sp;
  sp.sm = reinterpret_cast<double*>(smem_raw);
  sp.base = static_cast<int64_t>(blockIdx.x) * kp.spins_per_cta + threadIdx.x;
  sp.bd = bd;
  sp.n = kp.n;
  Strip<R> strip;  // one partial row per warp of the grid
  strip.lane = threadIdx.x & 31;
  strip.row = reinterpret_cast<R*>(kp.partial) +
              (static_cast<int64_t>(blockIdx.x) * nw + (threadIdx.x >> 5)) * kp.part_stride;
  R* part_row = strip.row;

#pragma unroll
  for (int s = 0; s < S; ++s) {
    const bool a = sp.act(s);
    const int64_t i = a ? sp.idx(s) : 0;
    sp.mx(s) = a ? kp.mx0[i] : 0.0;
    sp.my(s) = a ? kp.my0[i] : 0.0;
    sp.mz(s) = a ? kp.mz0[i] : 0.0;
  }

  for (int o = 0; o < kp.n_ops; ++o) {
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
      const int flags = __ldg(&op->count), snap = __ldg(&op->aux), cls = __ldg(&op->cls), rc = __ldg(&op->rot);
      if (rc >= 0) {  // repeated interval: tabulated propagator
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!sp.act(s)) continue;
          const RotCoef k = rot_coef(kp, rc, sp.idx(s));
          const double x = sp.mx(s), y = sp.my(s);
          sp.mx(s) = k.cr * x - k.ci * y;
          sp.my(s) = k.cr * y + k.ci * x;
          sp.mz(s) = fma(sp.mz(s), k.a, k.b);
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

    if (kind == OP_RFTRAIN) {  // discretised shaped pulse: (pulse_j, identical interval) x count
      const int cnt = __ldg(&op->count), m0i = __ldg(&op->aux), flags = __ldg(&op->flags), cls = __ldg(&op->cls);
      const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]), dmz = __ldg(&op->p[3]);
      const double* mats = kp.mats + static_cast<int64_t>(m0i) * 9;
      constexpr int G = S < 4 ? S : 4;  // spins per register group
#pragma unroll
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
          if (!sp.act(s)) continue;
          const int64_t i = sp.idx(s);
          if (flags & EV_MOVE) {
            double sn, cs;
            phase_sincos<double>(spin_theta(kp, i, dt, dmx, dmy, dmz), sn, cs);
            const double e2 = cls >= 0 ? rt_e2(kp, cls, i) : 1.0;
            zr[g] = e2 * cs;
            zi[g] = -e2 * sn;
            if (cls >= 0) {
              e1[g] = rt_e1(kp, cls, i);
              rg[g] = kp.m0[i] * (1.0 - e1[g]);
            }
          }
        }
        for (int j = 0; j < cnt; ++j) {
          double r[9];
#pragma unroll
          for (int k = 0; k < 9; ++k) r[k] = __ldg(mats + 9 * j + k);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const double nx = r[0] * x[g] + r[1] * y[g] + r[2] * z[g];
            const double ny = r[3] * x[g] + r[4] * y[g] + r[5] * z[g];
            const double nz = r[6] * x[g] + r[7] * y[g] + r[8] * z[g];
            x[g] = nx * zr[g] - ny * zi[g];
            y[g] = nx * zi[g] + ny * zr[g];
            z[g] = fma(nz, e1[g], rg[g]);
          }
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
      const int cnt = __ldg(&op->count), g0 = __ldg(&op->aux), s0 = __ldg(&op->s0);
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        strip.reserve(ck * NC, part_row);
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
      const int cnt = __ldg(&op->count), s0 = __ldg(&op->s0), cls = __ldg(&op->cls);
      const double dt = __ldg(&op->p[0]);
      const double d0x = __ldg(&op->p[1]), d0y = __ldg(&op->p[2]), d0z = __ldg(&op->p[3]);
      const double ddx = __ldg(&op->p[4]), ddy = __ldg(&op->p[5]), ddz = __ldg(&op->p[6]);
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        strip.reserve(ck * NC, part_row);
        R ar[kChunkSlots], ai[kChunkSlots];
#pragma unroll
        for (int j = 0; j < kChunkSlots; ++j) ar[j] = ai[j] = R(0);
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!sp.act(s)) continue;
          const int64_t i = sp.idx(s);
          // rotation factor of event k0 and the per-event phase step (exact per chunk)
          const double b = fma(kp.z[i], ddz, fma(kp.y[i], ddy, kp.x[i] * ddx));
          double sn, cs, qs, qc;
          phase_sincos<double>(fma(static_cast<double>(k0), b, spin_theta(kp, i, dt, d0x, d0y, d0z)), sn, cs);
          phase_sincos<double>(b, qs, qc);
          const double e2 = cls >= 0 ? rt_e2(kp, cls, i) : 1.0;
          const double e1 = cls >= 0 ? rt_e1(kp, cls, i) : 1.0;
          const double rgw = kp.m0[i] * (1.0 - e1);
          double rr = e2 * cs, ri = -e2 * sn;
          double x = sp.mx(s), y = sp.my(s), z = sp.mz(s);
          double wr[NC], wi[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            wr[c] = 1.0;
            wi[c] = 0.0;
            if (kp.w != nullptr) {
              const double* p = kp.w + (static_cast<int64_t>(c) * kp.n + i) * 2;
              wr[c] = p[0];
              wi[c] = p[1];
            }
          }
#pragma unroll
          for (int j = 0; j < kSampPerChunk; ++j) {
            if (j < ck) {
              const double nx = x * rr - y * ri;
              y = x * ri + y * rr;
              x = nx;
              if (cls >= 0) z = fma(z, e1, rgw);
              const double a = rr;
              rr = a * qc + ri * qs;  // r <- r * exp(-i b)
              ri = ri * qc - a * qs;
#pragma unroll
              for (int c = 0; c < NC; ++c) {
                ar[j * NC + c] += static_cast<R>(wr[c] * x - wi[c] * y);
                ai[j * NC + c] += static_cast<R>(wr[c] * y + wi[c] * x);
              }
            }
          }
          sp.mx(s) = x;
          sp.my(s) = y;
          sp.mz(s) = z;
        }
        strip.push(ar, ai, ck * NC, (s0 + k0) * NC);
      }
      continue;
    }

    // OP_WINDOW
    {
      const int cnt = __ldg(&op->count), lead = __ldg(&op->aux), s0 = __ldg(&op->s0), rc = __ldg(&op->rot);
      // per-spin setup from the rotation-class table: sample factor z and the
      // closed-form exit propagator (C, A, B) of the whole window
      R zr[S], zi[S], ur[S], ui[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        zr[s] = R(1);
        zi[s] = R(0);
        ur[s] = R(0);
        ui[s] = R(0);
        if (!sp.act(s)) continue;
        const int64_t i = sp.idx(s);
        double pr = 1.0, pi = 0.0;
        RotCoef k;
        if (rc >= 0) {  // tabulated (pre, window, post) propagators
          const double* t = rot_ptr(kp, rc, i);
          pr = __ldg(t);
          pi = __ldg(t + kp.n);
          k = rot_coef(kp, rc, i);
          zr[s] = static_cast<R>(__ldg(t + 6 * kp.n));
          zi[s] = static_cast<R>(__ldg(t + 7 * kp.n));
        } else {  // on the fly: a window whose interval is not reused
          const int c1 = __ldg(&op->cls), cw = __ldg(&op->flags);
          const double dt = __ldg(&op->p[0]);
          const double th = spin_theta(kp, i, dt, __ldg(&op->p[1]), __ldg(&op->p[2]), __ldg(&op->p[3]));
          double sn, cs, SN, CS;
          sincos(reduce_2pi(th), &sn, &cs);
          sincos(reduce_2pi(th * static_cast<double>(cnt - lead)), &SN, &CS);
          const double e2 = c1 >= 0 ? rt_e2(kp, c1, i) : 1.0;
          const double E2 = cw >= 0 ? rt_e2(kp, cw, i) : 1.0;
          k.a = cw >= 0 ? rt_e1(kp, cw, i) : 1.0;
          k.b = kp.m0[i] * (1.0 - k.a);
          k.cr = E2 * CS;
          k.ci = -E2 * SN;
          zr[s] = static_cast<R>(e2 * cs);
          zi[s] = static_cast<R>(-e2 * sn);
        }
        double w0r = 1.0, w0i = 0.0;
        if (kp.w != nullptr && NC == 1) {
          w0r = __ldg(kp.w + 2 * i);
          w0i = __ldg(kp.w + 2 * i + 1);
        }
        const double x = sp.mx(s), y = sp.my(s);
        // state at the first sample: the absorbed pre-interval applied
        const double x0 = pr * x - pi * y, y0 = pr * y + pi * x;
        // NC == 1: track u = w*m (the weight rides along the recurrence); else m
        ur[s] = static_cast<R>(w0r * x0 - w0i * y0);
        ui[s] = static_cast<R>(w0r * y0 + w0i * x0);
        sp.mx(s) = k.cr * x - k.ci * y;
        sp.my(s) = k.cr * y + k.ci * x;
        sp.mz(s) = fma(sp.mz(s), k.a, k.b);
      }
      if constexpr (kPacked) {
        constexpr int P = S / 2;
        float2 U[P], V[P], ZR[P], ZI[P], NZI[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          ZR[p] = make_float2(zr[2 * p], zr[2 * p + 1]);
          ZI[p] = make_float2(zi[2 * p], zi[2 * p + 1]);
          U[p] = make_float2(ur[2 * p], ur[2 * p + 1]);
          V[p] = make_float2(ui[2 * p], ui[2 * p + 1]);
          NZI[p] = make_float2(-ZI[p].x, -ZI[p].y);
        }
        int k0 = 0;
        if (lead && cnt >= kChunkSlots) {
          strip.reserve(kChunkSlots, part_row);
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk_f2<P, true, true>(U, V, ZR, ZI, NZI, ar, ai, kChunkSlots);
          strip.push(ar, ai, kChunkSlots, s0);
          k0 = kChunkSlots;
        }
        // two chunks per trip in one basic block: the warp transpose-reduction of
        // the first (shuffle latency) overlaps the complex multiplies of the second
        for (; k0 + 2 * kChunkSlots <= cnt; k0 += 2 * kChunkSlots) {
          strip.reserve(2 * kChunkSlots, part_row);
          R ar[kChunkSlots], ai[kChunkSlots], br[kChunkSlots], bi[kChunkSlots];
          window_chunk_f2<P, true, false>(U, V, ZR, ZI, NZI, ar, ai, kChunkSlots);
          window_chunk_f2<P, true, false>(U, V, ZR, ZI, NZI, br, bi, kChunkSlots);
          strip.push(ar, ai, kChunkSlots, s0 + k0);
          strip.push(br, bi, kChunkSlots, s0 + k0 + kChunkSlots);
        }
        for (; k0 + kChunkSlots <= cnt; k0 += kChunkSlots) {
          strip.reserve(kChunkSlots, part_row);
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk_f2<P, true, false>(U, V, ZR, ZI, NZI, ar, ai, kChunkSlots);
          strip.push(ar, ai, kChunkSlots, s0 + k0);
        }
        if (k0 < cnt) {
          const int ck = cnt - k0;
          strip.reserve(ck, part_row);
          R ar[kChunkSlots], ai[kChunkSlots];
          if (lead && k0 == 0)
            window_chunk_f2<P, false, true>(U, V, ZR, ZI, NZI, ar, ai, ck);
          else
            window_chunk_f2<P, false, false>(U, V, ZR, ZI, NZI, ar, ai, ck);
          strip.push(ar, ai, ck, s0 + k0);
        }
      } else {
        R wr[NC][S], wi[NC][S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            wr[c][s] = wi[c][s] = R(0);
            if (NC > 1 && sp.act(s)) {
              const double* q = kp.w + (static_cast<int64_t>(c) * kp.n + sp.idx(s)) * 2;
              wr[c][s] = static_cast<R>(q[0]);
              wi[c][s] = static_cast<R>(q[1]);
            }
          }
        }
        int k0 = 0;
        if (lead && cnt >= kSampPerChunk) {
          strip.reserve(kChunkSlots, part_row);
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk<R, S, NC, true, true>(ur, ui, zr, zi, wr, wi, ar, ai, kSampPerChunk);
          strip.push(ar, ai, kChunkSlots, s0 * NC);
          k0 = kSampPerChunk;
        }
        for (; k0 + kSampPerChunk <= cnt; k0 += kSampPerChunk) {
          strip.reserve(kChunkSlots, part_row);
          R ar[kChunkSlots], ai[kChunkSlots];
          window_chunk<R, S, NC, true, false>(ur, ui, zr, zi, wr, wi, ar, ai, kSampPerChunk);
          strip.push(ar, ai, kChunkSlots, (s0 + k0) * NC);
        }
        if (k0 < cnt) {
          const int ck = cnt - k0;
          strip.reserve(ck * NC, part_row);
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
}

// ---------------------------------------------------------------------------
// staging + fold
// ---------------------------------------------------------------------------

__global__ void prep_kernel(int64_t n, const double* __restrict__ pos, const double* __restrict__ t1,
                            const double* __restrict__ t2, double* __restrict__ x, double* __restrict__ y,
                            double* __restrict__ z, double* __restrict__ r1, double* __restrict__ r2) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    x[i] = pos[3 * i + 0];
    y[i] = pos[3 * i + 1];
    z[i] = pos[3 * i + 2];
    r1[i] = 1.0 / t1[i];  // engine.py:270 (inf -> 0: no relaxation)
    r2[i] = 1.0 / t2[i];
  }
}

// relax_cache restated (engine.py:292-299): e1 = exp(-T*inv_t1), e2 = exp(-T*inv_t2)
__global__ void relax_table_kernel(int64_t n, int n_cls, const double* __restrict__ T, const double* __restrict__ r1,
                                   const double* __restrict__ r2, double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n_cls) * n;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = t / n, i = t - c * n;
    const double dt = T[c];
    out[(2 * c) * n + i] = exp(-dt * r1[i]);
    out[(2 * c + 1) * n + i] = exp(-dt * r2[i]);
  }
}

// rotation-class propagators, fp64 (program.h RotClass): for class c and spin i
//   theta = pos.dmom + dw*dt; C = e2^m exp(-i m theta); A = e1^m; B = m0 (1 - A);
//   z = e2 exp(-i theta)
__global__ void rot_table_kernel(int64_t n, int n_cls, const RotClass* __restrict__ rc, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 const double* __restrict__ dw, const double* __restrict__ r1,
                                 const double* __restrict__ r2, const double* __restrict__ m0,
                                 double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n_cls) * n;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = t / n, i = t - c * n;
    const RotClass& k = rc[c];
    const double xi = x[i], yi = y[i], zi = z[i], wi = dw[i];
    auto theta = [&](const double* iv) { return fma(zi, iv[3], fma(yi, iv[2], xi * iv[1])) + wi * iv[0]; };
    const double th_pre = theta(k.pre), th = theta(k.main), th_post = theta(k.post);
    const double T = k.pre[0] + k.main[0] * k.mult + k.post[0];
    double sp, cp, s1, c1, st, ct;
    sincos(reduce_2pi(th_pre), &sp, &cp);
    sincos(reduce_2pi(th), &s1, &c1);
    sincos(reduce_2pi(th_pre + th * k.mult + th_post), &st, &ct);
    const double ep = exp(-k.pre[0] * r2[i]);
    const double e2 = exp(-k.main[0] * r2[i]);
    const double E2 = exp(-T * r2[i]);
    const double E1 = exp(-T * r1[i]);
    double* o = out + c * kRotFields * n + i;
    o[0] = ep * cp;
    o[n] = -ep * sp;
    o[2 * n] = E2 * ct;
    o[3 * n] = -E2 * st;
    o[4 * n] = E1;
    o[5 * n] = m0[i] * (1.0 - E1);
    o[6 * n] = e2 * c1;
    o[7 * n] = -e2 * s1;
  }
}

// pad [nc][n][2] weights to [ncp][n][2] (zero coils beyond nc)
__global__ void pad_weights_kernel(int64_t n, int nc, int ncp, const double* __restrict__ w, double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = t / (n * 2);
    out[t] = c < nc ? w[t] : 0.0;
  }
}

template <typename R>
__global__ void reduce_partials_kernel(const R* __restrict__ part, int grid, int64_t n_slots, int nc, int ncp,
                                       const int64_t* __restrict__ sample_g, int64_t G, double* __restrict__ out) {
  const int64_t total = n_slots * 2;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t sl = t >> 1;
    const int comp = static_cast<int>(t & 1);
    const int64_t s = sl / ncp;
    const int c = static_cast<int>(sl % ncp);
    if (c >= nc) continue;
    double acc = 0.0;
    for (int b = 0; b < grid; ++b) acc += static_cast<double>(part[static_cast<int64_t>(b) * total + t]);
    out[(static_cast<int64_t>(c) * G + sample_g[s]) * 2 + comp] = acc;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

template <typename R, int S, int NC>
size_t integrate_smem_bytes(int threads) {
  const int nw = threads / 32;
  (void)nw;
  return static_cast<size_t>(3 * S * threads) * sizeof(double);
}

template <typename R, int S, int NC>
cudaError_t launch_integrate(const KParams& kp, int grid, int threads, cudaStream_t stream) {
  const size_t smem = integrate_smem_bytes<R, S, NC>(threads);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(integrate_kernel<R, S, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  integrate_kernel<R, S, NC><<<grid, threads, smem, stream>>>(kp);
  return cudaGetLastError();
}

static int grid_for(int64_t total, int threads) {
  const int64_t blocks = (total + threads - 1) / threads;
  return static_cast<int>(blocks < 8192 ? blocks : 8192);
}

cudaError_t launch_prep(int64_t n, const double* pos, const double* t1, const double* t2, double* x, double* y,
                        double* z, double* r1, double* r2, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  prep_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, pos, t1, t2, x, y, z, r1, r2);
  return cudaGetLastError();
}

cudaError_t launch_relax_table(int64_t n, int n_cls, const double* T, const double* r1, const double* r2, double* out,
                               cudaStream_t stream) {
  if (n == 0 || n_cls == 0) return cudaSuccess;
  relax_table_kernel<<<grid_for(static_cast<int64_t>(n_cls) * n, 256), 256, 0, stream>>>(n, n_cls, T, r1, r2, out);
  return cudaGetLastError();
}

cudaError_t launch_rot_table(int64_t n, int n_cls, const RotClass* rc, const double* x, const double* y,
                             const double* z, const double* dw, const double* r1, const double* r2, const double* m0,
                             double* out, cudaStream_t stream) {
  if (n == 0 || n_cls == 0) return cudaSuccess;
  rot_table_kernel<<<grid_for(static_cast<int64_t>(n_cls) * n, 256), 256, 0, stream>>>(n, n_cls, rc, x, y, z, dw, r1,
                                                                                        r2, m0, out);
  return cudaGetLastError();
}

cudaError_t launch_pad_weights(int64_t n, int nc, int ncp, const double* w, double* out, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  if (total == 0) return cudaSuccess;
  pad_weights_kernel<<<grid_for(total, 256), 256, 0, stream>>>(n, nc, ncp, w, out);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_reduce(const R* part, int grid, int64_t n_slots, int nc, int ncp, const int64_t* sample_g,
                          int64_t G, double* out, cudaStream_t stream) {
  const int64_t total = n_slots * 2;
  if (total == 0) return cudaSuccess;
  const int64_t blocks = (total + 255) / 256;
  reduce_partials_kernel<R><<<static_cast<int>(blocks < 65535 ? blocks : 65535), 256, 0, stream>>>(
      part, grid, n_slots, nc, ncp, sample_g, G, out);
  return cudaGetLastError();
}

template <typename R, int S, int NC>
cudaError_t kernel_attrs(int* max_threads, int* regs) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, integrate_kernel<R, S, NC>);
  if (e != cudaSuccess) return e;
  *max_threads = a.maxThreadsPerBlock;
  *regs = a.numRegs;
  return cudaSuccess;
}

#define BLOCH_INST(R, S, NC)                                                              \
  template cudaError_t launch_integrate<R, S, NC>(const KParams&, int, int, cudaStream_t); \
  template cudaError_t kernel_attrs<R, S, NC>(int*, int*);                                 \
  template size_t integrate_smem_bytes<R, S, NC>(int);
BLOCH_FOR_EACH_VARIANT(BLOCH_INST)
#undef BLOCH_INST

template cudaError_t launch_reduce<float>(const float*, int, int64_t, int, int, const int64_t*, int64_t, double*,
                                          cudaStream_t);
template cudaError_t launch_reduce<double>(const double*, int, int64_t, int, int, const int64_t*, int64_t, double*,
                                           cudaStream_t);

}  // namespace bloch
