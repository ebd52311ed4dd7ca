// sm_100a kernels of the Bloch event-stream engine.
//
// integrate_kernel<R, S, NC>  — the hot path: restates engine.compute_block
//   (engine.py:259-310) for S spins per thread, each spin's magnetisation held
//   in registers across the whole op stream (program.h).  The op stream is
//   identical for every thread, so all control flow is CTA-uniform and op
//   fields are broadcast loads.  ADC samples are reduced without atomics:
//   per-thread sum over its S spins -> warp transpose-reduction of 8 slots
//   (sample x coil) -> per-warp strip in shared memory -> CTA sum written to
//   this CTA's row of the partial buffer; reduce_partials() then folds the rows
//   in a fixed order in fp64 (deterministic, like the reference's ordered fold,
//   engine.py:594-595).
//
// Precision: the per-spin state (mx, my, mz) is fp64 in every mode — it only
// changes at pulses, generic intervals, RF trains, chirps and window exits.
// R is the type of the ADC sample recurrence inside uniform windows, the
// dominant work: fp32 (BLOCH_PREC_F32) or fp64 (BLOCH_PREC_F64).
//
// Uniform ADC windows (OP_WINDOW): per spin the window rotation
// z = e2 * exp(-i*theta) is formed once (fp64 phase, reduced mod 2pi) and the
// receive-weighted transverse magnetisation u = w * (mx + i*my) is advanced by
// one complex multiply per sample (engine.py:289-305 for every sample of the
// window: same theta, same e2 from the relax cache).  The state that leaves the
// window comes from the closed form m * E2^n * exp(-i*n*theta),
// mz -> m0 + (mz - m0) * E1^n in fp64, so per-sample rounding never feeds back
// into the spin state.
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
__device__ __forceinline__ R relax_exp(double a);
template <>
__device__ __forceinline__ float relax_exp<float>(double a) {
  return expf(static_cast<float>(a));
}
template <>
__device__ __forceinline__ double relax_exp<double>(double a) {
  return exp(a);
}

template <typename R>
__device__ __forceinline__ R shfl_x(R v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Transpose-reduce 8 per-lane slots across the warp.  Afterwards v[0] of lane
// l holds the warp total of slot ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1)
// (identical on the 4 lanes l, l^1, l^2, l^3).  16 shuffles for 8 slots
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

template <typename R>
struct Strip {
  R* val;        // [2][nw][kStripSlots][2]
  int32_t* idx;  // [2][kStripSlots] compact slot id of each strip position
  int nw, warp, lane, slots, buf;

  __device__ __forceinline__ R& at(int b, int w, int s, int comp) {
    return val[((b * nw + w) * kStripSlots + s) * 2 + comp];
  }

  // Reduce one chunk (cnt <= 8 slots) across the warp and append it.
  __device__ __forceinline__ void push(R (&re)[kChunkSlots], R (&im)[kChunkSlots], int cnt,
                                       int32_t first_id) {
    transpose_reduce8(re, lane);
    transpose_reduce8(im, lane);
    const int j = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && j < cnt) {
      at(buf, warp, slots + j, 0) = re[0];
      at(buf, warp, slots + j, 1) = im[0];
    }
    if (warp == 0 && lane < cnt) idx[buf * kStripSlots + slots + lane] = first_id + lane;
    slots += cnt;
  }

  // CTA-wide: sum the warps' strips and write this CTA's partial row.
  // Must be reached by every thread of the CTA (uniform control flow).
  __device__ __forceinline__ void flush(R* part_row) {
    __syncthreads();
    const int total = slots * 2;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int s = t >> 1, comp = t & 1;
      R acc = R(0);
      for (int w = 0; w < nw; ++w) acc += at(buf, w, s, comp);
      part_row[static_cast<int64_t>(idx[buf * kStripSlots + s]) * 2 + comp] = acc;
    }
    buf ^= 1;
    slots = 0;
  }
  __device__ __forceinline__ void reserve(int cnt, R* part_row) {
    if (slots + cnt > kStripSlots) flush(part_row);
  }
};

// ---------------------------------------------------------------------------
// the integrator
// ---------------------------------------------------------------------------

template <int S>
struct SpinState {
  double mx[S], my[S], mz[S];
  int64_t idx[S];
  bool act[S];
};

__device__ __forceinline__ double spin_theta(const KParams& kp, int64_t i, double dt, double dmx,
                                             double dmy, double dmz) {
  // engine.py:289 — theta = pos @ dmom + domega * dt
  return fma(kp.z[i], dmz, fma(kp.y[i], dmy, kp.x[i] * dmx)) + kp.dw[i] * dt;
}

// one interval: precession (+ relaxation) in fp64 — engine.py:288-302
template <int S>
__device__ __forceinline__ void apply_interval(const KParams& kp, SpinState<S>& st, int flags, double dt,
                                               double dmx, double dmy, double dmz) {
  if (!(flags & EV_MOVE)) return;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    if (!st.act[s]) continue;
    const int64_t i = st.idx[s];
    double sn, cs;
    phase_sincos<double>(spin_theta(kp, i, dt, dmx, dmy, dmz), sn, cs);
    const double x = st.mx[s], y = st.my[s];
    st.mx[s] = cs * x + sn * y;  // clockwise, bloch.py:10-17
    st.my[s] = cs * y - sn * x;
    if (flags & EV_RELAX) {
      const double e1 = exp(-dt * kp.r1[i]);
      const double e2 = exp(-dt * kp.r2[i]);
      st.mx[s] *= e2;
      st.my[s] *= e2;
      st.mz[s] = st.mz[s] * e1 + kp.m0[i] * (1.0 - e1);
    }
  }
}

// receive-weighted transverse magnetisation of the current (fp64) state, summed
// over the thread's spins, into slots [base, base+NC) — engine.py:303-305
template <typename R, int S, int NC>
__device__ __forceinline__ void record_state(const KParams& kp, const SpinState<S>& st, R (&ar)[kChunkSlots],
                                             R (&ai)[kChunkSlots], int base) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (!st.act[s]) continue;
      double wr = 1.0, wi = 0.0;
      if (kp.w != nullptr) {
        const double* p = kp.w + (static_cast<int64_t>(c) * kp.n + st.idx[s]) * 2;
        wr = p[0];
        wi = p[1];
      }
      re += wr * st.mx[s] - wi * st.my[s];
      im += wr * st.my[s] + wi * st.mx[s];
    }
    ar[base + c] = static_cast<R>(re);
    ai[base + c] = static_cast<R>(im);
  }
}

template <typename R, int S, int NC>
__global__ void __launch_bounds__(KernelTraits<R, S, NC>::kMaxThreads, 1)
    integrate_kernel(const KParams kp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kSampPerChunk = kChunkSlots / NC;
  const int nw = blockDim.x >> 5;
  Strip<R> strip;
  strip.val = reinterpret_cast<R*>(smem_raw);
  strip.idx = reinterpret_cast<int32_t*>(strip.val + 2 * nw * kStripSlots * 2);
  strip.nw = nw;
  strip.warp = threadIdx.x >> 5;
  strip.lane = threadIdx.x & 31;
  strip.slots = 0;
  strip.buf = 0;
  R* part_row = reinterpret_cast<R*>(kp.partial) + static_cast<int64_t>(blockIdx.x) * kp.part_stride;

  SpinState<S> st;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kp.spins_per_cta + threadIdx.x;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    st.idx[s] = base + static_cast<int64_t>(s) * blockDim.x;
    st.act[s] = st.idx[s] < kp.n;
    const int64_t i = st.act[s] ? st.idx[s] : 0;
    st.mx[s] = st.act[s] ? kp.mx0[i] : 0.0;
    st.my[s] = st.act[s] ? kp.my0[i] : 0.0;
    st.mz[s] = st.act[s] ? kp.mz0[i] : 0.0;
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
        const double x = st.mx[s], y = st.my[s], z = st.mz[s];
        st.mx[s] = r[0] * x + r[1] * y + r[2] * z;
        st.my[s] = r[3] * x + r[4] * y + r[5] * z;
        st.mz[s] = r[6] * x + r[7] * y + r[8] * z;
      }
      continue;
    }

    if (kind == OP_EVENT) {
      const int flags = __ldg(&op->count);
      const int snap = __ldg(&op->aux);
      apply_interval<S>(kp, st, flags, __ldg(&op->p[0]), __ldg(&op->p[1]), __ldg(&op->p[2]), __ldg(&op->p[3]));
      if (snap >= 0 && kp.snaps != nullptr) {  // engine.py:306-308
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!st.act[s]) continue;
          double* q = kp.snaps + (static_cast<int64_t>(snap) * kp.n + st.idx[s]) * 3;
          q[0] = st.mx[s];
          q[1] = st.my[s];
          q[2] = st.mz[s];
        }
      }
      continue;
    }

    if (kind == OP_RFTRAIN) {  // discretised shaped pulse: (pulse_j, identical interval) x count
      const int cnt = __ldg(&op->count);
      const int m0i = __ldg(&op->aux);
      const int flags = __ldg(&op->flags);
      const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]),
                   dmz = __ldg(&op->p[3]);
      double zr[S], zi[S], e1[S], rg[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        zr[s] = 1.0;
        zi[s] = 0.0;
        e1[s] = 1.0;
        rg[s] = 0.0;
        if (!st.act[s]) continue;
        const int64_t i = st.idx[s];
        if (flags & EV_MOVE) {
          double sn, cs;
          phase_sincos<double>(spin_theta(kp, i, dt, dmx, dmy, dmz), sn, cs);
          const double e2 = (flags & EV_RELAX) ? exp(-dt * kp.r2[i]) : 1.0;
          zr[s] = e2 * cs;
          zi[s] = -e2 * sn;
          if (flags & EV_RELAX) {
            e1[s] = exp(-dt * kp.r1[i]);
            rg[s] = kp.m0[i] * (1.0 - e1[s]);
          }
        }
      }
      const double* mats = kp.mats + static_cast<int64_t>(m0i) * 9;
      for (int j = 0; j < cnt; ++j) {
        double r[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) r[k] = __ldg(mats + 9 * j + k);
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double x = st.mx[s], y = st.my[s], z = st.mz[s];
          const double nx = r[0] * x + r[1] * y + r[2] * z;
          const double ny = r[3] * x + r[4] * y + r[5] * z;
          const double nz = r[6] * x + r[7] * y + r[8] * z;
          st.mx[s] = nx * zr[s] - ny * zi[s];
          st.my[s] = nx * zi[s] + ny * zr[s];
          st.mz[s] = (flags & EV_RELAX) ? nz * e1[s] + rg[s] : nz;
        }
      }
      continue;
    }

    if (kind == OP_GSAMP) {  // generic sampled intervals
      const int cnt = __ldg(&op->count);
      const int g0 = __ldg(&op->aux);
      const int s0 = __ldg(&op->s0);
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        strip.reserve(ck * NC, part_row);
        R ar[kChunkSlots], ai[kChunkSlots];
#pragma unroll
        for (int j = 0; j < kSampPerChunk; ++j) {
          if (j < ck) {
            const GEv* g = kp.gev + g0 + k0 + j;
            apply_interval<S>(kp, st, __ldg(&g->flags), __ldg(&g->dt), __ldg(&g->dmx), __ldg(&g->dmy),
                              __ldg(&g->dmz));
            record_state<R, S, NC>(kp, st, ar, ai, j * NC);
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
      const int cnt = __ldg(&op->count);
      const int s0 = __ldg(&op->s0);
      const double dt = __ldg(&op->p[0]);
      const double d0x = __ldg(&op->p[1]), d0y = __ldg(&op->p[2]), d0z = __ldg(&op->p[3]);
      const double ddx = __ldg(&op->p[4]), ddy = __ldg(&op->p[5]), ddz = __ldg(&op->p[6]);
      double rr[S], ri[S], qr[S], qi[S], e1[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        rr[s] = 1.0;
        ri[s] = 0.0;
        qr[s] = 1.0;
        qi[s] = 0.0;
        e1[s] = 1.0;
        if (!st.act[s]) continue;
        const int64_t i = st.idx[s];
        double sn, cs;
        phase_sincos<double>(spin_theta(kp, i, dt, d0x, d0y, d0z), sn, cs);
        const double e2 = dt != 0.0 ? exp(-dt * kp.r2[i]) : 1.0;
        rr[s] = e2 * cs;
        ri[s] = -e2 * sn;
        phase_sincos<double>(fma(kp.z[i], ddz, fma(kp.y[i], ddy, kp.x[i] * ddx)), sn, cs);
        qr[s] = cs;
        qi[s] = -sn;
        if (dt != 0.0) e1[s] = exp(-dt * kp.r1[i]);
      }
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        strip.reserve(ck * NC, part_row);
        R ar[kChunkSlots], ai[kChunkSlots];
#pragma unroll
        for (int j = 0; j < kSampPerChunk; ++j) {
          if (j < ck) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const double x = st.mx[s], y = st.my[s];
              st.mx[s] = x * rr[s] - y * ri[s];
              st.my[s] = x * ri[s] + y * rr[s];
              if (dt != 0.0 && st.act[s]) st.mz[s] = st.mz[s] * e1[s] + kp.m0[st.idx[s]] * (1.0 - e1[s]);
              const double a = rr[s];
              rr[s] = a * qr[s] - ri[s] * qi[s];
              ri[s] = a * qi[s] + ri[s] * qr[s];
            }
            record_state<R, S, NC>(kp, st, ar, ai, j * NC);
          } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) ar[j * NC + c] = ai[j * NC + c] = R(0);
          }
        }
        strip.push(ar, ai, ck * NC, (s0 + k0) * NC);
      }
      continue;
    }

    // OP_WINDOW
    {
      const int cnt = __ldg(&op->count);
      const int lead = __ldg(&op->aux);
      const int s0 = __ldg(&op->s0);
      const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]),
                   dmz = __ldg(&op->p[3]);
      const int nrot = cnt - lead;
      R wr[NC][S], wi[NC][S];
      R zr[S], zi[S], ur[S], ui[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        zr[s] = R(1);
        zi[s] = R(0);
        ur[s] = R(0);
        ui[s] = R(0);
#pragma unroll
        for (int c = 0; c < NC; ++c) wr[c][s] = wi[c][s] = R(0);
        if (!st.act[s]) continue;
        const int64_t i = st.idx[s];
        double w0r = 1.0, w0i = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double a = 1.0, b = 0.0;
          if (kp.w != nullptr) {
            const double* p = kp.w + (static_cast<int64_t>(c) * kp.n + i) * 2;
            a = p[0];
            b = p[1];
          }
          if (c == 0) {
            w0r = a;
            w0i = b;
          }
          wr[c][s] = static_cast<R>(a);
          wi[c][s] = static_cast<R>(b);
        }
        const double th = spin_theta(kp, i, dt, dmx, dmy, dmz);
        const double r1 = kp.r1[i], r2 = kp.r2[i];
        R sn, cs;
        phase_sincos<R>(th, sn, cs);
        const R e2 = dt != 0.0 ? relax_exp<R>(-dt * r2) : R(1);
        zr[s] = e2 * cs;
        zi[s] = -e2 * sn;
        const double x = st.mx[s], y = st.my[s];
        if (NC == 1) {  // track u = w*m: the weight rides along the recurrence
          ur[s] = static_cast<R>(w0r * x - w0i * y);
          ui[s] = static_cast<R>(w0r * y + w0i * x);
        } else {
          ur[s] = static_cast<R>(x);
          ui[s] = static_cast<R>(y);
        }
        // exit state (fp64): m * E2^nrot * exp(-i*nrot*theta); mz relaxes over nrot*dt
        double SN, CS;
        phase_sincos<double>(th * static_cast<double>(nrot), SN, CS);
        const double tn = dt * static_cast<double>(nrot);
        const double E2 = dt != 0.0 ? exp(-tn * r2) : 1.0;
        st.mx[s] = E2 * (CS * x + SN * y);
        st.my[s] = E2 * (CS * y - SN * x);
        if (dt != 0.0) {
          const double m0 = kp.m0[i];
          st.mz[s] = m0 + (st.mz[s] - m0) * exp(-tn * r1);
        }
      }
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        strip.reserve(ck * NC, part_row);
        R ar[kChunkSlots], ai[kChunkSlots];
        const bool first_norot = lead && k0 == 0;
#pragma unroll
        for (int j = 0; j < kSampPerChunk; ++j) {
          if (j < ck) {
            if (!(first_norot && j == 0)) {
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
          } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) ar[j * NC + c] = ai[j * NC + c] = R(0);
          }
        }
        strip.push(ar, ai, ck * NC, (s0 + k0) * NC);
      }
    }
  }
  if (strip.slots > 0) strip.flush(part_row);
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

// pad [nc][n][2] weights to [ncp][n][2] (zero coils beyond nc)
__global__ void pad_weights_kernel(int64_t n, int nc, int ncp, const double* __restrict__ w,
                                   double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = t / (n * 2);
    out[t] = c < nc ? w[t] : 0.0;
  }
}

template <typename R>
__global__ void reduce_partials_kernel(const R* __restrict__ part, int grid, int64_t n_slots, int nc, int ncp,
                                       const int64_t* __restrict__ sample_g, int64_t G,
                                       double* __restrict__ out) {
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
cudaError_t launch_integrate(const KParams& kp, int grid, int threads, cudaStream_t stream) {
  const int nw = threads / 32;
  const size_t smem = static_cast<size_t>(2 * nw * kStripSlots * 2) * sizeof(R) +
                      static_cast<size_t>(2 * kStripSlots) * sizeof(int32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(integrate_kernel<R, S, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  integrate_kernel<R, S, NC><<<grid, threads, smem, stream>>>(kp);
  return cudaGetLastError();
}

cudaError_t launch_prep(int64_t n, const double* pos, const double* t1, const double* t2, double* x, double* y,
                        double* z, double* r1, double* r2, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  prep_kernel<<<static_cast<int>(blocks < 4096 ? blocks : 4096), threads, 0, stream>>>(n, pos, t1, t2, x, y, z,
                                                                                       r1, r2);
  return cudaGetLastError();
}

cudaError_t launch_pad_weights(int64_t n, int nc, int ncp, const double* w, double* out, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  pad_weights_kernel<<<static_cast<int>(blocks < 4096 ? blocks : 4096), threads, 0, stream>>>(n, nc, ncp, w, out);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_reduce(const R* part, int grid, int64_t n_slots, int nc, int ncp, const int64_t* sample_g,
                          int64_t G, double* out, cudaStream_t stream) {
  const int64_t total = n_slots * 2;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  reduce_partials_kernel<R><<<static_cast<int>(blocks < 65535 ? blocks : 65535), threads, 0, stream>>>(
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
  template cudaError_t kernel_attrs<R, S, NC>(int*, int*);
BLOCH_FOR_EACH_VARIANT(BLOCH_INST)
#undef BLOCH_INST

template cudaError_t launch_reduce<float>(const float*, int, int64_t, int, int, const int64_t*, int64_t, double*,
                                          cudaStream_t);
template cudaError_t launch_reduce<double>(const double*, int, int64_t, int, int, const int64_t*, int64_t,
                                           double*, cudaStream_t);

}  // namespace bloch
