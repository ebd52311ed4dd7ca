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
// Uniform ADC windows (OP_WINDOW) are the dominant work.  Per spin the window
// rotation z = e2 * exp(-i*theta) is formed once (fp64 phase, reduced mod 2pi)
// and the receive-weighted transverse magnetisation u = w * (mx + i*my) is
// advanced by one complex multiply per sample (engine.py:289-305 for every
// sample of the window: same theta, same e2 from the relax cache).  The state
// that leaves the window is computed directly from the closed form
// m * E2^n * exp(-i*n*theta), mz -> m0 + (mz - m0) * E1^n, so per-sample
// rounding never feeds back into the spin state.
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
// (identical on the 4 lanes l, l^1, l^2, l^3).  31 shuffles for 8 slots
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

template <typename R, int S, int NC>
struct SpinRegs {
  R mx[S], my[S], mz[S];
  int64_t idx[S];
  bool act[S];
};

template <typename R, int S, int NC>
__device__ __forceinline__ double spin_theta(const KParams& kp, int64_t i, bool a, double dt,
                                             double dmx, double dmy, double dmz) {
  // engine.py:289 — theta = pos @ dmom + domega * dt
  if (!a) return 0.0;
  return fma(kp.z[i], dmz, fma(kp.y[i], dmy, kp.x[i] * dmx)) + kp.dw[i] * dt;
}

template <typename R, int S, int NC>
__device__ __forceinline__ void load_weights(const KParams& kp, const SpinRegs<R, S, NC>& st,
                                             R (&wr)[NC][S], R (&wi)[NC][S]) {
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (!st.act[s]) {
        wr[c][s] = R(0);
        wi[c][s] = R(0);
      } else if (kp.w == nullptr) {
        wr[c][s] = R(1);
        wi[c][s] = R(0);
      } else {
        const double* p = kp.w + (static_cast<int64_t>(c) * kp.n + st.idx[s]) * 2;
        wr[c][s] = static_cast<R>(p[0]);
        wi[c][s] = static_cast<R>(p[1]);
      }
    }
}

// one interval: precession (+ relaxation) — engine.py:288-302
template <typename R, int S, int NC>
__device__ __forceinline__ void apply_interval(const KParams& kp, SpinRegs<R, S, NC>& st,
                                               int flags, double dt, double dmx, double dmy,
                                               double dmz) {
  if (!(flags & EV_MOVE)) return;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const double th = spin_theta<R, S, NC>(kp, st.idx[s], st.act[s], dt, dmx, dmy, dmz);
    R sn, cs;
    phase_sincos<R>(th, sn, cs);
    const R x = st.mx[s], y = st.my[s];
    st.mx[s] = cs * x + sn * y;  // clockwise, bloch.py:10-17
    st.my[s] = cs * y - sn * x;
  }
  if (flags & EV_RELAX) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (!st.act[s]) continue;
      const int64_t i = st.idx[s];
      const R e1 = relax_exp<R>(-dt * kp.r1[i]);
      const R e2 = relax_exp<R>(-dt * kp.r2[i]);
      const R m0 = static_cast<R>(kp.m0[i]);
      st.mx[s] *= e2;
      st.my[s] *= e2;
      st.mz[s] = st.mz[s] * e1 + m0 * (R(1) - e1);
    }
  }
}

// record the receive-weighted transverse magnetisation of the current state into
// slots [base, base+NC) of the chunk accumulators — engine.py:303-305
template <typename R, int S, int NC>
__device__ __forceinline__ void record(const SpinRegs<R, S, NC>& st, const R (&wr)[NC][S],
                                       const R (&wi)[NC][S], R (&ar)[kChunkSlots],
                                       R (&ai)[kChunkSlots], int base) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    R re = R(0), im = R(0);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      re += wr[c][s] * st.mx[s] - wi[c][s] * st.my[s];
      im += wr[c][s] * st.my[s] + wi[c][s] * st.mx[s];
    }
    ar[base + c] = re;
    ai[base + c] = im;
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

  SpinRegs<R, S, NC> st;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kp.spins_per_cta + threadIdx.x;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    st.idx[s] = base + static_cast<int64_t>(s) * blockDim.x;
    st.act[s] = st.idx[s] < kp.n;
    const int64_t i = st.act[s] ? st.idx[s] : 0;
    st.mx[s] = st.act[s] ? static_cast<R>(kp.mx0[i]) : R(0);
    st.my[s] = st.act[s] ? static_cast<R>(kp.my0[i]) : R(0);
    st.mz[s] = st.act[s] ? static_cast<R>(kp.mz0[i]) : R(0);
  }

  for (int o = 0; o < kp.n_ops; ++o) {
    const DevOp* op = kp.ops + o;
    const int kind = __ldg(&op->kind);

    if (kind == OP_ROT) {  // engine.py:277-283
      R r[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        if constexpr (sizeof(R) == 4)
          r[k] = __ldg(&op->f[k]);
        else
          r[k] = __ldg(&op->p[k]);
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const R x = st.mx[s], y = st.my[s], z = st.mz[s];
        st.mx[s] = r[0] * x + r[1] * y + r[2] * z;
        st.my[s] = r[3] * x + r[4] * y + r[5] * z;
        st.mz[s] = r[6] * x + r[7] * y + r[8] * z;
      }
      continue;
    }

    if (kind == OP_EVENT) {
      const int flags = __ldg(&op->count);
      const int snap = __ldg(&op->aux);
      apply_interval<R, S, NC>(kp, st, flags, __ldg(&op->p[0]), __ldg(&op->p[1]),
                               __ldg(&op->p[2]), __ldg(&op->p[3]));
      if (snap >= 0 && kp.snaps != nullptr) {  // engine.py:306-308
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!st.act[s]) continue;
          double* q = kp.snaps + (static_cast<int64_t>(snap) * kp.n + st.idx[s]) * 3;
          q[0] = static_cast<double>(st.mx[s]);
          q[1] = static_cast<double>(st.my[s]);
          q[2] = static_cast<double>(st.mz[s]);
        }
      }
      continue;
    }

    if (kind == OP_GSAMP) {  // generic sampled intervals
      const int cnt = __ldg(&op->count);
      const int g0 = __ldg(&op->aux);
      const int s0 = __ldg(&op->s0);
      R wr[NC][S], wi[NC][S];
      load_weights<R, S, NC>(kp, st, wr, wi);
      for (int k0 = 0; k0 < cnt; k0 += kSampPerChunk) {
        const int ck = min(kSampPerChunk, cnt - k0);
        strip.reserve(ck * NC, part_row);
        R ar[kChunkSlots], ai[kChunkSlots];
#pragma unroll
        for (int j = 0; j < kSampPerChunk; ++j) {
          if (j < ck) {
            const GEv* g = kp.gev + g0 + k0 + j;
            apply_interval<R, S, NC>(kp, st, __ldg(&g->flags), __ldg(&g->dt), __ldg(&g->dmx),
                                     __ldg(&g->dmy), __ldg(&g->dmz));
            record<R, S, NC>(st, wr, wi, ar, ai, j * NC);
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
      load_weights<R, S, NC>(kp, st, wr, wi);
      // per-spin window propagator z and the closed-form exit state
      R zr[S], zi[S], ur[S], ui[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double th = spin_theta<R, S, NC>(kp, st.idx[s], st.act[s], dt, dmx, dmy, dmz);
        const int64_t i = st.act[s] ? st.idx[s] : 0;
        const double r1 = st.act[s] ? kp.r1[i] : 0.0, r2 = st.act[s] ? kp.r2[i] : 0.0;
        R sn, cs;
        phase_sincos<R>(th, sn, cs);
        const R e2 = dt != 0.0 ? relax_exp<R>(-dt * r2) : R(1);
        zr[s] = e2 * cs;
        zi[s] = -e2 * sn;
        if (NC == 1) {  // track u = w*m: the weight rides along the recurrence
          ur[s] = wr[0][s] * st.mx[s] - wi[0][s] * st.my[s];
          ui[s] = wr[0][s] * st.my[s] + wi[0][s] * st.mx[s];
        } else {
          ur[s] = st.mx[s];
          ui[s] = st.my[s];
        }
        // exit state: m * E2^nrot * exp(-i*nrot*theta); mz relaxes over nrot*dt
        R SN, CS;
        phase_sincos<R>(th * static_cast<double>(nrot), SN, CS);
        const double tn = dt * static_cast<double>(nrot);
        const R E2 = dt != 0.0 ? relax_exp<R>(-tn * r2) : R(1);
        const R x = st.mx[s], y = st.my[s];
        st.mx[s] = E2 * (CS * x + SN * y);
        st.my[s] = E2 * (CS * y - SN * x);
        if (dt != 0.0 && st.act[s]) {
          const R E1 = relax_exp<R>(-tn * r1);
          const R m0 = static_cast<R>(kp.m0[i]);
          st.mz[s] = m0 + (st.mz[s] - m0) * E1;
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
                            const double* __restrict__ t2, double* __restrict__ x,
                            double* __restrict__ y, double* __restrict__ z, double* __restrict__ r1,
                            double* __restrict__ r2) {
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
__global__ void reduce_partials_kernel(const R* __restrict__ part, int grid, int64_t n_slots, int nc,
                                       int ncp, const int64_t* __restrict__ sample_g, int64_t G,
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
    cudaError_t e = cudaFuncSetAttribute(integrate_kernel<R, S, NC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  integrate_kernel<R, S, NC><<<grid, threads, smem, stream>>>(kp);
  return cudaGetLastError();
}

cudaError_t launch_prep(int64_t n, const double* pos, const double* t1, const double* t2, double* x,
                        double* y, double* z, double* r1, double* r2, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  prep_kernel<<<static_cast<int>(blocks < 4096 ? blocks : 4096), threads, 0, stream>>>(
      n, pos, t1, t2, x, y, z, r1, r2);
  return cudaGetLastError();
}

cudaError_t launch_pad_weights(int64_t n, int nc, int ncp, const double* w, double* out,
                               cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(ncp) * n * 2;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  pad_weights_kernel<<<static_cast<int>(blocks < 4096 ? blocks : 4096), threads, 0, stream>>>(
      n, nc, ncp, w, out);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_reduce(const R* part, int grid, int64_t n_slots, int nc, int ncp,
                          const int64_t* sample_g, int64_t G, double* out, cudaStream_t stream) {
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

template cudaError_t launch_reduce<float>(const float*, int, int64_t, int, int, const int64_t*,
                                          int64_t, double*, cudaStream_t);
template cudaError_t launch_reduce<double>(const double*, int, int64_t, int, int, const int64_t*,
                                           int64_t, double*, cudaStream_t);

}  // namespace bloch
