// The ADC window contraction on tcgen05 (contract.h): warp-specialised, one CTA per SM.
//
//   warp 0     TMA producer: the U tile of each 16-spin stage (hi and lo, SWIZZLE_64B) -> smem
//   warp 1     TMEM owner; lane 0 issues the MMAs (3 bf16 passes per 16-element K step) and
//              commits each stage back to its producers
//   warps 2-5  generate the A tile of each stage (z^k of 16 spins for the CTA's samples, split
//              into bf16 hi/lo, real-embedded, written in the SWIZZLE_64B layout the MMA reads),
//              then read the accumulators out of TMEM into the split-K partial rows
//
// Pipelines: full_u (TMA tx bytes), full_z (4 generator-warp arrivals) -> MMA -> empty
// (tcgen05.commit) -> producers; acc_full (final commit) -> epilogue.  No CTA barrier inside
// the stage loop.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "contract.h"

namespace bloch {
namespace ct {

constexpr int kThreads(int gen_warps) { return 64 + 32 * gen_warps; }  // + A generators (and drains)
constexpr int kStageSpins = 16;            // K = 32 bf16 = 64 B per operand row (one SWIZZLE_64B row)
constexpr int kRowBytes = 64;
constexpr int kTileBytes = 128 * kRowBytes;  // one 128-row operand tile: 8 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// K-major SWIZZLE_64B operand: 64-B rows, 8-row groups 512 B apart (SBO), sm_100 descriptor version 1
__device__ __forceinline__ uint64_t sw64_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fff) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(4) << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ double reduce_2pi(double th) {
  const double k = rint(th * 0.15915494309189535);
  return fma(-k, 2.4492935982947064e-16, fma(-k, 6.283185307179586, th));
}
// z^k = exp(-k a) exp(-i k theta) in fp32 from the tabulated (theta_hi, theta_lo, a): theta_hi has 12
// significant bits, so k theta_hi is exact for k < 4096; the 2 pi reduction is exact up to 2pi_lo
__device__ __forceinline__ float2 zpow32(float4 t, float k) {
  const float p = k * t.x;
  const float nn = __fadd_rn(__fmaf_rn(p, 0.15915494309189535f, 12582912.0f), -12582912.0f);  // rint(p / 2 pi)
  float r = __fmaf_rn(-nn, 6.28125f, p);                   // exact: nn and 6.28125 are short
  r = __fmaf_rn(-nn, 0.0019353071795864769f, r);           // 2 pi - 6.28125
  r = __fmaf_rn(k, t.y, r);
  float sn, cs;
  __sincosf(r, &sn, &cs);
  const float amp = __expf(-k * t.z);
  return make_float2(amp * cs, -amp * sn);
}
// a phase m * head (exact: m and the 12-bit head are short) reduced to [-pi, pi] up to 2pi_lo
__device__ __forceinline__ float red2pi(float p) {
  const float nn = __fadd_rn(__fmaf_rn(p, 0.15915494309189535f, 12582912.0f), -12582912.0f);
  return __fmaf_rn(-nn, 0.0019353071795864769f, __fmaf_rn(-nn, 6.28125f, p));
}
// chirp sample factor r0^m1 q^m2 = exp(-m1 a) exp(-i (m1 theta0 + m2 theta_q)), m1 = k + 1, m2 = k (k + 1) / 2
__device__ __forceinline__ float2 zchirp32(float4 t, float ql, float m1, float m2) {
  float r = red2pi(m1 * t.x) + red2pi(m2 * t.w);
  r = __fmaf_rn(m1, t.y, __fmaf_rn(m2, ql, r));
  float sn, cs;
  __sincosf(r, &sn, &cs);
  const float amp = __expf(-m1 * t.z);
  return make_float2(amp * cs, -amp * sn);
}
// bf16 hi part (round to nearest: Veltkamp split keeping 8 significant bits) and the residual
__device__ __forceinline__ void split_bf16(float x, float& hi, float& lo) {
  const float c = __fmul_rn(x, 65537.0f);
  hi = __fsub_rn(c, __fsub_rn(c, x));
  lo = __fsub_rn(x, hi);
}
__device__ __forceinline__ uint32_t pack2(float lo_elem, float hi_elem) {  // bf16x2: (element 2s, element 2s+1)
  return __byte_perm(__float_as_uint(lo_elem), __float_as_uint(hi_elem), 0x7632);
}

}  // namespace ct

template <int MT, int GW, bool CH>
__global__ void __launch_bounds__(ct::kThreads(GW), 1)
    contract_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                    const ContractJob j, const ContractPlan p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B aligned base (the swizzle pattern is anchored on 512-B boundaries); derived from smem_raw so
  // that the stores below stay STS
  unsigned char* smem = smem_raw + ((1024u - (ct::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = p.nw, nsub = p.nsub, depth = p.depth;
  const int ncol = nsub * nw;                        // windows (accumulator columns) per M-tile
  const int a_bytes = MT * ct::kTileBytes;           // one of A hi / A lo
  const int b_bytes = ncol * ct::kRowBytes;          // one of B hi / B lo
  const int stage_bytes = 2 * a_bytes + 2 * b_bytes;
  auto A = [&](int s, int part) { return smem + s * stage_bytes + part * a_bytes; };
  auto B = [&](int s, int part) { return smem + s * stage_bytes + 2 * a_bytes + part * b_bytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + depth * stage_bytes);
  uint64_t* full_u = bars;
  uint64_t* full_z = bars + depth;
  uint64_t* empty = bars + 2 * depth;
  uint64_t* acc_full = bars + 3 * depth;   // MMA -> drain: a segment's accumulation is complete
  uint64_t* acc_empty = bars + 3 * depth + 1;  // drain -> MMA: the accumulator has been read out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * depth + 2);

  const int tk = blockIdx.x % p.tiles_k;
  const int rest = blockIdx.x / p.tiles_k;
  const int tw = rest % p.tiles_w, kc = rest / p.tiles_w;
  const int coil = tk / p.tpc;
  const int k0 = (tk - coil * p.tpc) * 64 * MT, w0 = tw * ncol;
  const int64_t total_st = (j.n + ct::kStageSpins - 1) / ct::kStageSpins;
  const int64_t st0 = static_cast<int64_t>(kc) * p.stages;
  const int nst = static_cast<int>(min(static_cast<int64_t>(p.stages), total_st - st0));
  const int seg = p.seg;
  auto seg_end = [&](int e) { return min((e + 1) * seg, nst) - 1; };  // last stage of segment e

  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s) {
      ct::mbar_init(full_u + s, 1);
      ct::mbar_init(full_z + s, GW);
      ct::mbar_init(empty + s, 1);
    }
    ct::mbar_init(acc_full, 1);
    ct::mbar_init(acc_empty, GW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ct::smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_hi) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_lo) : "memory");
      for (int t = 0; t < nst; ++t) {
        const int s = t % depth;
        if (t >= depth) ct::mbar_wait(empty + s, ((t / depth) - 1) & 1);
        ct::mbar_expect_tx(full_u + s, 2u * static_cast<uint32_t>(b_bytes));
        const int blk = static_cast<int>(st0 + t);  // 16-spin block = stage
        for (int sub = 0; sub < nsub; ++sub) {
          ct::tma_load_3d(B(s, 0) + sub * nw * ct::kRowBytes, &map_hi, full_u + s, 0, j.row0 + w0 + sub * nw, blk);
          ct::tma_load_3d(B(s, 1) + sub * nw * ct::kRowBytes, &map_lo, full_u + s, 0, j.row0 + w0 + sub * nw, blk);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(nw >> 3) << 17) |
                             (static_cast<uint32_t>(128 >> 4) << 24);
      for (int t = 0; t < nst; ++t) {
        const int s = t % depth;
        const uint32_t ph = (t / depth) & 1;
        const int e = t / seg;
        const bool first = t == e * seg;  // a segment starts: overwrite the accumulator
        if (first && e > 0) ct::mbar_wait(acc_empty, (e - 1) & 1);  // segment e-1 has been read out
        ct::mbar_wait(full_u + s, ph);
        ct::mbar_wait(full_z + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bh = ct::smem_u32(B(s, 0)), bl = ct::smem_u32(B(s, 1));
        if (!(p.dbg & 2)) {
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const uint32_t ah = ct::smem_u32(A(s, 0)) + m * ct::kTileBytes, al = ct::smem_u32(A(s, 1)) + m * ct::kTileBytes;
            for (int sub = 0; sub < nsub; ++sub) {
              const uint32_t d = tmem + static_cast<uint32_t>((m * nsub + sub) * nw);
              const uint32_t bo = sub * nw * ct::kRowBytes;
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {  // two K steps of 16 bf16 (32 B) per 64-B row
                const uint32_t o = ks * 32;
                const uint32_t acc = (!first || ks > 0) ? 1u : 0u;
                ct::mma_bf16(d, ct::sw64_desc(ah + o), ct::sw64_desc(bh + bo + o), idesc, acc);
                ct::mma_bf16(d, ct::sw64_desc(ah + o), ct::sw64_desc(bl + bo + o), idesc, 1u);
                ct::mma_bf16(d, ct::sw64_desc(al + o), ct::sw64_desc(bh + bo + o), idesc, 1u);
              }
            }
          }
        }
        ct::mma_commit(empty + s);
        if (t == seg_end(e)) ct::mma_commit(acc_full);
      }
    }
  } else {
    // ---- generators.  An M-tile holds 64 samples: row r = the sample's real row [Re z^k, -Im z^k],
    // row 64 + r its imaginary row [Im z^k, Re z^k].  Warp q owns samples [8 MT q, 8 MT (q+1)) of the
    // tile, lanes 0-15 the even ones and lanes 16-31 the odd ones (of spin lane & 15): every STS.32 of
    // the warp covers an even and an odd 64-B row, i.e. banks 0-15 and 16-31, and the SWIZZLE_64B chunk
    // permutation ((row >> 1) & 3) is the same for both halves
    const int q = warp - 2, half = lane >> 4, sl = lane & 15;
    constexpr int kSamp = 64 * MT / GW;  // samples per warp per stage
    constexpr int kVals = kSamp / 2;                // per lane
    const int m = (kSamp * q) >> 6;
    const int r0 = ((kSamp * q) & 63) + half;     // row of value 0 (value v: r0 + 2 v)
    const int kfirst = k0 + kSamp * q + half;     // absolute sample of value 0
    const uint32_t off0 = m * ct::kTileBytes + 64 * r0 + ((sl & 3) << 2);
    uint32_t chk[4];                              // swizzled 16-B chunk of this lane's spin, by (row >> 1) & 3
#pragma unroll
    for (int x = 0; x < 4; ++x) chk[x] = ((sl >> 2) ^ ((((kSamp * q) & 63) >> 1) + x & 3)) << 4;
    // ---- drain of accumulation segment e: TMEM lanes of this warp's quarter (two warps per quarter,
    // half of the columns each) -> partial slot (chunk, e); the MMA of the next segment waits for the
    // generator warps' acc_empty arrivals
    const int quarter = warp & 3, colh = q >> 2;  // GW / 4 warps per TMEM lane quarter share the columns
    const int row = 32 * quarter + lane;  // accumulator row: sample k0 + 64 m + (row & 63), component row >> 6
    auto drain = [&](int e) {
      ct::mbar_wait(acc_full, e & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // one slot per (chunk, coil): the first segment stores, the later ones add in fp32 with a reduction
      // (RED.ADD.F32 at L2; the same thread owns an element in every segment, so the order is fixed; the slots
      // of a call fit L2, so they never reach DRAM — one slot per segment wrote and re-read 0.75 GB on config 2)
      // Slot layout [K][2][Wr] (Wr = W rounded up to 16): a thread's 16 accumulator columns are 16 consecutive
      // windows of one (sample, component) row, i.e. 64 contiguous bytes: four 16-byte stores / reductions
      // instead of 16 scattered 4-byte ones.
      const int Wr = (j.W + 15) & ~15;
      float* slot = j.part + (static_cast<int64_t>(kc) * j.C + coil) * j.K * 2 * Wr;
      for (int mm = 0; mm < MT; ++mm) {
        const int k = k0 + 64 * mm + (row & 63);
        for (int c0 = 16 * colh; c0 < ncol; c0 += 16 * (GW / 4)) {
          uint32_t r[16];
          const uint32_t addr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + static_cast<uint32_t>(mm * ncol + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
              : "r"(addr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (k < j.K) {
            float* q = slot + (static_cast<int64_t>(k) * 2 + (row >> 6)) * Wr + (w0 + c0);
            if (((w0 + c0) & 3) == 0 && w0 + c0 + 16 <= Wr) {
#pragma unroll
              for (int c = 0; c < 16; c += 4) {
                if (e == 0)
                  *reinterpret_cast<uint4*>(q + c) = make_uint4(r[c], r[c + 1], r[c + 2], r[c + 3]);
                else  // RED: no load on the drain's path; one thread per element
                  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(q + c), "f"(__uint_as_float(r[c])),
                               "f"(__uint_as_float(r[c + 1])), "f"(__uint_as_float(r[c + 2])),
                               "f"(__uint_as_float(r[c + 3]))
                               : "memory");
              }
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                if (w0 + c0 + c < Wr) {
                  if (e == 0) q[c] = __uint_as_float(r[c]);
                  else atomicAdd(q + c, __uint_as_float(r[c]));
                }
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) ct::mbar_arrive(acc_empty);
    };
    // per-spin phase tables are loaded two stages ahead (one stage of generation does not cover an L2 miss)
    auto load_z = [&](int t, float4& zt, float2& zq, float2& wc) {
      const int64_t i = (st0 + t) * ct::kStageSpins + sl;
      if (t < nst && i < j.n) {
        zt = __ldg(j.zt + i);
        zq = __ldg(j.zq + i);
        wc = j.C > 1 ? __ldg(j.w32 + i * j.ncp + coil) : make_float2(1.f, 0.f);
      } else {
        zt = make_float4(0.f, 0.f, 0.f, 0.f);
        zq = wc = make_float2(0.f, 0.f);
      }
    };
    float4 nzt, mzt;
    float2 nzq, nwc, mzq, mwc;
    load_z(0, nzt, nzq, nwc);
    load_z(1, mzt, mzq, mwc);
    const float kf = static_cast<float>(kfirst);
    int e_next = 0;  // next segment to drain
    for (int t = 0; t < nst; ++t) {
      const float4 czt = nzt;
      const float2 czq = nzq, cwc = nwc;
      nzt = mzt;
      nzq = mzq;
      nwc = mwc;
      load_z(t + 2, mzt, mzq, mwc);
      const int s = t % depth;
      if (t >= depth) {
        ct::mbar_wait(empty + s, ((t / depth) - 1) & 1);
        // stage t - depth completed: when it closed a segment, read that accumulator out now
        // (the MMA has the next depth - 1 stages in hand while it waits)
        if (t - depth == seg_end(e_next)) drain(e_next++);
      }
      if (p.dbg & 1) {
        __syncwarp();
        if (lane == 0) ct::mbar_arrive(full_z + s);
        continue;
      }
      float2 P = make_float2(0.f, 0.f), Q = make_float2(0.f, 0.f);
      const bool live = (st0 + t) * ct::kStageSpins + sl < j.n;
      if (!CH && live) {
        const float2 z0 = ct::zpow32(czt, kf);
        P = make_float2(cwc.x * z0.x - cwc.y * z0.y, cwc.x * z0.y + cwc.y * z0.x);  // the coil weight rides along
        Q = czq;
      }
      unsigned char* ab = A(s, 0) + off0;
#pragma unroll
      for (int v = 0; v < kVals; ++v) {
        unsigned char* o = ab + 128 * v + chk[v & 3];
        if constexpr (CH) {  // chirp: each sample's factor directly (short runs, no recurrence)
          // Rows interleaved over the warps (value v of warp q: row 2 q + half + 2 GW v), so the K <= 64 samples of
          // a short run are shared by all generator warps, and rows beyond the run are skipped: their
          // accumulator rows are never read (a 10-sample ramp costs 1 value per lane in 5 warps, not 4 in 2)
          const int kr = 2 * q + half + 2 * GW * v;
          if (k0 + kr >= j.K) continue;
          const float k = static_cast<float>(k0 + kr);
          const float2 z0 = live ? ct::zchirp32(czt, czq.x, k + 1.f, 0.5f * k * (k + 1.f)) : make_float2(0.f, 0.f);
          P = make_float2(cwc.x * z0.x - cwc.y * z0.y, cwc.x * z0.y + cwc.y * z0.x);
          o = A(s, 0) + 64 * kr + ((sl & 3) << 2) + (((sl >> 2) ^ ((kr >> 1) & 3)) << 4);
        }
        // bf16 hi parts rounded to nearest (Veltkamp, both components packed) and the residuals
        // (scalar __fmul_rn: never contracted into the following subtraction, which would void the split)
        const float2 c = make_float2(__fmul_rn(P.x, 65537.0f), __fmul_rn(P.y, 65537.0f));
        const float2 d = __fadd2_rn(c, make_float2(-P.x, -P.y));
        const float2 hi = __fadd2_rn(c, make_float2(-d.x, -d.y));
        const float2 lo = __fadd2_rn(P, make_float2(-hi.x, -hi.y));
        *reinterpret_cast<uint32_t*>(o) = ct::pack2(hi.x, -hi.y);                   // real row
        *reinterpret_cast<uint32_t*>(o + 4096) = ct::pack2(hi.y, hi.x);             // imaginary row
        *reinterpret_cast<uint32_t*>(o + a_bytes) = ct::pack2(lo.x, -lo.y);
        *reinterpret_cast<uint32_t*>(o + a_bytes + 4096) = ct::pack2(lo.y, lo.x);
        if constexpr (!CH) {
          const float nx = P.x * Q.x - P.y * Q.y;
          P.y = P.x * Q.y + P.y * Q.x;
          P.x = nx;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) ct::mbar_arrive(full_z + s);
    }
    while (e_next * seg < nst) drain(e_next++);  // the remaining segments
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

// per-spin phase tables of one job (fp64 in, fp32 out): theta = pos . d + dw tw (plane_kernel's
// expression) reduced mod 2 pi and split into a 12-significant-bit head and the rest; a = T r2;
// z^2 = exp(-2 a) exp(-2 i theta)
__global__ void contract_prep_kernel(const SpinConst* __restrict__ sc, int64_t n, double T, double d0, double d1,
                                     double d2, double tw, float4* __restrict__ zt, float2* __restrict__ zq,
                                     int chirp, double q0, double q1, double q2, int qconj) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const SpinConst c = sc[i];
    if (chirp) {  // r0 = exp(-T r2) exp(-i theta0), q = exp(-i theta_q): both phases split head / tail
      const double th = ct::reduce_2pi(fma(c.z, d2, fma(c.y, d1, c.x * d0)) + c.dw * tw);
      double thq = ct::reduce_2pi(fma(c.z, q2, fma(c.y, q1, c.x * q0)));
      if (qconj) thq = -thq;
      const float hi = __uint_as_float(__float_as_uint(static_cast<float>(th)) & 0xfffff000u);
      const float hq = __uint_as_float(__float_as_uint(static_cast<float>(thq)) & 0xfffff000u);
      const double a = T != 0.0 ? T * c.r2 : 0.0;
      zt[i] = make_float4(hi, static_cast<float>(th - static_cast<double>(hi)), static_cast<float>(a), hq);
      zq[i] = make_float2(static_cast<float>(thq - static_cast<double>(hq)), 0.f);
      continue;
    }
    const double th = ct::reduce_2pi(fma(c.z, d2, fma(c.y, d1, c.x * d0)) + c.dw * tw);
    const float hi = __uint_as_float(__float_as_uint(static_cast<float>(th)) & 0xfffff000u);
    const float lo = static_cast<float>(th - static_cast<double>(hi));
    const double a = T != 0.0 ? T * c.r2 : 0.0;  // as plane_kernel: no decay without duration
    zt[i] = make_float4(hi, lo, static_cast<float>(a), 0.f);
    double s2, c2;
    sincos(ct::reduce_2pi(2.0 * th), &s2, &c2);
    const double e2 = exp(-2.0 * a);
    zq[i] = make_float2(static_cast<float>(e2 * c2), static_cast<float>(-e2 * s2));
  }
}

// fixed-order fp64 fold of the chunks' partial slots into the echo array (stored, not added)
__global__ void contract_fold_kernel(const float* __restrict__ part, int chunks, int segs, int seg, int stages,
                                     int64_t total_st, int C, int W, int K, int64_t G, const int64_t* __restrict__ out0,
                                     double* __restrict__ echo) {
  const int Wr = (W + 15) & ~15;
  const int64_t per = static_cast<int64_t>(C) * K * 2 * Wr;  // slot layout [C][K][2][Wr]
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < per;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t % Wr, kr = t / Wr;  // kr = (c K + k) 2 + component
    if (w >= W) continue;
    const int64_t comp = kr & 1, ck = kr >> 1, c = ck / K, k = ck - c * K;
    double acc = 0.0;
    for (int ch = 0; ch < chunks; ++ch)
      if (total_st - static_cast<int64_t>(ch) * stages > 0) acc += static_cast<double>(part[static_cast<int64_t>(ch) * per + t]);
    echo[(c * G + out0[w] + k) * 2 + comp] = acc;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

ContractPlan contract_plan(int K, int W, int64_t n, int n_sm, int C) {
  ContractPlan p{};
  // windows per CTA: up to two N-subtiles of <= 256 sharing one generated A tile (generation per MMA
  // halves; the U tile is then re-read by twice as many sample tiles), split evenly (W = 384: 2 x 192)
  static const int nsub_env = [] {
    const char* e = getenv("BLOCH_CONTRACT_NSUB");
    return e ? atoi(e) : 0;
  }();
  const int Wr = ((W + 15) / 16) * 16;
  // two N-subtiles only while the pipeline stays 3 deep (W <= 384): config 4 (W = 384) contraction
  // 5.54 -> 5.36 ms; config 2 (W = 512, depth 2) 3.65 -> 3.81 ms, kept at one (profiles/r2aa_nsub.txt)
  p.nsub = nsub_env == 1 ? 1 : (nsub_env == 2 ? 2 : (Wr > 256 && Wr <= 384 ? 2 : 1));
  const int tw = (W + 256 * p.nsub - 1) / (256 * p.nsub);
  p.nw = (((W + tw * p.nsub - 1) / (tw * p.nsub) + 15) / 16) * 16;
  if (p.nw < 16) p.nw = 16;
  const int ktiles64 = (K + 63) / 64;
  p.mt = 1;
  for (int m : {4, 2}) {
    if (m * p.nsub * p.nw <= 512 && m <= ktiles64) {
      p.mt = m;
      break;
    }
  }
  p.tmem_cols = 32;
  while (p.tmem_cols < p.mt * p.nsub * p.nw) p.tmem_cols <<= 1;
  const int stage = 2 * p.mt * ct::kTileBytes + 2 * p.nsub * p.nw * ct::kRowBytes;
  const int budget = 227 * 1024 - 1024 - 256;  // alignment slack, barriers
  p.depth = budget / stage;
  if (p.depth > 4) p.depth = 4;
  if (p.depth < 2) p.depth = 2;
  p.smem = p.depth * stage + 1024 + 256;
  p.dbg = 0;
  p.tpc = (K + 64 * p.mt - 1) / (64 * p.mt);
  p.tiles_k = C * p.tpc;
  p.tiles_w = (W + p.nsub * p.nw - 1) / (p.nsub * p.nw);
  const int64_t total_st = (n + ct::kStageSpins - 1) / ct::kStageSpins;
  int64_t chunks = n_sm / (p.tiles_k * p.tiles_w);
  if (chunks < 1) chunks = 1;
  if (chunks > total_st) chunks = total_st > 0 ? total_st : 1;
  const int64_t per = (total_st + chunks - 1) / chunks;
  p.stages = static_cast<int>(per > 0 ? per : 1);
  p.chunks = static_cast<int>((total_st + p.stages - 1) / p.stages);
  if (p.chunks < 1) p.chunks = 1;
  // accumulation segments of at most kSegStages stages (6 MMAs each: measured rel. error 1.9e-5 at 128
  // stages, 3.8e-5 at 325, 2.9e-4 unsegmented at 2600, profiles/r2n_*), at most kMaxSegs per chunk
  constexpr int kSegStages = 128, kMaxSegs = 32;
  static const int seg_env = [] {
    const char* e = getenv("BLOCH_CONTRACT_SEG");
    return e ? atoi(e) : 0;
  }();
  p.seg = seg_env > 0 ? seg_env : std::max(kSegStages, (p.stages + kMaxSegs - 1) / kMaxSegs);
  p.segs = (p.stages + p.seg - 1) / p.seg;
  return p;
}

size_t contract_part_bytes(const ContractPlan& p, const ContractJob& j) {
  return static_cast<size_t>(p.chunks) * j.C * ((j.W + 15) & ~15) * j.K * 2 * sizeof(float);
}

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

cudaError_t make_map(CUtensorMap* m, const uint32_t* base, const ContractJob& j, int nw) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // [block][row][32 bf16]: one 64-B row per (block, window)
  const cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(j.rows), static_cast<cuuint64_t>((j.n + 15) / 16)};
  const cuuint64_t strides[2] = {64, static_cast<cuuint64_t>(j.rows) * 64};
  const cuuint32_t box[3] = {32, static_cast<cuuint32_t>(nw), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint32_t*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

std::mutex g_contract_mu;

template <int MT, int GW, bool CH = false>
cudaError_t launch_mt(const CUtensorMap& mh, const CUtensorMap& ml, const ContractJob& j, const ContractPlan& p,
                      cudaStream_t st) {
  static int smem_set[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  {
    std::lock_guard<std::mutex> lk(g_contract_mu);
    if (p.smem > smem_set[dev]) {
      e = cudaFuncSetAttribute(contract_kernel<MT, GW, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
      if (e != cudaSuccess) return e;
      smem_set[dev] = p.smem;
    }
  }
  const int grid = p.tiles_k * p.tiles_w * p.chunks;
  contract_kernel<MT, GW, CH><<<grid, ct::kThreads(GW), p.smem, st>>>(mh, ml, j, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_contract(const ContractJob& j, const ContractPlan& p, cudaStream_t st) {
  if (j.n <= 0 || j.W <= 0 || j.K <= 0) return cudaSuccess;
  if (j.K > kContractMaxSamples || j.C < 1 || (j.C > 1 && !j.w32) || (j.chirp && j.K > 64))
    return cudaErrorInvalidValue;
  {
    const int64_t blocks = (j.n + 255) / 256;
    contract_prep_kernel<<<static_cast<int>(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(
        j.sc, j.n, j.T, j.d[0], j.d[1], j.d[2], j.tw, j.zt, j.zq, j.chirp, j.qd[0], j.qd[1], j.qd[2], j.qconj);
  }
  CUtensorMap mh, ml;
  cudaError_t e = make_map(&mh, j.uhi, j, p.nw);
  if (e == cudaSuccess) e = make_map(&ml, j.ulo, j, p.nw);
  if (e != cudaSuccess) return e;
  // generator warps: 8 (4 for one-M-tile CTAs halve the per-stage overhead per value but hide less latency:
  // config 4 contraction 6.27 vs 5.93 ms, profiles/r2ff_generator_warps.txt; BLOCH_CONTRACT_GW=4 to compare)
  static const int gw_env = [] {
    const char* e = getenv("BLOCH_CONTRACT_GW");
    return e ? atoi(e) : 0;
  }();
  if (j.chirp) {  // chirps: at most kMaxDeferChirp samples, one M-tile
    if (p.mt != 1) return cudaErrorInvalidValue;
    e = launch_mt<1, 8, true>(mh, ml, j, p, st);
  } else switch (p.mt) {
    case 4: e = launch_mt<4, 8>(mh, ml, j, p, st); break;
    case 2: e = launch_mt<2, 8>(mh, ml, j, p, st); break;
    default: e = gw_env == 4 ? launch_mt<1, 4>(mh, ml, j, p, st) : launch_mt<1, 8>(mh, ml, j, p, st); break;
  }
  if (e != cudaSuccess) return e;
  const int64_t per = static_cast<int64_t>(j.C) * ((j.W + 15) & ~15) * j.K * 2;
  const int64_t blocks = (per + 255) / 256;
  const int64_t total_st = (j.n + ct::kStageSpins - 1) / ct::kStageSpins;
  contract_fold_kernel<<<static_cast<int>(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(
      j.part, p.chunks, p.segs, p.seg, p.stages, total_st, j.C, j.W, j.K, j.G, j.out0, j.echo);
  return cudaGetLastError();
}

}  // namespace bloch
