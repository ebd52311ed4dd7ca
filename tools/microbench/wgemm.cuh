// Window contraction on the 5th-generation tensor cores (tcgen05 / UMMA, sm_100a).
//
// All ADC windows of one rotation class share the per-sample factor z_s of
// every spin, so their samples form ONE product over spins:
//
//     S[w][k] = sum_s U[w][s] z_s^k        w < R windows, k < NS samples
//
// U[w][s] is the weighted transverse magnetisation of spin s at the first
// sample of window w (written by the integrator).  The complex product is
// embedded as a real GEMM D = A B^T with K = (spin, re/im):
//     A[w][(s,re)] = Re U,  A[w][(s,im)] = Im U                       (M = windows)
//     B[(k,re)][(s,re)] = Re z^k, B[(k,re)][(s,im)] = -Im z^k        (N = 2 x samples)
//     B[(k,im)][(s,re)] = Im z^k, B[(k,im)][(s,im)] =  Re z^k
// so D[w][(k,re)] = Re S, D[w][(k,im)] = Im S.  Every operand x is split into
// tf32 parts x = hi + lo and the product runs as three tcgen05.mma kind::tf32
// passes (hi hi + hi lo + lo hi, ~2^-21 relative per product).
//
// One CTA owns all windows of the group (up to 4 M-tiles of 128 rows, one TMEM
// accumulator region each), one N-tile of samples and one K-chunk of spins
// (split-K; partial sums per chunk, folded in a fixed order afterwards).  Per
// stage of 8 spins: A (pre-split by the integrator) arrives by cp.async, B is
// generated in shared memory from z (a complex power chain per spin and
// segment), then one thread issues the MMAs and commits them to the stage's
// mbarrier; the next stage's loads and generation overlap those MMAs.
// Shared-memory operands use the canonical K-major SWIZZLE_NONE layout: core
// matrices of 8 rows x 16 B, LBO = 128 B between the two K-halves of a k8
// step, SBO = 256 B between 8-row groups (tools/microbench/umma_tf32.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bloch {

struct WGemmArgs {
  const float* uhi;  // [R][ldu]: (Re U, Im U) per spin, tf32-exact hi parts
  const float* ulo;  // [R][ldu]: lo parts (x - hi)
  const float2* z;   // [npad] per-spin sample factor, fp32; zero beyond the spin count
  int R;             // windows (rows), <= 512
  int NS;            // samples per window
  int npad;          // spins, a multiple of 8 (U and z zero-padded)
  int64_t ldu;       // floats per U row (>= 2 npad)
  float2* part;      // [k_chunks][R][NS] complex partial sums
};

struct WGemmShape {
  int m_tiles, n_tile, n_tiles, k_chunks, stages_per_chunk, na, smem;
};

constexpr int kWgThreads = 256;
constexpr int kWgStageSpins = 8;  // K = 16 floats per row per stage = two k8 MMA steps

inline WGemmShape wgemm_shape(int R, int NS, int npad, int n_sm) {
  WGemmShape s{};
  s.m_tiles = (R + 127) / 128;
  const int cols = 512 / s.m_tiles;                  // TMEM columns per M-tile
  int nt = (cols < 256 ? cols : 256) / 2;           // samples per N-tile (N = 2 nt <= 256)
  nt = nt / 8 * 8;                                  // N a multiple of 16
  if (nt > (NS + 7) / 8 * 8) nt = (NS + 7) / 8 * 8;
  s.n_tile = nt;
  s.n_tiles = (NS + nt - 1) / nt;
  const int stages = npad / kWgStageSpins;
  int kc = (n_sm + s.n_tiles - 1) / s.n_tiles;
  if (kc > stages) kc = stages;
  if (kc < 1) kc = 1;
  s.stages_per_chunk = (stages + kc - 1) / kc;
  s.k_chunks = (stages + s.stages_per_chunk - 1) / s.stages_per_chunk;  // no empty chunk
  const int ra = s.m_tiles * 128, rb = 2 * nt;
  const int a_slot = 2 * ra * 16 * 4, b_slot = 2 * rb * 16 * 4;  // hi + lo, 16 floats per row
  int na = (227 * 1024 - 2 * b_slot - 256) / a_slot;             // A ring depth (loads run ahead)
  s.na = na > 4 ? 4 : (na < 2 ? 2 : na);
  s.smem = s.na * a_slot + 2 * b_slot + 256;
  return s;
}

namespace wg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// canonical K-major, no swizzle: [k8 step][row / 8][K half][row % 8][4 floats]
__device__ __forceinline__ int off(int row, int k, int rows) {
  return (k >> 3) * rows * 8 + (row >> 3) * 64 + ((k >> 2) & 1) * 32 + (row & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fff) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (static_cast<uint64_t>(1) << 46);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
struct c32 {
  float r, i;
};
__device__ __forceinline__ c32 cm(c32 a, c32 b) { return c32{a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ c32 cpow(c32 z, int e) {  // z^e, e >= 0, binary powering in fp32
  c32 r{1.f, 0.f};
  while (e) {
    if (e & 1) r = cm(r, z);
    z = cm(z, z);
    e >>= 1;
  }
  return r;
}
__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
  lo = x - hi;
}

}  // namespace wg

__global__ void __launch_bounds__(kWgThreads, 1) wgemm_kernel(const WGemmArgs a, const WGemmShape sh) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ra = sh.m_tiles * 128, rb = 2 * sh.n_tile, na = sh.na;
  float* base = reinterpret_cast<float*>(smem);
  // A ring [na][hi, lo][ra x 16], then B [2][hi, lo][rb x 16], then barriers
  auto sA = [&](int slot, int part) { return base + (slot * 2 + part) * ra * 16; };
  auto sB = [&](int slot, int part) { return base + na * 2 * ra * 16 + (slot * 2 + part) * rb * 16; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + na * 2 * ra * 16 + 2 * 2 * rb * 16);  // [na] + done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);

  const int nt = blockIdx.x, kc = blockIdx.y;
  const int k0 = nt * sh.n_tile;  // first sample of this N-tile
  const int st0 = kc * sh.stages_per_chunk;
  int st1 = st0 + sh.stages_per_chunk;
  if (st1 > a.npad / kWgStageSpins) st1 = a.npad / kWgStageSpins;
  const int nst = st1 - st0;

  if (tid == 0) {
    for (int b = 0; b < 5; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wg::smem_u32(bars + b)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(wg::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(rb >> 3) << 17) |
                         (static_cast<uint32_t>(128 >> 4) << 24);
  const int seg_len = sh.n_tile / 8;  // B generation: 64 threads = (spin, segment of seg_len samples)

  auto load_a = [&](int i) {  // stage i's A (hi and lo) into ring slot i % na; always commits a group
    if (i < nst) {
      const int s0 = (st0 + i) * kWgStageSpins, slot = i % na;
      for (int c = tid; c < 2 * ra * 4; c += kWgThreads) {
        const int part = c / (ra * 4), rc = c % (ra * 4), row = rc >> 2, q = rc & 3;
        const bool valid = row < a.R;
        const float* src = (part ? a.ulo : a.uhi) + static_cast<int64_t>(valid ? row : 0) * a.ldu + 2 * s0 + 4 * q;
        wg::cp16(sA(slot, part) + wg::off(row, 4 * q, ra), src, valid);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto mma_done = [&](int i) { wg::wait(bars + i % na, (i / na) & 1); };  // stage i's MMAs completed

  for (int i = 0; i < na - 1; ++i) load_a(i);  // prologue: stages 0 .. na-2 in flight
  for (int i = 0; i < nst; ++i) {
    const int b = i & 1;
    if (i >= 2) mma_done(i - 2);  // B slot b free (normally long done)
    if (tid < 64) {
      const int s = tid >> 3, seg = tid & 7;
      const float2 zf = __ldg(a.z + (st0 + i) * kWgStageSpins + s);
      const wg::c32 z{zf.x, zf.y};
      wg::c32 p = wg::cpow(z, k0 + seg * seg_len);
      float* bh = sB(b, 0);
      float* bl = sB(b, 1);
      const int kk = 2 * s;  // K index of (s, re)
      for (int j = 0; j < seg_len; ++j) {
        const int kl = seg * seg_len + j;  // sample within the N-tile
        float rh, rl, ih, il;
        wg::split(p.r, rh, rl);
        wg::split(p.i, ih, il);
        // row (k, re) = [Re, -Im]; row (k, im) = [Im, Re]
        *reinterpret_cast<float2*>(bh + wg::off(2 * kl, kk, rb)) = make_float2(rh, -ih);
        *reinterpret_cast<float2*>(bh + wg::off(2 * kl + 1, kk, rb)) = make_float2(ih, rh);
        *reinterpret_cast<float2*>(bl + wg::off(2 * kl, kk, rb)) = make_float2(rl, -il);
        *reinterpret_cast<float2*>(bl + wg::off(2 * kl + 1, kk, rb)) = make_float2(il, rl);
        p = wg::cm(p, z);
      }
    }
    // stage i's A group: committed groups are stages <= i + na - 2
    if (na == 2) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    else if (na == 3) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int slot = i % na;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t bhi = wg::smem_u32(sB(b, 0) + ks * rb * 8), blo = wg::smem_u32(sB(b, 1) + ks * rb * 8);
        for (int m = 0; m < sh.m_tiles; ++m) {
          const uint32_t ahi = wg::smem_u32(sA(slot, 0) + ks * ra * 8 + m * 128 * 8);
          const uint32_t alo = wg::smem_u32(sA(slot, 1) + ks * ra * 8 + m * 128 * 8);
          const uint32_t d = tmem + static_cast<uint32_t>(m * rb);
          const uint32_t acc0 = (i > 0 || ks > 0) ? 1u : 0u;
          wg::mma(d, wg::desc(ahi), wg::desc(bhi), idesc, acc0);
          wg::mma(d, wg::desc(ahi), wg::desc(blo), idesc, 1u);
          wg::mma(d, wg::desc(alo), wg::desc(bhi), idesc, 1u);
        }
      }
      wg::commit(bars + slot);
    }
    // refill: stage i + na - 1 goes to slot (i - 1) % na, read by stage i - 1's MMAs
    if (i >= 1) mma_done(i - 1);
    load_a(i + na - 1);
  }
  if (tid == 0) wg::commit(bars + 4);
  wg::wait(bars + 4, 0);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (rows), half of the columns
  const int q = warp & 3, half = warp >> 2;
  for (int m = 0; m < sh.m_tiles; ++m) {
    const int row = m * 128 + q * 32 + lane;
    for (int c0 = half * (rb / 2); c0 < (half + 1) * (rb / 2); c0 += 8) {
      uint32_t r[8];
      const uint32_t addr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(m * rb + c0);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (row < a.R) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = k0 + c0 / 2 + j;
          if (k < a.NS)
            a.part[(static_cast<int64_t>(kc) * a.R + row) * a.NS + k] =
                make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

inline cudaError_t launch_wgemm(const WGemmArgs& a, const WGemmShape& sh, cudaStream_t stream) {
  static int smem_set = 0;
  if (sh.smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(wgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem);
    if (e != cudaSuccess) return e;
    smem_set = sh.smem;
  }
  wgemm_kernel<<<dim3(sh.n_tiles, sh.k_chunks), kWgThreads, sh.smem, stream>>>(a, sh);
  return cudaGetLastError();
}

}  // namespace bloch
