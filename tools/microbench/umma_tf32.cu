// tcgen05 (UMMA) kind::tf32 microtest: one CTA, D[128][256] = A[128][K] * B[256][K]^T, K-major SWIZZLE_NONE
// operands in shared memory, accumulator in TMEM, read back with tcgen05.ld.  Checks against a host fp64
// product of the tf32-truncated inputs, then times back-to-back MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_tf32 umma_tf32.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

constexpr int M = 128, N = 256, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// canonical K-major, no swizzle: [row/8][kchunk(2 per 8-k step)][row%8][4 tf32]; k-steps of 8 stacked
__device__ __forceinline__ int koff(int row, int k, int rows) {
  const int ks = k >> 3, kc = (k >> 2) & 1, ke = k & 3;
  return ks * rows * 8 + (row >> 3) * 64 + kc * 32 + (row & 7) * 4 + ke;  // in floats
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3fff);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3fff) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3fff) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version 1 (sm100)
  return d;                             // base offset 0, layout SWIZZLE_NONE (0)
}

__global__ void umma_test(const float* A, const float* B, float* D, int reps, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sa = reinterpret_cast<float*>(smem);
  float* sb = sa + M * K;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) sa[koff(i / K, i % K, M)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) sb[koff(i / K, i % K, N)] = B[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                         (static_cast<uint32_t>(M >> 4) << 24);
  long long t0 = 0, t1 = 0;
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (tid == 0) {
      t0 = clock64();
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t da = sdesc(smem_u32(sa + ks * M * 8), 128, 256);
        const uint64_t db = sdesc(smem_u32(sb + ks * N * 8), 128, 256);
        const uint32_t acc = ks > 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // everyone waits for the MMAs of this rep
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(phase));
    }
    phase ^= 1;
    if (tid == 0) t1 = clock64();
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // TMEM -> registers: warp w reads lanes 32w..32w+31 (= rows), 8 columns at a time
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    const uint32_t addr = tm + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + (tid & 31);
    for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
  if (tid == 0) cycles[0] = t1 - t0;
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2.f - 1.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2.f - 1.f;
  float *dA, *dB, *dD;
  long long* dc;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 4;
  cudaFuncSetAttribute(umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_test<<<1, 128, smem>>>(dA, dB, dD, 1, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  auto tf32 = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return (double)y; };
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += tf32(A[m * K + k]) * tf32(B[n * K + k]);
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("umma tf32 M=%d N=%d K=%d: max |err| %.3e (max |ref| %.3e) D[0]=%f D[1]=%f D[N]=%f\n", M, N, K, maxerr, maxref,
         D[0], D[1], D[N]);
  // timing: reps of K/8 MMAs each
  const int reps = 200;
  umma_test<<<1, 128, smem>>>(dA, dB, dD, reps, dc);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("last rep: %lld cycles for %d MMAs of %d MAC -> %.1f MAC/clk/SM (one rep, issue to commit)\n", cyc, K / 8,
         M * N * 8, (double)M * N * K / cyc);
  return 0;
}
