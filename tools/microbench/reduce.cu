// ADC-sum reduction strategies, measured on their own (no compute), B200.
//
// Each warp of a (grid x NW-warp) launch owns a stream of "windows" of K complex samples
// and, per window, hands its warp-partial sums to one of:
//   mode 0  rows:   its own fp32 partial row (st.global.cs), as integrate_kernel does today
//   mode 1  bulk:   int64 fixed point staged in shared memory, one
//                   cp.reduce.async.bulk.global.shared::cta.add.u64 into replica (cta % R)
//   mode 2  red:    per-lane red.global.add.u64 into replica (cta % R)
//   mode 3  smem:   atom.shared.add.u64 into a per-CTA ring slot (D slots), last-arriving warp
//                   pushes the slot with one bulk add.u64 into replica (cta % R) and frees it
// and reports GB/s of warp-partial payload (K * 8 B per warp per window, the fp32 row size).
//
//   ./reduce MODE K WINDOWS R [GRID NW]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int kD = 4;

__global__ void bench(int mode, int K, int W, int R, float* rows, unsigned long long* rep, int64_t row_stride) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + warp;
  unsigned long long* my_rep = rep + static_cast<int64_t>(blockIdx.x % R) * W * K * 2;
  unsigned long long* stage = reinterpret_cast<unsigned long long*>(sm) + static_cast<int64_t>(warp) * K * 2;
  unsigned long long* ring = reinterpret_cast<unsigned long long*>(sm) + static_cast<int64_t>(nw) * K * 2;
  int* cnt = reinterpret_cast<int*>(ring + kD * K * 2);
  int* gen = cnt + kD;
  if (mode == 3) {
    for (int i = threadIdx.x; i < kD * K * 2; i += blockDim.x) ring[i] = 0;
    if (threadIdx.x < kD) {
      cnt[threadIdx.x] = 0;
      gen[threadIdx.x] = threadIdx.x;  // slot d is free for window d
    }
    __syncthreads();
  }
  float v = 1.0f + 1e-3f * lane;
  for (int w = 0; w < W; ++w) {
    v = v * 1.0001f + 0.5f;
    if (mode == 0) {
      float* row = rows + gw * row_stride + static_cast<int64_t>(w) * K * 2;
      for (int k = lane; k < K * 2; k += 32) __stcs(row + k, v + k);
    } else if (mode == 1) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      __syncwarp();
      for (int k = lane; k < K * 2; k += 32) stage[k] = static_cast<unsigned long long>(__float2ll_rn((v + k) * 1048576.f));
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(stage));
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;\n" ::"l"(
                         my_rep + static_cast<int64_t>(w) * K * 2),
                     "r"(sa), "r"(K * 16)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    } else if (mode == 2) {
      unsigned long long* dst = my_rep + static_cast<int64_t>(w) * K * 2;
      for (int k = lane; k < K * 2; k += 32) atomicAdd(dst + k, static_cast<unsigned long long>(__float2ll_rn((v + k) * 1048576.f)));
    } else {
      const int d = w % kD;
      // wait until slot d belongs to window w
      if (lane == 0)
        while (atomicAdd(gen + d, 0) != w) __nanosleep(64);
      __syncwarp();
      unsigned long long* slot = ring + d * K * 2;
      for (int k = lane; k < K * 2; k += 32) atomicAdd(slot + k, static_cast<unsigned long long>(__float2ll_rn((v + k) * 1048576.f)));
      __threadfence_block();
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(cnt + d, 1) == nw - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence_block();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(slot));
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;\n" ::"l"(
                           my_rep + static_cast<int64_t>(w) * K * 2),
                       "r"(sa), "r"(K * 16)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        }
        __syncwarp();
        for (int k = lane; k < K * 2; k += 32) slot[k] = 0;
        __threadfence_block();
        __syncwarp();
        if (lane == 0) {
          cnt[d] = 0;
          __threadfence_block();
          atomicExch(gen + d, w + kD);
        }
      }
    }
  }
  if (mode == 1 || mode == 3) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int K = argc > 2 ? atoi(argv[2]) : 256;
  const int W = argc > 3 ? atoi(argv[3]) : 256;
  const int R = argc > 4 ? atoi(argv[4]) : 296;
  const int grid = argc > 5 ? atoi(argv[5]) : 296;
  const int nw = argc > 6 ? atoi(argv[6]) : 10;
  const int64_t warps = static_cast<int64_t>(grid) * nw;
  const int64_t row_stride = static_cast<int64_t>(W) * K * 2;
  float* rows = nullptr;
  unsigned long long* rep = nullptr;
  if (mode == 0) CK(cudaMalloc(&rows, warps * row_stride * sizeof(float)));
  CK(cudaMalloc(&rep, static_cast<int64_t>(R) * W * K * 2 * sizeof(unsigned long long)));
  CK(cudaMemset(rep, 0, static_cast<int64_t>(R) * W * K * 2 * sizeof(unsigned long long)));
  size_t smem = static_cast<size_t>(nw) * K * 2 * 8;
  if (mode == 3) smem += kD * K * 2 * 8 + 2 * kD * sizeof(int);
  if (mode == 0 || mode == 2) smem = 0;
  CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  bench<<<grid, nw * 32, smem>>>(mode, K, W, R, rows, rep, row_stride);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    CK(cudaEventRecord(a));
    bench<<<grid, nw * 32, smem>>>(mode, K, W, R, rows, rep, row_stride);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  const double payload = static_cast<double>(warps) * W * K * 8;  // fp32 complex per warp-sample
  printf("mode %d K %d W %d R %d grid %d nw %d smem %zu: %.3f ms, %.1f GB/s of warp partials, %.3f us/window\n", mode,
         K, W, R, grid, nw, smem, best, payload / best / 1e6, best * 1e3 / W);
  return 0;
}
