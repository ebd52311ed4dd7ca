// Legacy warp-level tensor-core throughput on sm_100a (HMMA via mma.sync), plus the
// f32 -> bf16x2 conversion the split-precision window formulation would need.
// Each warp runs NCH independent accumulator chains; cycles from clock64().
// Prints MAC/clk/SM so it compares directly with the FFMA pipe (128 FMA/clk/SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define ITERS 2048

template <int NCH>
__global__ void k_bf16(float* out, long long* cyc) {
  uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a1 + 3;
  uint32_t b0 = a0 ^ 0x3f803f80u, b1 = b0 + 5;
  float c[NCH][4];
  for (int i = 0; i < NCH; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NCH>
__global__ void k_tf32(float* out, long long* cyc) {
  uint32_t a0 = __float_as_uint(threadIdx.x * 1e-3f), a1 = a0 + 11, a2 = a0 + 13, a3 = a0 + 17;
  uint32_t b0 = __float_as_uint(0.5f + threadIdx.x), b1 = b0 + 3;
  float c[NCH][4];
  for (int i = 0; i < NCH; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// f32 pair -> bf16x2 hi, residual -> bf16x2 lo (the split the window would do per operand pair)
__global__ void k_split(float* out, long long* cyc) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, 0.3f * i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 hi = __float22bfloat162_rn(x[i]);
      float2 hf = __bfloat1622float2(hi);
      float2 r = make_float2(x[i].x - hf.x, x[i].y - hf.y);
      __nv_bfloat162 lo = __float22bfloat162_rn(r);
      acc ^= *reinterpret_cast<uint32_t*>(&hi) + *reinterpret_cast<uint32_t*>(&lo);
      x[i].x += 1.0f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int threads, int blocks_per_sm, double work_per_thread_iter, const char* unit) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * blocks_per_sm;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * grid * threads);
  cudaMalloc(&cyc, sizeof(long long) * grid);
  kern<<<grid, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  kern<<<grid, threads>>>(out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long* h = new long long[grid];
  cudaMemcpy(h, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  double per_sm = work_per_thread_iter * threads * blocks_per_sm * ITERS / mx;
  printf("%-28s threads=%4d x%d/SM  %8.1f %s/clk/SM  (%s)\n", name, threads, blocks_per_sm, per_sm, unit,
         cudaGetErrorString(e));
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  // per thread per iter: NCH mma; one m16n8k16 = 2048 MAC per warp = 64 MAC per thread
  run("mma bf16 m16n8k16 NCH=4", k_bf16<4>, 128, 1, 4 * 64.0, "MAC");
  run("mma bf16 m16n8k16 NCH=4", k_bf16<4>, 256, 2, 4 * 64.0, "MAC");
  run("mma bf16 m16n8k16 NCH=8", k_bf16<8>, 512, 2, 8 * 64.0, "MAC");
  run("mma bf16 m16n8k16 NCH=4", k_bf16<4>, 640, 2, 4 * 64.0, "MAC");
  // m16n8k8 tf32 = 1024 MAC per warp = 32 per thread
  run("mma tf32 m16n8k8 NCH=4", k_tf32<4>, 128, 1, 4 * 32.0, "MAC");
  run("mma tf32 m16n8k8 NCH=8", k_tf32<8>, 512, 2, 8 * 32.0, "MAC");
  run("mma tf32 m16n8k8 NCH=4", k_tf32<4>, 640, 2, 4 * 32.0, "MAC");
  // split: 8 float pairs per iter -> 16 floats
  run("bf16 hi/lo split", k_split, 512, 2, 16.0, "floats");
  return 0;
}
