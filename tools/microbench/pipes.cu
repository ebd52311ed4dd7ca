// Pipe-throughput microbenchmark for the Bloch integrator design (sm_100a).
// Measures per-SM-per-clock throughput of the instruction mixes the kernel
// relies on: FFMA (3 distinct regs), FFMA2 / FMUL2 / FADD2 (packed f32x2),
// MUFU sin/cos/ex2, DFMA, SHFL.  Each thread runs NCH independent chains so
// the result is throughput, not latency.  Cycles come from clock64() per CTA.
#include <cstdio>
#include <cuda_runtime.h>

#define NCH 8
#define ITERS 4096

__global__ void k_ffma(float* out, float a, float b, long long* cyc) {
  float x[NCH];
  for (int i = 0; i < NCH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  float c = a * threadIdx.x;  // per-thread register operand (no immediate)
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) x[i] = fmaf(x[i], b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, float a, float b, long long* cyc) {
  float2 x[NCH];
  for (int i = 0; i < NCH; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 bb = make_float2(b, b * 0.5f);
  float2 c = make_float2(a * threadIdx.x, a);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) x[i] = __ffma2_rn(x[i], bb, c);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// complex multiply of NCH/2 spin pairs, packed: the kernel's window inner loop
__global__ void k_cmul2(float* out, float a, float b, long long* cyc) {
  float2 X[NCH / 2], Y[NCH / 2], C[NCH / 2], D[NCH / 2], ND[NCH / 2];
  for (int i = 0; i < NCH / 2; ++i) {
    X[i] = make_float2(1.f, 0.5f); Y[i] = make_float2(0.f, 0.1f);
    float ang = a * (threadIdx.x + i);
    C[i] = make_float2(cosf(ang) * b, cosf(ang + 1) * b);
    D[i] = make_float2(sinf(ang) * b, sinf(ang + 1) * b);
    ND[i] = make_float2(-D[i].x, -D[i].y);
  }
  float2 acx = make_float2(0, 0), acy = make_float2(0, 0);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH / 2; ++i) {
      float2 t1 = __fmul2_rn(Y[i], ND[i]);
      float2 t2 = __fmul2_rn(Y[i], C[i]);
      X[i] = __ffma2_rn(X[i], C[i], t1);
      Y[i] = __ffma2_rn(X[i], D[i], t2);
      acx = __fadd2_rn(acx, X[i]);
      acy = __fadd2_rn(acy, Y[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acx.x + acx.y + acy.x + acy.y;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// same complex multiply, scalar FFMA/FMUL
__global__ void k_cmul1(float* out, float a, float b, long long* cyc) {
  float X[NCH], Y[NCH], C[NCH], D[NCH];
  for (int i = 0; i < NCH; ++i) {
    X[i] = 1.f; Y[i] = 0.f;
    float ang = a * (threadIdx.x + i);
    C[i] = cosf(ang) * b; D[i] = sinf(ang) * b;
  }
  float acx = 0, acy = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      float xn = fmaf(X[i], C[i], Y[i] * D[i]);
      float yn = fmaf(-X[i], D[i], Y[i] * C[i]);
      X[i] = xn; Y[i] = yn;
      acx += xn; acy += yn;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acx + acy;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_mufu_sin(float* out, float a, float b, long long* cyc) {
  float x[NCH];
  for (int i = 0; i < NCH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) x[i] = __sinf(x[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_mufu_ex2(float* out, float a, float b, long long* cyc) {
  float x[NCH];
  for (int i = 0; i < NCH; ++i) x[i] = -(threadIdx.x * 1e-3f + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) x[i] = exp2f(x[i]) - 1.0f;  // ex2.approx + fadd
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(float* out, float a, float b, long long* cyc) {
  double x[NCH];
  for (int i = 0; i < NCH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  double c = (double)a * threadIdx.x, bb = b;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) x[i] = fma(x[i], bb, c);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < NCH; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_shfl(float* out, float a, float b, long long* cyc) {
  float x[NCH];
  for (int i = 0; i < NCH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 << (i & 3));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kern_t)(float*, float, float, long long*);

static void run(const char* name, kern_t k, int ops_per_iter_per_thread, int threads) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks = nsm;  // one CTA per SM
  float* out; long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  k<<<blocks, threads>>>(out, 1e-4f, 0.9999f, cyc);  // warm
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, 1e-4f, 0.9999f, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
  double ops = (double)ops_per_iter_per_thread * ITERS * threads;  // per SM
  printf("%-10s thr=%4d  ops/clk/SM=%7.2f  time=%.3f ms  eff_clk=%.0f MHz  %s\n", name, threads,
         ops / mean, ms, mean / (ms * 1e3), cudaGetErrorString(err));
  delete[] h; cudaFree(out); cudaFree(cyc);
}

int main() {
  int threads_list[2] = {512, 1024};
  for (int t : threads_list) {
    run("ffma", k_ffma, NCH, t);
    run("ffma2(x2)", k_ffma2, 2 * NCH, t);
    run("cmul1", k_cmul1, NCH, t);   // counts spin-samples (complex mul + acc)
    run("cmul2", k_cmul2, NCH, t);   // counts spin-samples
    run("sin", k_mufu_sin, NCH, t);
    run("ex2+fadd", k_mufu_ex2, NCH, t);
    run("dfma", k_dfma, NCH, t);
    run("shfl", k_shfl, NCH, t);
  }
  return 0;
}
