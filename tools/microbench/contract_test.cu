// Standalone check + timing of the tcgen05 window contraction (paper_1305_6861_b200/csrc/contract_kernels.cu):
//   S[w][k] = sum_s U[w][s] z_s^k,  z_s = exp(-T r2_s) exp(-i (pos_s . d + dw_s tw))
// against an fp64 host sum on sampled (w, k) entries.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1305_6861_b200/csrc \
//        tools/microbench/contract_test.cu -o tools/microbench/contract_test
//   contract_test W K n [row0] [extra_rows]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cmath>
#include <complex>
#include <random>
#include <vector>

#include "../../paper_1305_6861_b200/csrc/contract_kernels.cu"

using namespace bloch;

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 256, K = argc > 2 ? atoi(argv[2]) : 256;
  const int64_t n = argc > 3 ? atoll(argv[3]) : 4096;
  const int row0 = argc > 4 ? atoi(argv[4]) : 0, extra = argc > 5 ? atoi(argv[5]) : 0;
  const int64_t rows = row0 + W + extra;
  std::mt19937_64 rng(1234);
  std::uniform_real_distribution<double> U01(0.0, 1.0);
  std::normal_distribution<double> N01(0.0, 1.0);
  std::vector<SpinConst> sc(n);
  for (int64_t i = 0; i < n; ++i) {
    sc[i].x = (U01(rng) - 0.5) * 0.25;
    sc[i].y = (U01(rng) - 0.5) * 0.25;
    sc[i].z = 0.0;
    sc[i].dw = 2 * M_PI * 20.0 * N01(rng);
    sc[i].m0 = 1.0;
    sc[i].r1 = 1.0 / 0.8;
    sc[i].r2 = 1.0 / (0.04 + 0.16 * U01(rng));
    sc[i].pad = 0.0;
  }
  const double T = 1e-5, d0 = 2 * M_PI / 0.25 * 1.0, d1 = 0.3, tw = 1e-5;
  std::vector<std::complex<double>> U(static_cast<size_t>(W) * n);
  std::vector<uint32_t> hi(contract_u_words(rows, n), 0u), lo(contract_u_words(rows, n), 0u);
  for (int w = 0; w < W; ++w)
    for (int64_t i = 0; i < n; ++i) {
      // a coherent part (k-space centre) plus a random one
      const std::complex<double> u = std::polar(0.6 * U01(rng), 0.3 * w) + std::polar(0.4 * U01(rng), 6.283 * U01(rng));
      U[static_cast<size_t>(w) * n + i] = u;
      const int64_t q = contract_u_index(rows, row0 + w, i);
      contract_split(u.real(), u.imag(), hi[q], lo[q]);
    }
  SpinConst* d_sc;
  uint32_t *d_hi, *d_lo;
  int64_t* d_out0;
  double* d_echo;
  float* d_part;
  cudaMalloc(&d_sc, n * sizeof(SpinConst));
  cudaMalloc(&d_hi, hi.size() * 4);
  cudaMalloc(&d_lo, lo.size() * 4);
  cudaMemcpy(d_sc, sc.data(), n * sizeof(SpinConst), cudaMemcpyHostToDevice);
  cudaMemcpy(d_hi, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_lo, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice);
  std::vector<int64_t> out0(W);
  for (int w = 0; w < W; ++w) out0[w] = static_cast<int64_t>(w) * K;
  cudaMalloc(&d_out0, W * 8);
  cudaMemcpy(d_out0, out0.data(), W * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&d_echo, static_cast<size_t>(W) * K * 16);
  cudaMemset(d_echo, 0, static_cast<size_t>(W) * K * 16);
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  ContractJob j{};
  j.sc = d_sc;
  j.n = n;
  j.T = T;
  j.d[0] = d0;
  j.d[1] = d1;
  j.d[2] = 0.0;
  j.tw = tw;
  j.K = K;
  j.W = W;
  j.row0 = row0;
  j.uhi = d_hi;
  j.ulo = d_lo;
  j.rows = rows;
  j.out0 = d_out0;
  j.echo = d_echo;
  j.C = 1;
  j.chirp = 0;
  j.ncp = 1;
  j.w32 = nullptr;
  j.G = static_cast<int64_t>(W) * K;
  cudaMalloc(&j.zt, n * sizeof(float4));
  cudaMalloc(&j.zq, n * sizeof(float2));
  ContractPlan p = contract_plan(K, W, n, n_sm);
  if (getenv("CONTRACT_DBG")) p.dbg = atoi(getenv("CONTRACT_DBG"));
  cudaMalloc(&d_part, contract_part_bytes(p, j));
  j.part = d_part;
  printf("W=%d K=%d n=%lld row0=%d: mt=%d nw=%d tiles %dx%d chunks=%d stages=%d seg=%d segs=%d depth=%d smem=%d tmem=%d grid=%d dbg=%d\n", W,
         K, (long long)n, row0, p.mt, p.nw, p.tiles_k, p.tiles_w, p.chunks, p.stages, p.seg, p.segs, p.depth, p.smem, p.tmem_cols,
         p.tiles_k * p.tiles_w * p.chunks, p.dbg);
  cudaError_t e = launch_contract(j, p, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<double> echo(static_cast<size_t>(W) * K * 2);
  cudaMemcpy(echo.data(), d_echo, echo.size() * 8, cudaMemcpyDeviceToHost);
  // fp64 host reference on sampled entries (all of them when small)
  const int64_t total = static_cast<int64_t>(W) * K;
  const int64_t want = total * n <= 400000000LL ? total : std::max<int64_t>(64, 400000000LL / n);
  double num = 0.0, den = 0.0, maxrel = 0.0;
  std::mt19937_64 pick(99);
  for (int64_t c = 0; c < want; ++c) {
    const int64_t t = want == total ? c : static_cast<int64_t>(pick() % total);
    const int w = static_cast<int>(t / K), k = static_cast<int>(t % K);
    std::complex<double> acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double th = sc[i].z * 0.0 + std::fma(sc[i].y, d1, sc[i].x * d0) + sc[i].dw * tw;
      const std::complex<double> zk = std::polar(std::exp(-k * T * sc[i].r2), -k * th);
      acc += U[static_cast<size_t>(w) * n + i] * zk;
    }
    const std::complex<double> g(echo[2 * t], echo[2 * t + 1]);
    num += std::norm(g - acc);
    den += std::norm(acc);
    maxrel = std::max(maxrel, std::abs(g - acc) / std::max(1e-300, std::abs(acc)));
  }
  printf("rel L2 error vs fp64 (%lld entries): %.3e  (max rel %.2e)\n", (long long)want, std::sqrt(num / den), maxrel);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  const int reps = 5;
  cudaEventRecord(t0);
  for (int r = 0; r < reps; ++r) launch_contract(j, p, 0);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  ms /= reps;
  const double macs = 3.0 * 4.0 * static_cast<double>(W) * K * n;  // 3 bf16 passes x 4 real MAC per complex term
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("contract: %.3f ms  %.1f TMAC/s bf16  (%.0f MAC/clk/SM at %.0f MHz; floor %.3f ms at 4096 MAC/clk/SM)\n", ms,
         macs / ms * 1e-9, macs / (ms * 1e-3) / n_sm / (clk_khz * 1e3), clk_khz / 1e3,
         macs / (4096.0 * n_sm * clk_khz * 1e3) * 1e3);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
