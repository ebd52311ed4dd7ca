// Standalone test of the window contraction as a tcgen05 GEMM:
//   S[w][k] = sum_s U[w][s] z_s^k,  w < R windows, k < NS samples, s < n spins
// A = U (K-major: row w, K = (s, re/im)), pre-split hi/lo tf32, by cp.async;
// B = Z real-embedded (row (k, re) = [Re z^k, -Im z^k], row (k, im) = [Im z^k, Re z^k]) generated in
// shared memory per stage; 3 tf32 passes (hh, hl, lh) into TMEM; split-K partials reduced on the host.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <vector>
#include <complex>

#include "wgemm.cuh"

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 256, NS = argc > 2 ? atoi(argv[2]) : 256;
  const int n = argc > 3 ? atoi(argv[3]) : 4096, check = argc > 4 ? atoi(argv[4]) : 1;
  const int npad = (n + 7) / 8 * 8;
  std::vector<float> Uhi((size_t)R * 2 * npad, 0.f), Ulo((size_t)R * 2 * npad, 0.f);
  std::vector<std::complex<double>> U((size_t)R * n), Z(n);
  srand(7);
  auto rnd = [] { return rand() / (double)RAND_MAX; };
  for (int s = 0; s < n; ++s) Z[s] = std::polar(0.999 - 0.002 * rnd(), 6.283 * rnd() * 0.05);
  for (int w = 0; w < R; ++w)
    for (int s = 0; s < n; ++s) {
      const std::complex<double> u = std::polar(rnd(), 6.283 * rnd());
      const float ur = (float)u.real(), ui = (float)u.imag();
      U[(size_t)w * n + s] = {ur, ui};
      auto split = [](float x, float& h, float& l) { uint32_t b; memcpy(&b, &x, 4); b &= 0xffffe000u; memcpy(&h, &b, 4); l = x - h; };
      split(ur, Uhi[(size_t)w * 2 * npad + 2 * s], Ulo[(size_t)w * 2 * npad + 2 * s]);
      split(ui, Uhi[(size_t)w * 2 * npad + 2 * s + 1], Ulo[(size_t)w * 2 * npad + 2 * s + 1]);
    }
  std::vector<float2> z32(npad, make_float2(0.f, 0.f));
  for (int s = 0; s < n; ++s) z32[s] = make_float2((float)Z[s].real(), (float)Z[s].imag());
  float *dUh, *dUl;
  float2 *dz, *dP;
  cudaMalloc(&dUh, Uhi.size() * 4);
  cudaMalloc(&dUl, Ulo.size() * 4);
  cudaMalloc(&dz, npad * 8);
  cudaMemcpy(dUh, Uhi.data(), Uhi.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dUl, Ulo.data(), Ulo.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dz, z32.data(), npad * 8, cudaMemcpyHostToDevice);
  bloch::WGemmShape sh = bloch::wgemm_shape(R, NS, npad, 148);
  printf("R=%d NS=%d n=%d: m_tiles=%d n_tile=%d n_tiles=%d k_chunks=%d stages/chunk=%d na=%d smem=%d\n", R, NS, n, sh.m_tiles,
         sh.n_tile, sh.n_tiles, sh.k_chunks, sh.stages_per_chunk, sh.na, sh.smem);
  cudaMalloc(&dP, (size_t)sh.k_chunks * R * NS * 8);
  bloch::WGemmArgs a{dUh, dUl, dz, R, NS, npad, 2 * npad, dP};
  cudaError_t e = bloch::launch_wgemm(a, sh, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  for (int i = 0; i < 5; ++i) bloch::launch_wgemm(a, sh, 0);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  ms /= 5;
  const double macs = 3.0 * 4.0 * R * (double)NS * n;
  printf("wgemm: %.3f ms, %.1f TMAC/s (3 tf32 passes x 4 real MAC per complex term), %.1f MAC/clk/SM @1.965GHz\n", ms,
         macs / ms / 1e9, macs / (ms * 1e-3) / 148 / 1.965e9);
  if (!check) return 0;
  std::vector<float2> P((size_t)sh.k_chunks * R * NS);
  cudaMemcpy(P.data(), dP, P.size() * 8, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int w = 0; w < R; w += (R > 64 ? 7 : 1))
    for (int k = 0; k < NS; ++k) {
      std::complex<double> ref = 0, got = 0;
      for (int s = 0; s < n; ++s) ref += U[(size_t)w * n + s] * std::pow(Z[s], k);
      for (int c = 0; c < sh.k_chunks; ++c) {
        const float2 p = P[((size_t)c * R + w) * NS + k];
        got += std::complex<double>(p.x, p.y);
      }
      num += std::norm(ref - got);
      den += std::norm(ref);
    }
  printf("rel L2 error vs fp64 host: %.3e\n", sqrt(num / den));
  return 0;
}
