// ADC window contraction on the 5th-generation tensor cores (tcgen05 / UMMA, TMA, TMEM).
//
// Every uniform ADC window of one rotation class applies the same per-sample
// factor z_s to spin s (the class's `z` plane: same interval, same gradient),
// so the samples of all those windows are ONE complex product over spins:
//
//     S[w][k] = sum_s U[w][s] z_s^k          w < W windows, k < K samples
//
// U[w][s] is the receive-weighted transverse magnetisation of spin s at the
// first sample of window w (u z when the window has no leading no-op sample),
// written by the integrator (OP_UWIN) instead of summing the samples itself.
// This replaces the reference's per-sample weighted sum (engine.py:303-305)
// for those windows; the integrator still advances every spin through the
// window with the closed-form propagator of its rotation class.
//
// The complex product is embedded as a real GEMM D = A B^T, K-dimension =
// (spin, re/im), both operands K-major:
//     A[(k, re)] = [Re z^k, -Im z^k],  A[(k, im)] = [Im z^k, Re z^k]  per spin  (M: 2 rows per sample;
//                                       an M-tile is 64 real rows then the 64 imaginary rows)
//     B[w]       = [Re U, Im U]                                        per spin  (N: windows)
// so D[(k, re)][w] = Re S, D[(k, im)][w] = Im S.  Every operand is split into
// bf16 parts x = hi + lo and the product runs as three kind::f16 passes
// (hi hi + hi lo + lo hi; ~2^-16 relative per product, fp32 accumulation in
// TMEM).  A is generated in shared memory from (pos, dw, T2) by four warps,
// B arrives by TMA (SWIZZLE_64B), one thread issues the MMAs; split-K over spin
// chunks, the chunk partials are folded in a fixed order in fp64 (the
// reference's deterministic block fold, engine.py:493-496).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "kernels.h"

namespace bloch {

struct ContractJob {
  const SpinConst* sc;  // [n] per-spin constants
  int64_t n;            // spins (contraction length)
  double T, d[3], tw;   // the group's per-sample factor: z = exp(-T r2) exp(-i (pos . d + dw tw))
  int32_t K;            // samples per window
  int32_t W;            // windows of the group
  int32_t row0;         // the group's first U row
  const uint32_t* uhi;  // U, spin-block major (contract_u_index): bf16x2 (Re, Im) words, hi part
  const uint32_t* ulo;  // lo part
  int64_t rows;         // rows (windows of every group) of the U arrays
  float* part;          // [chunks][C][K][2][Wr] partial sums per spin chunk (its accumulation segments added in fp32)
  const int64_t* out0;  // [W] complex index (coil 0) of each window's first sample in the echo array
  double* echo;         // echo array (complex128) [C][G], samples stored
  int32_t C;            // receive coils: coil c's samples are sum_s w_cs U[w][s] z_s^k (w folded into A)
  int32_t ncp;          // coil stride of w32
  const float2* w32;    // [n][ncp] fp32 coil weights (C > 1; one coil carries its weight in U)
  int64_t G;            // complex samples per coil in the echo array
  float4* zt;           // [n] scratch: per-spin (theta_hi, theta_lo, a, 0), theta = phase per sample mod 2 pi
  float2* zq;           // [n] scratch: per-spin z^2 (chirp: (theta_q lo, 0), theta_q hi in zt.w)
  int32_t chirp;        // 1: a chirp group, sample k = u r0^(k+1) q^(k(k+1)/2); (T, d, tw) describe r0 and
  double qd[3];         //    q = exp(-i pos . qd), conjugated when qconj
  int32_t qconj;
};

constexpr int kContractMaxSamples = 4096;  // windows up to this long (the fp32 phase k theta_hi is exact)

struct ContractPlan {
  int mt;          // 64-sample M-tiles per CTA (1, 2, 4)
  int nw;          // windows per N-subtile (MMA N, multiple of 16, <= 256)
  int nsub;        // N-subtiles per CTA (1 or 2): the CTA covers nsub * nw windows, one generated A tile
  int tiles_k;     // CTA tiles along the samples (all coils: C x tiles per coil)
  int tpc;         // CTA sample tiles per coil
  int tiles_w;     // CTA tiles along the windows
  int chunks;      // split-K chunks along the spins
  int stages;      // 16-spin stages per chunk
  int depth;       // shared-memory pipeline depth
  int smem;        // dynamic shared memory bytes
  int tmem_cols;   // TMEM columns allocated (power of two >= mt * nw)
  int seg;         // stages per accumulation segment: the accumulator is drained into its own
                   // partial slot every `seg` stages (the tensor core's fp32 accumulation truncates
                   // at every MMA, so a long accumulation drifts; measured 2.9e-4 rel over 15.6k MMAs)
  int segs;        // segments per chunk (partial slots per chunk)
  int dbg;         // experiment hook: 1 = skip A generation stores, 2 = skip MMAs
};

ContractPlan contract_plan(int K, int W, int64_t n, int n_sm, int C = 1);
size_t contract_part_bytes(const ContractPlan& p, const ContractJob& j);
// the GEMM (partials) and the fold into the echo array, on `st`
cudaError_t launch_contract(const ContractJob& j, const ContractPlan& p, cudaStream_t st);

// U word of (row r, spin i): blocks of 16 spins, each [rows][16] words (64 B per row), so the 16-spin
// stage tile of any run of rows is one contiguous piece (one TMA box, full-line DRAM bursts)
__host__ __device__ inline int64_t contract_u_index(int64_t rows, int64_t r, int64_t i) {
  return ((i >> 4) * rows + r) * 16 + (i & 15);
}
inline int64_t contract_u_words(int64_t rows, int64_t n) { return ((n + 15) / 16) * rows * 16; }

// bf16 (round to nearest even) of a float, as the high half of a 32-bit word
__host__ __device__ inline uint32_t bf16_rn_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
}
// U word pair of an fp32 complex value: hi = bf16x2 (Re, Im) rounded, lo = bf16x2 of the residuals (the
// integrator's path: no fp64 <-> fp32 conversions beyond the state's own)
__host__ __device__ inline void contract_split_f(float re, float im, uint32_t& hi, uint32_t& lo) {
  const uint32_t hr = bf16_rn_bits(re), hm = bf16_rn_bits(im);
  float fr, fm;
  memcpy(&fr, &hr, 4);
  memcpy(&fm, &hm, 4);
  const uint32_t lr = bf16_rn_bits(re - fr), lm = bf16_rn_bits(im - fm);  // exact residuals
  hi = (hr >> 16) | hm;
  lo = (lr >> 16) | lm;
}
// U word pair of a complex value: hi = bf16x2 (Re, Im) rounded, lo = bf16x2 of the residuals
__host__ __device__ inline void contract_split(double re, double im, uint32_t& hi, uint32_t& lo) {
  const uint32_t hr = bf16_rn_bits(static_cast<float>(re)), hm = bf16_rn_bits(static_cast<float>(im));
  float fr, fm;
  memcpy(&fr, &hr, 4);
  memcpy(&fm, &hm, 4);
  const uint32_t lr = bf16_rn_bits(static_cast<float>(re - static_cast<double>(fr)));
  const uint32_t lm = bf16_rn_bits(static_cast<float>(im - static_cast<double>(fm)));
  hi = (hr >> 16) | hm;
  lo = (lr >> 16) | lm;
}

}  // namespace bloch
