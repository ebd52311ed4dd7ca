// Kernel parameter block, compile-time variants and host launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "program.h"

namespace bloch {

constexpr int kMaxDevices = 64;  // per-device launch state (shared-memory opt-in) is kept for this many

// per-spin constants, one 64-byte record (4 x 16-byte loads)
struct alignas(16) SpinConst {
  double x, y, z, dw;  // position (m), off-resonance (rad/s)
  double m0, r1, r2;   // equilibrium magnetisation, 1/T1, 1/T2
  double pad;
};

struct KParams {
  const DevOp* ops;
  int32_t n_ops;
  int32_t spins_per_cta;  // S * blockDim.x
  const GEv* gev;
  const double* mats;            // OP_RFTRAIN matrices, 9 per pair
  int64_t n;                     // spins
  const SpinConst* sc;           // [n]
  const double *mx0, *my0, *mz0; // initial state (SpinBlock.mx/my/mz, or the previous segment's state)
  double *mx1, *my1, *mz1;       // state at the end of this launch's op range, or nullptr
  int32_t op_begin;              // this launch runs ops [op_begin, n_ops): a program segment
  int32_t sample_base;           // compact index of the segment's first sample (partial rows start there)
  const double* w;               // [NC][n][2] complex weights, or nullptr = 1+0j
  void* partial;                 // [warps of the grid][part_stride] of R
  int64_t part_stride;           // n_samples * NC * 2
  double* snaps;                 // [n_snap][n][3] or nullptr
  const double* relax;           // [n_relax][n][2]: exp(-T_c/T1_i), exp(-T_c/T2_i)
  double2* planes;               // [n_planes][n]: class quantities (plane_kernel); progression running
                                 // factors are updated in place, every other plane is read-only
  const float2* planes32;        // fp32 mode: [n_planes][n] float2 copies of the PL_SAMPLE planes (same ids)
  const double* train;           // [n_train][n][12]: train-class affine propagators (train_table_kernel)
  const float2* w32;             // fp32 multi-coil weights, spin-major [n][NC] (tensor-core windows), or nullptr
  uint32_t* uhi;                 // OP_UWIN: U of bf16x2 (Re, Im) words, hi part (contract.h, contract_u_index)
  uint32_t* ulo;                 //          lo part
  int64_t urows;                 //          U rows
  int32_t n_mats_smem;           // pulse matrices staged in shared memory by the register-state kernels (0: read
                                 // from global); the fused pulses of a program, when they fit kMatsSmemMax
  int32_t n_prog_smem;           // progression classes whose running factors the register-state kernels keep in
                                 // shared memory for the whole launch (0: read-modify-write through L2)
  int32_t prog_plane[32];        // running-factor plane of each progression class
};
constexpr int kMatsSmemMax = 640;  // 45 KB of fp64 3x3 matrices

// Launch shape per variant: max threads per CTA and min resident CTAs per SM
// (registers per thread <= 64K / (kMaxThreads * kMinBlocks)).
template <typename R, int S, int NC>
struct KernelTraits {
  static constexpr int kMaxThreads = 512;
  static constexpr int kMinBlocks = 1;
  static constexpr int kMinBlocksNoWin = 1;  // the variant without window code (every window deferred)
  static constexpr int kMaxThreadsNoWin = 512;
};
#ifndef BLOCH_NOWIN_MINB
#define BLOCH_NOWIN_MINB 2
#endif
template <>
struct KernelTraits<float, 8, 1> {  // the fp32 single-coil workhorse: 2 CTAs x 10 warps per SM
  static constexpr int kMaxThreads = 320;   // measured: 1 x 16 warps 17.6 ms, 2 x 10 warps 14.1 ms,
  static constexpr int kMinBlocks = 2;      // 3 x 8 warps (80 regs, spills) 15.5 ms on config 1
  static constexpr int kMinBlocksNoWin = BLOCH_NOWIN_MINB;
  static constexpr int kMaxThreadsNoWin = 320;
};

// (real type, spins per thread, coils) instantiated in bloch_kernels.cu
#define BLOCH_FOR_EACH_VARIANT(X) \
  X(float, 8, 1)                  \
  X(float, 4, 1)                  \
  X(float, 2, 1)                  \
  X(float, 1, 1)                  \
  X(float, 4, 2)                  \
  X(float, 4, 4)                  \
  X(float, 4, 8)                  \
  X(float, 2, 8)                  \
  X(float, 1, 8)                  \
  X(double, 4, 1)                 \
  X(double, 1, 1)                 \
  X(double, 2, 2)                 \
  X(double, 2, 4)                 \
  X(double, 1, 8)

template <>
struct KernelTraits<float, 4, 1> {  // long windows (>= 384 samples): 2 CTAs x 12 warps, 4 spins per thread
  static constexpr int kMaxThreads = 384;
  static constexpr int kMinBlocks = 2;
  static constexpr int kMinBlocksNoWin = BLOCH_NOWIN_MINB;
  static constexpr int kMaxThreadsNoWin = 320;  // register state: 102 registers, no spills (384: 80, spilling)
};

template <>
struct KernelTraits<float, 1, 1> {  // small blocks (spin shards): one spin per thread, 2 CTAs x 10 warps
  static constexpr int kMaxThreads = 320;
  static constexpr int kMinBlocks = 2;
  static constexpr int kMinBlocksNoWin = BLOCH_NOWIN_MINB;
  static constexpr int kMaxThreadsNoWin = 320;
};

template <>
struct KernelTraits<float, 1, 8> {  // small eight-coil blocks: one spin per thread
  static constexpr int kMaxThreads = 320;
  static constexpr int kMinBlocks = 2;
  static constexpr int kMinBlocksNoWin = BLOCH_NOWIN_MINB;
  static constexpr int kMaxThreadsNoWin = 320;
};

template <typename R, int S, int NC>
cudaError_t launch_integrate(const KParams& kp, int grid, int threads, cudaStream_t stream, bool full, bool win);
template <typename R, int S, int NC>
cudaError_t kernel_attrs(int* max_threads, int* regs);
template <typename R, int S, int NC>
size_t integrate_smem_bytes(int threads, bool win);
cudaError_t launch_prep(int64_t n, const double* pos, const double* dw, const double* m0, const double* t1,
                        const double* t2, SpinConst* sc, cudaStream_t stream);
cudaError_t launch_relax_table(int64_t n, int n_cls, const double* T, const SpinConst* sc, double* out,
                               cudaStream_t stream);
cudaError_t launch_planes(int64_t n, int n_planes, const PlaneDesc* pd, const SpinConst* sc, const double* w1,
                          double* out, float2* out32, cudaStream_t stream);
cudaError_t launch_train_table(int64_t n, int n_cls, const TrainClass* tc, const double* mats, const SpinConst* sc,
                               double* out, cudaStream_t stream);
cudaError_t launch_pad_weights(int64_t n, int nc, int ncp, const double* w, double* out,
                               cudaStream_t stream);
cudaError_t launch_weights_f32(int64_t n, int ncp, const double* w, float2* out, cudaStream_t stream);
// out[t] = sum_r rows[r * len + t] in rank order (fp64): the device-set context's one reduction
cudaError_t launch_sum_rows(const double* rows, int n_rows, int64_t len, double* out, cudaStream_t stream);
template <typename R>
cudaError_t launch_reduce(const R* part, int rows, int64_t row_stride, int64_t n_slots, int nc, int ncp,
                          const int64_t* sample_g, int64_t G, double* out, cudaStream_t stream);

}  // namespace bloch
