// Device-side object model: lattice rasterisation + per-spin fold, straight
// into the SoA the integrator reads.
//
// Reference semantics (restated, see include/bloch_b200.h):
//   phantom._lattice / rasterize   phantom.py:91-142   site order box, z, y, x (x fastest); M0 == 0 -> no spin
//   build_spin_arrays              engine.py:192-226   mx = my = 0, mz = M0; domega; receive weight
//   complex_weight                 system.py:203-211   w = Sx - i Sy
//
// Three passes over the lattice sites (a few M at most, HBM-trivial next to
// the integrator): (1) label each site and flag the emitted ones, (2) an
// order-preserving exclusive scan of the flags (CUB), (3) emit each kept
// spin at its scanned index.  All fp64 arithmetic that the host computes
// with numpy is written with explicit _rn intrinsics so no FMA contraction
// changes the rounding: lattice coordinates and ellipse labels (hence M0,
// T1, T2 and the spin order) are bit-identical to the host rasteriser.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cub/device/device_scan.cuh>

#include "../../include/bloch_b200.h"
#include "raster.h"

namespace bloch {
namespace {

constexpr int kRasterThreads = 256;
constexpr int kMaxBoxes = kMaxRasterBoxes;

struct BoxTable {
  bloch_box_t box[kMaxBoxes];
  int64_t first_site[kMaxBoxes + 1];
  int32_t n_boxes;
};

__device__ __forceinline__ int find_box(const BoxTable& bt, int64_t g) {
  int b = 0;
  while (b + 1 < bt.n_boxes && g >= bt.first_site[b + 1]) ++b;
  return b;
}

__device__ __forceinline__ void site_coords(const bloch_box_t& bx, int64_t local, double* x, double* y, double* z) {
  const int64_t nx = bx.count[0], ny = bx.count[1];
  const int64_t ix = local % nx;
  const int64_t t = local / nx;
  const int64_t iy = t % ny;
  const int64_t iz = t / ny;
  // numpy: (origin + offset) + spacing * arange(n); base holds origin + offset
  *x = __dadd_rn(bx.base[0], __dmul_rn(bx.step[0], (double)ix));
  *y = __dadd_rn(bx.base[1], __dmul_rn(bx.step[1], (double)iy));
  *z = __dadd_rn(bx.base[2], __dmul_rn(bx.step[2], (double)iz));
}

// last shape containing the site, or -1 (label map: later shapes override)
__device__ __forceinline__ int site_label(const bloch_box_t& bx, const bloch_shape_t* __restrict__ shapes, double x,
                                          double y, double z) {
  int lab = -1;
  for (int k = 0; k < bx.shape_count; ++k) {
    const bloch_shape_t& s = shapes[bx.shape_begin + k];
    const double dx = __dsub_rn(x, s.c[0]), dy = __dsub_rn(y, s.c[1]);
    const double u = __ddiv_rn(__dadd_rn(__dmul_rn(dx, s.cos_a), __dmul_rn(dy, s.sin_a)), s.ax[0]);
    const double v = __ddiv_rn(__dadd_rn(__dmul_rn(-dx, s.sin_a), __dmul_rn(dy, s.cos_a)), s.ax[1]);
    double r = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    if (s.ax[2] > 0.0) {
      const double w = __ddiv_rn(__dsub_rn(z, s.c[2]), s.ax[2]);
      r = __dadd_rn(r, __dmul_rn(w, w));
    }
    if (r <= 1.0) lab = k;
  }
  return lab;
}

__global__ void __launch_bounds__(kRasterThreads) label_kernel(const BoxTable* __restrict__ bt_g,
                                                               const bloch_shape_t* __restrict__ shapes,
                                                               int64_t n_sites, int32_t* __restrict__ label,
                                                               uint32_t* __restrict__ keep) {
  __shared__ BoxTable bt;
  for (int i = threadIdx.x; i < (int)(sizeof(BoxTable) / 8); i += blockDim.x)
    reinterpret_cast<int64_t*>(&bt)[i] = reinterpret_cast<const int64_t*>(bt_g)[i];
  __syncthreads();
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_sites;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int b = find_box(bt, g);
    const bloch_box_t& bx = bt.box[b];
    double x, y, z;
    site_coords(bx, g - bt.first_site[b], &x, &y, &z);
    const int lab = site_label(bx, shapes, x, y, z);
    const double m0 = lab >= 0 ? shapes[bx.shape_begin + lab].m0 : bx.m0;
    label[g] = lab;
    keep[g] = m0 != 0.0 ? 1u : 0u;
  }
}

struct FieldDev {
  double const_dw, poly_len, poly_scale;
  int32_t n_poly, n_bumps, peak_mode;
  double poly[4 * kMaxPoly];
  double bumps[5 * kMaxBumps];
};

struct CoilDev {
  bloch_coil_t coil[kMaxCoils];
  int32_t n_coils;
  double uniform_s;
};

__device__ __forceinline__ double ipow(double b, int e) {
  double r = 1.0;
  for (int i = 0; i < e; ++i) r = __dmul_rn(r, b);
  return r;
}

__global__ void __launch_bounds__(kRasterThreads) emit_kernel(
    const BoxTable* __restrict__ bt_g, const bloch_shape_t* __restrict__ shapes, const FieldDev* __restrict__ fd,
    const CoilDev* __restrict__ cd, int64_t n_sites, const int32_t* __restrict__ label,
    const uint32_t* __restrict__ keep, const uint32_t* __restrict__ slot, int64_t n_out, RasterOut out,
    double* __restrict__ poly_raw, unsigned long long* __restrict__ poly_absmax, int* __restrict__ bad) {
  __shared__ BoxTable bt;
  for (int i = threadIdx.x; i < (int)(sizeof(BoxTable) / 8); i += blockDim.x)
    reinterpret_cast<int64_t*>(&bt)[i] = reinterpret_cast<const int64_t*>(bt_g)[i];
  __syncthreads();
  unsigned long long local_max = 0ull;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_sites;
       g += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[g]) continue;
    const int64_t i = slot[g];
    const int b = find_box(bt, g);
    const bloch_box_t& bx = bt.box[b];
    double x, y, z;
    site_coords(bx, g - bt.first_site[b], &x, &y, &z);
    const int lab = label[g];
    const bloch_shape_t* sh = lab >= 0 ? &shapes[bx.shape_begin + lab] : nullptr;
    const double m0 = sh ? sh->m0 : bx.m0;
    const double t1 = sh ? sh->t1 : bx.t1;
    const double t2 = sh ? sh->t2 : bx.t2;
    if (!(m0 >= 0.0) || !(t1 > 0.0) || !(t2 > 0.0)) atomicOr(bad, 1);
    out.pos[3 * i + 0] = x;
    out.pos[3 * i + 1] = y;
    out.pos[3 * i + 2] = z;
    out.mx[i] = 0.0;
    out.my[i] = 0.0;
    out.mz[i] = m0;
    out.m0[i] = m0;
    out.t1[i] = t1;
    out.t2[i] = t2;
    // off-resonance: tissue + constant + polynomial + bumps, summed in that order
    double dw = __dadd_rn(sh ? sh->dw : bx.dw, fd->const_dw);
    if (fd->n_poly > 0) {
      const double len = fd->poly_len;
      const double u = __ddiv_rn(x, len), v = __ddiv_rn(y, len), w = __ddiv_rn(z, len);
      double p = 0.0;
      for (int k = 0; k < fd->n_poly; ++k) {
        const double* c = &fd->poly[4 * k];
        const double t = __dmul_rn(__dmul_rn(ipow(u, (int)c[1]), ipow(v, (int)c[2])), ipow(w, (int)c[3]));
        p = __dadd_rn(p, __dmul_rn(c[0], t));
      }
      if (fd->peak_mode) {
        poly_raw[i] = p;
        const unsigned long long a = __double_as_longlong(fabs(p));  // ordered like the value for p >= 0
        local_max = a > local_max ? a : local_max;
      } else {
        dw = __dadd_rn(dw, __dmul_rn(p, fd->poly_scale));
      }
    }
    for (int k = 0; k < fd->n_bumps; ++k) {
      const double* bp = &fd->bumps[5 * k];
      const double ex = __dsub_rn(x, bp[0]), ey = __dsub_rn(y, bp[1]);
      double d2 = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
      if (bp[2] == bp[2]) {  // not NaN: 3-D bump
        const double ez = __dsub_rn(z, bp[2]);
        d2 = __dadd_rn(d2, __dmul_rn(ez, ez));
      }
      const double den = __dmul_rn(2.0, __dmul_rn(bp[3], bp[3]));
      dw = __dadd_rn(dw, __dmul_rn(bp[4], exp(__ddiv_rn(-d2, den))));
    }
    out.domega[i] = dw;
    // receive weights [coil][spin], stride n_out
    if (cd->n_coils == 0) {
      out.weight[2 * i + 0] = cd->uniform_s;
      out.weight[2 * i + 1] = 0.0;
    } else {
      for (int c = 0; c < cd->n_coils; ++c) {
        const bloch_coil_t& co = cd->coil[c];
        const double ex = __dsub_rn(x, co.c[0]), ey = __dsub_rn(y, co.c[1]), ez = __dsub_rn(z, co.c[2]);
        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
        const double mag = exp(__ddiv_rn(-d2, __dmul_rn(2.0, __dmul_rn(co.sigma, co.sigma))));
        out.weight[2 * (c * n_out + i) + 0] = __dmul_rn(mag, co.cos_p);
        out.weight[2 * (c * n_out + i) + 1] = -__dmul_rn(mag, co.sin_p);
      }
    }
  }
  if (fd->peak_mode && fd->n_poly > 0) {
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, local_max, o);
      local_max = v > local_max ? v : local_max;
    }
    if ((threadIdx.x & 31) == 0 && local_max) atomicMax(poly_absmax, local_max);
  }
}

// polynomial peak normalisation: dw += p * (peak / max(max|p|, 1e-30))
__global__ void peak_kernel(int64_t n, const double* __restrict__ poly_raw,
                            const unsigned long long* __restrict__ poly_absmax, double peak,
                            double* __restrict__ domega) {
  const double m = __longlong_as_double((long long)*poly_absmax);
  const double scale = __ddiv_rn(peak, m > 1e-30 ? m : 1e-30);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    domega[i] = __dadd_rn(domega[i], __dmul_rn(poly_raw[i], scale));
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

size_t raster_staging_bytes() {
  return align256(sizeof(BoxTable)) + align256(sizeof(FieldDev)) + align256(sizeof(CoilDev));
}

size_t raster_scratch_bytes(int64_t n_sites) {
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)(n_sites > 0 ? n_sites : 1));
  return align256(sizeof(BoxTable)) + align256(sizeof(FieldDev)) + align256(sizeof(CoilDev)) +
         align256(sizeof(bloch_shape_t) * kMaxShapes) + 3 * align256(4 * (size_t)(n_sites + 1)) +
         align256(8 * (size_t)(n_sites + 1)) + align256(64) + align256(cub_bytes);
}

cudaError_t raster_run(const RasterArgs& a, void* scratch, size_t scratch_bytes, void* host_staging,
                       int n_sm, cudaStream_t st, int64_t* n_out, int* bad_out) {
  // host staging (pinned or pageable) for the small descriptor tables
  auto* bt = static_cast<BoxTable*>(host_staging);
  auto* fd = reinterpret_cast<FieldDev*>(static_cast<char*>(host_staging) + align256(sizeof(BoxTable)));
  auto* cd = reinterpret_cast<CoilDev*>(reinterpret_cast<char*>(fd) + align256(sizeof(FieldDev)));
  memset(bt, 0, sizeof(BoxTable));
  memset(fd, 0, sizeof(FieldDev));
  memset(cd, 0, sizeof(CoilDev));
  bt->n_boxes = a.n_boxes;
  int64_t sites = 0;
  for (int b = 0; b < a.n_boxes; ++b) {
    bt->box[b] = a.boxes[b];
    bt->first_site[b] = sites;
    sites += a.boxes[b].count[0] * a.boxes[b].count[1] * a.boxes[b].count[2];
  }
  bt->first_site[a.n_boxes] = sites;
  fd->const_dw = a.field.const_dw;
  fd->n_poly = a.field.n_poly;
  fd->n_bumps = a.field.n_bumps;
  fd->poly_len = a.field.poly_len;
  fd->poly_scale = a.field.poly_scale;
  fd->peak_mode = a.field.poly_peak > 0.0;
  for (int i = 0; i < 4 * a.field.n_poly; ++i) fd->poly[i] = a.field.poly[i];
  for (int i = 0; i < 5 * a.field.n_bumps; ++i) fd->bumps[i] = a.field.bumps[i];
  cd->n_coils = a.n_coils;
  cd->uniform_s = a.uniform_s;
  for (int c = 0; c < a.n_coils; ++c) cd->coil[c] = a.coils[c];

  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align256(bytes);
    return r;
  };
  auto* d_bt = reinterpret_cast<BoxTable*>(take(sizeof(BoxTable)));
  auto* d_fd = reinterpret_cast<FieldDev*>(take(sizeof(FieldDev)));
  auto* d_cd = reinterpret_cast<CoilDev*>(take(sizeof(CoilDev)));
  auto* d_shapes = reinterpret_cast<bloch_shape_t*>(take(sizeof(bloch_shape_t) * kMaxShapes));
  auto* d_label = reinterpret_cast<int32_t*>(take(4 * (size_t)(sites + 1)));
  auto* d_keep = reinterpret_cast<uint32_t*>(take(4 * (size_t)(sites + 1)));
  auto* d_slot = reinterpret_cast<uint32_t*>(take(4 * (size_t)(sites + 1)));
  auto* d_poly = reinterpret_cast<double*>(take(8 * (size_t)(sites + 1)));
  auto* d_misc = reinterpret_cast<unsigned long long*>(take(64));  // [0] absmax, [1] bad flag, [2] count
  size_t cub_bytes = scratch_bytes - (size_t)(p - static_cast<char*>(scratch));
  void* d_cub = p;

  cudaError_t e;
#define RCK(x)                        \
  do {                                \
    if ((e = (x)) != cudaSuccess) return e; \
  } while (0)
  RCK(cudaMemcpyAsync(d_bt, bt, sizeof(BoxTable), cudaMemcpyHostToDevice, st));
  RCK(cudaMemcpyAsync(d_fd, fd, sizeof(FieldDev), cudaMemcpyHostToDevice, st));
  RCK(cudaMemcpyAsync(d_cd, cd, sizeof(CoilDev), cudaMemcpyHostToDevice, st));
  if (a.n_shapes) RCK(cudaMemcpyAsync(d_shapes, a.shapes, sizeof(bloch_shape_t) * a.n_shapes,
                                      cudaMemcpyHostToDevice, st));
  RCK(cudaMemsetAsync(d_misc, 0, 64, st));
  *n_out = 0;
  *bad_out = 0;
  if (sites == 0) return cudaStreamSynchronize(st);
  const int grid = (int)std::min<int64_t>((sites + kRasterThreads - 1) / kRasterThreads, (int64_t)n_sm * 8);
  label_kernel<<<grid, kRasterThreads, 0, st>>>(d_bt, d_shapes, sites, d_label, d_keep);
  RCK(cudaGetLastError());
  RCK(cub::DeviceScan::ExclusiveSum(d_cub, cub_bytes, d_keep, d_slot, (int)sites, st));
  // count = slot[last] + keep[last]
  uint32_t tail[2];
  RCK(cudaMemcpyAsync(&tail[0], d_slot + sites - 1, 4, cudaMemcpyDeviceToHost, st));
  RCK(cudaMemcpyAsync(&tail[1], d_keep + sites - 1, 4, cudaMemcpyDeviceToHost, st));
  RCK(cudaStreamSynchronize(st));
  const int64_t n = (int64_t)tail[0] + tail[1];
  if (n > a.capacity) {
    *n_out = n;
    return cudaSuccess;  // caller reports the capacity error
  }
  emit_kernel<<<grid, kRasterThreads, 0, st>>>(d_bt, d_shapes, d_fd, d_cd, sites, d_label, d_keep, d_slot, n,
                                               a.out, d_poly, d_misc, reinterpret_cast<int*>(d_misc + 1));
  RCK(cudaGetLastError());
  if (fd->peak_mode && fd->n_poly > 0) {
    const int g2 = (int)std::min<int64_t>((n + kRasterThreads - 1) / kRasterThreads, (int64_t)n_sm * 8);
    if (g2 > 0) peak_kernel<<<g2, kRasterThreads, 0, st>>>(n, d_poly, d_misc, a.field.poly_peak, a.out.domega);
    RCK(cudaGetLastError());
  }
  int bad = 0;
  RCK(cudaMemcpyAsync(&bad, d_misc + 1, 4, cudaMemcpyDeviceToHost, st));
  RCK(cudaStreamSynchronize(st));
  *n_out = n;
  *bad_out = bad;
  return cudaSuccess;
#undef RCK
}

}  // namespace bloch
