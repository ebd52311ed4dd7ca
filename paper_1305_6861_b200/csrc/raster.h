// Device-side object model (raster_kernels.cu): host-facing launch interface.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bloch_b200.h"

namespace bloch {

constexpr int kMaxShapes = 1024;
constexpr int kMaxPoly = 64;
constexpr int kMaxBumps = 64;
constexpr int kMaxCoils = 32;
constexpr int kMaxRasterBoxes = 64;

struct RasterOut {
  double *pos, *mx, *my, *mz, *t1, *t2, *m0, *domega, *weight;
};

struct RasterArgs {
  const bloch_box_t* boxes;
  int32_t n_boxes;
  const bloch_shape_t* shapes;
  int32_t n_shapes;
  bloch_field_t field;
  const bloch_coil_t* coils;
  int32_t n_coils;
  double uniform_s;
  int64_t capacity;
  RasterOut out;
};

// bytes of device scratch raster_run needs for n_sites lattice sites
size_t raster_scratch_bytes(int64_t n_sites);
// bytes of host staging raster_run needs
size_t raster_staging_bytes();
// label -> scan -> emit on `st`; synchronises `st` (twice).  *n_out = emitted spins (may exceed
// a.capacity, in which case nothing was written); *bad_out != 0 when an emitted tissue value is invalid.
cudaError_t raster_run(const RasterArgs& a, void* scratch, size_t scratch_bytes, void* host_staging, int n_sm,
                       cudaStream_t st, int64_t* n_out, int* bad_out);

}  // namespace bloch
