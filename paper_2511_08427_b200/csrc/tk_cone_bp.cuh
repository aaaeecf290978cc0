// tk_cone_bp.cuh -- per-view constants and launch parameters shared by the
// cone-beam back projectors (tk_cone.cu, tk_bp_tma.cu).
#pragma once

#include "tk_common.cuh"

namespace tk {

struct ConeVoxView {  // per-view back constants (float32), see pack_bp_views
  float a[4];  // column numerator (principal-point shifted)
  float b[4];  // row numerator (principal-point shifted)
  float w[4];  // depth
};

struct BpParams {
  const float *sino;
  long long view_stride;  // elements between views of the (band) sinogram
  int n_views, band_rows, cols;
  const ConeVoxView *views;
  float cu, cv;  // column / row shift constants (cv already minus row_begin)
  float sid;
  int nx, ny, z_begin, z_count;
  float cx, cy, cz;  // volume centre (index units)
  int accumulate;
  float *out;
  cudaTextureObject_t tex;  // layered sinogram (texture variants only)
};

// TMA-staged back projector (tk_bp_tma.cu) for z-invariant trajectories.
// Returns TK_OK, or -1 when the geometry does not suit it (caller falls back).
int launch_bp_tma(const BpParams &p, const ConeVoxView *host_views, bool weighted, cudaStream_t st);

}  // namespace tk
