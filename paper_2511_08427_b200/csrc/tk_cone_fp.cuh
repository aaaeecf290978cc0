// tk_cone_fp.cuh -- per-view constants and per-ray set-up shared by the cone
// forward projector (tk_fp.cu), its texture comparison kernels (tk_fp_tex.cu)
// and its transpose (tk_fp_adjoint.cu).
#pragma once

#include "tk_common.cuh"

namespace tk {

struct ConeRayView {  // per-view forward constants (float64): source, M^-1
  double src[3];
  double minv[9];
};

// Zero margin (voxels) of the forward projectors' orientation copies.
constexpr int kFpMargin = 2;




// ---------------------------------------------------------------------------
// Ray set-up shared by the forward projector and its transpose.
// Returns false when the ray misses the box (reference _clip_ray_3d, t0 >= t1).
// ---------------------------------------------------------------------------
struct RaySetup {
  float ex, ey, ez;  // padded-index coordinates of the clip entry point
  float gx, gy, gz;  // padded-index increment per full step
  int n;             // number of samples (reference loop count)
  float last;        // fraction of a step covered by the last sample (0,1]
  int face;          // axis (0 x, 1 y, 2 z) whose slab sets the entry t0
};

__device__ __forceinline__ bool clip_axis(double p, double d, double h, double &t0,
                                          double &t1, int axis, int &face) {
  if (fabs(d) > kTiny) {
    const double rd = 1.0 / d;  // one fp64 division per axis instead of two
    double ta = (-h - p) * rd, tb = (h - p) * rd;
    const double tn = fmin(ta, tb);
    if (tn > t0) face = axis;
    t0 = fmax(t0, tn);
    t1 = fmin(t1, fmax(ta, tb));
    return true;
  }
  return !(p < -h || p > h);
}

__device__ __forceinline__ bool cone_ray_setup(const ConeRayView &V, int r, int c, int nx,
                                               int ny, int nz, double sx, double sy,
                                               double sz, double step, RaySetup &rs) {
  // _kernels.py:262-265
  double dx = V.minv[0] * c + V.minv[1] * r + V.minv[2];
  double dy = V.minv[3] * c + V.minv[4] * r + V.minv[5];
  double dz = V.minv[6] * c + V.minv[7] * r + V.minv[8];
  double inv = rsqrt(dx * dx + dy * dy + dz * dz);
  dx *= inv;
  dy *= inv;
  dz *= inv;
  const double px = V.src[0], py = V.src[1], pz = V.src[2];
  // _kernels.py:125-130 (_clip_ray_3d on the half-extents (n+1) s / 2)
  double t0 = -1e300, t1 = 1e300;
  int face = 2;
  if (!clip_axis(px, dx, (nx + 1) * sx / 2.0, t0, t1, 0, face)) return false;
  if (!clip_axis(py, dy, (ny + 1) * sy / 2.0, t0, t1, 1, face)) return false;
  if (!clip_axis(pz, dz, (nz + 1) * sz / 2.0, t0, t1, 2, face)) return false;
  if (!(t0 < t1)) return false;
  // _kernels.py:133: while t < t1 - TINY  ->  n = ceil((t1 - TINY - t0) / step)
  const double istep = 1.0 / step;
  double span = (t1 - kTiny - t0) * istep;
  if (!(span > 0.0)) return false;
  int n = (int)ceil(span);
  double last = (t1 - t0) * istep - (double)(n - 1);
  if (last > 1.0) last = 1.0;
  // padded-index coordinates (centre (n-1)/2 + 1, _kernels.py:122-124, 138-140)
  const double cx = (nx - 1) / 2.0 + 1.0, cy = (ny - 1) / 2.0 + 1.0, cz = (nz - 1) / 2.0 + 1.0;
  rs.ex = (float)((px + t0 * dx) / sx + cx);
  rs.ey = (float)((py + t0 * dy) / sy + cy);
  rs.ez = (float)((pz + t0 * dz) / sz + cz);
  rs.gx = (float)(step * dx / sx);
  rs.gy = (float)(step * dy / sy);
  rs.gz = (float)(step * dz / sz);
  rs.n = n;
  rs.last = (float)last;
  rs.face = face;
  return true;
}

// tk_fp.cu: z-mirror symmetry test of a scan and the default launch.
bool views_z_mirror(const double *sources, const double *minv, int n_views, int rows);
bool fp_use_mirror(const double *sources, const double *minv, int n_views, int rows, int nz, int ny, int nx);
// tk_fp_tex.cu: texture-unit comparison kernels (hw: hardware trilinear filtering).
int launch_fp_tex(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx, const double *sources,
                  const double *minv, int n_views, int rows, int cols, double step, bool hw, float *out,
                  cudaStream_t st);

}  // namespace tk
