// tk_2d.cu -- parallel-beam and fan-beam 2D projectors for sm_100a.
//
// Reference: /root/reference/pkg/src/tomokit/_kernels.py:80-114 (_march_2d),
// 160-251 (forward/back parallel & fan).  Same scheme as the cone kernels:
// float64 per-ray set-up, float32 midpoint march in padded-index space,
// voxel-driven float32 gathers for the back projectors.
#include <algorithm>
#include <cmath>
#include <vector>

#include "tk_common.cuh"

namespace tk {

struct Ray2Setup {
  float ex, ey, gx, gy;
  int n;
  float last;
};

__device__ __forceinline__ bool clip_axis2(double p, double d, double h, double &t0,
                                           double &t1) {
  if (fabs(d) > kTiny) {
    double ta = (-h - p) / d, tb = (h - p) / d;
    t0 = fmax(t0, fmin(ta, tb));
    t1 = fmin(t1, fmax(ta, tb));
    return true;
  }
  return !(p < -h || p > h);
}

// _kernels.py:80-98 (clip + loop bounds of _march_2d)
__device__ __forceinline__ bool ray2_setup(double px, double py, double dx, double dy, int nx,
                                           int ny, double sx, double sy, double step,
                                           Ray2Setup &rs) {
  double t0 = -1e300, t1 = 1e300;
  if (!clip_axis2(px, dx, (nx + 1) * sx / 2.0, t0, t1)) return false;
  if (!clip_axis2(py, dy, (ny + 1) * sy / 2.0, t0, t1)) return false;
  if (!(t0 < t1)) return false;
  double span = (t1 - kTiny - t0) / step;
  if (!(span > 0.0)) return false;
  int n = (int)ceil(span);
  double last = (t1 - t0) / step - (double)(n - 1);
  if (last > 1.0) last = 1.0;
  const double cx = (nx - 1) / 2.0 + 1.0, cy = (ny - 1) / 2.0 + 1.0;
  rs.ex = (float)((px + t0 * dx) / sx + cx);
  rs.ey = (float)((py + t0 * dy) / sy + cy);
  rs.gx = (float)(step * dx / sx);
  rs.gy = (float)(step * dy / sy);
  rs.n = n;
  rs.last = (float)last;
  return true;
}

// Bilinear sample of the zero-padded image (unpadded storage; out-of-range taps
// read as zero, which equals the reference's explicit one-pixel zero margin).
__device__ __forceinline__ float bilinear_padded(const float *__restrict__ img, int nx, int ny,
                                                 float fx, float fy) {
  const float flx = floorf(fx), fly = floorf(fy);
  const int ix = (int)flx, iy = (int)fly;  // padded indices
  if ((unsigned)ix >= (unsigned)(nx + 1) || (unsigned)iy >= (unsigned)(ny + 1)) return 0.f;
  const float wx = fx - flx, wy = fy - fly;
  const int x0 = ix - 1, y0 = iy - 1;  // unpadded indices of the lower taps
  const bool xa = x0 >= 0, xb = x0 + 1 < nx, ya = y0 >= 0, yb = y0 + 1 < ny;
  const float *r0 = img + (long long)y0 * nx + x0;
  const float *r1 = r0 + nx;
  const float p00 = (ya && xa) ? __ldg(r0) : 0.f;
  const float p01 = (ya && xb) ? __ldg(r0 + 1) : 0.f;
  const float p10 = (yb && xa) ? __ldg(r1) : 0.f;
  const float p11 = (yb && xb) ? __ldg(r1 + 1) : 0.f;
  return lerpf(lerpf(p00, p01, wx), lerpf(p10, p11, wx), wy);
}

__device__ __forceinline__ void bilinear_scatter(float *__restrict__ img, int nx, int ny,
                                                 float fx, float fy, float g) {
  const float flx = floorf(fx), fly = floorf(fy);
  const int ix = (int)flx, iy = (int)fly;
  if ((unsigned)ix >= (unsigned)(nx + 1) || (unsigned)iy >= (unsigned)(ny + 1)) return;
  const float wx = fx - flx, wy = fy - fly;
  const int x0 = ix - 1, y0 = iy - 1;
  const bool xa = x0 >= 0, xb = x0 + 1 < nx, ya = y0 >= 0, yb = y0 + 1 < ny;
  float *r0 = img + (long long)y0 * nx + x0;
  float *r1 = r0 + nx;
  if (ya && xa) atomicAdd(r0, g * (1.f - wx) * (1.f - wy));
  if (ya && xb) atomicAdd(r0 + 1, g * wx * (1.f - wy));
  if (yb && xa) atomicAdd(r1, g * (1.f - wx) * wy);
  if (yb && xb) atomicAdd(r1 + 1, g * wx * wy);
}

// Ray of (angle ia, detector pixel j): origin + unit direction (float64).
__device__ __forceinline__ void ray_2d(bool fan, double ct, double st, double sdd, double sid,
                                       double u, double &px, double &py, double &dx,
                                       double &dy) {
  if (!fan) {  // _kernels.py:169-171
    px = u * ct;
    py = u * st;
    dx = -st;
    dy = ct;
  } else {  // _kernels.py:207-216
    const double srcx = sid * ct, srcy = sid * st;
    const double pixx = -(sdd - sid) * ct - u * st;
    const double pixy = -(sdd - sid) * st + u * ct;
    double ddx = pixx - srcx, ddy = pixy - srcy;
    const double inv = 1.0 / sqrt(ddx * ddx + ddy * ddy);
    px = srcx;
    py = srcy;
    dx = ddx * inv;
    dy = ddy * inv;
  }
}

template <bool FAN, bool ADJ>
__global__ void __launch_bounds__(256)
    fp2d_kernel(const float *__restrict__ in, int nx, int ny, double sx, double sy,
                const double2 *__restrict__ cs, int n_ang, int n_det, double ds, double sdd,
                double sid, double step, float *__restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n_ang * n_det) return;
  const int ia = (int)(idx / n_det);
  const int j = (int)(idx % n_det);
  const double2 a = cs[ia];
  const double u = (j - (n_det - 1) / 2.0) * ds;
  double px, py, dx, dy;
  ray_2d(FAN, a.x, a.y, sdd, sid, u, px, py, dx, dy);
  Ray2Setup rs;
  const bool hit = ray2_setup(px, py, dx, dy, nx, ny, sx, sy, step, rs);
  if (!ADJ) {
    float acc = 0.f;
    if (hit) {
      const int nfull = rs.n - 1;
      for (int k = 0; k < nfull; ++k) {
        const float kf = (float)k + 0.5f;
        acc += bilinear_padded(in, nx, ny, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey));
      }
      const float kf = (float)nfull + 0.5f * rs.last;
      acc += rs.last * bilinear_padded(in, nx, ny, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey));
    }
    out[idx] = acc * (float)step;
  } else {
    const float y = __ldg(in + idx);
    if (!hit || y == 0.f) return;
    const float g = y * (float)step;
    const int nfull = rs.n - 1;
    for (int k = 0; k < nfull; ++k) {
      const float kf = (float)k + 0.5f;
      bilinear_scatter(out, nx, ny, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey), g);
    }
    const float kf = (float)nfull + 0.5f * rs.last;
    bilinear_scatter(out, nx, ny, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey), g * rs.last);
  }
}

struct Bp2View {  // per-angle float32 constants
  float c, s;     // cos, sin (fan) or cos/ds, sin/ds (parallel)
};

// Voxel-driven gathers, _kernels.py:174-195 (parallel) and 219-251 (fan).
template <bool FAN, bool WEIGHTED>
__global__ void __launch_bounds__(256)
    bp2d_kernel(const float *__restrict__ sino, int n_ang, int n_det,
                const Bp2View *__restrict__ views, float hfrac, int hint, float sdd_over_ds, float sid,
                int nx, int ny, float sx, float sy, float *__restrict__ out) {
  __shared__ Bp2View sv[256];
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const bool active = ix < nx && iy < ny;
  const float x = ((float)ix - (nx - 1) * 0.5f) * sx;
  const float y = ((float)iy - (ny - 1) * 0.5f) * sy;
  float acc = 0.f;
  for (int a0 = 0; a0 < n_ang; a0 += 256) {
    const int nch = min(256, n_ang - a0);
    __syncthreads();
    if ((int)threadIdx.x < nch) sv[threadIdx.x] = views[a0 + threadIdx.x];
    __syncthreads();
    if (!active) continue;
    for (int j = 0; j < nch; ++j) {
      const Bp2View V = sv[j];
      const float *row = sino + (long long)(a0 + j) * n_det;
      float t, q = 1.f;  // detector coordinate relative to the centre (fp32 stays fine for wide detectors)
      if (!FAN) {
        t = fmaf(x, V.c, y * V.s);
      } else {
        const float w = sid - x * V.c - y * V.s;
        if (!(w > 1e-12f)) continue;
        const float rw = 1.f / w;
        t = sdd_over_ds * (y * V.c - x * V.s) * rw;
        if (WEIGHTED) {
          q = sid * rw;
          q *= q;
        }
      }
      const float tt = t + hfrac, fl = floorf(tt);  // f = tt + hint, hint integer
      const int j0 = (int)fl + hint;
      const float w = tt - fl;
      const float g0 = ((unsigned)j0 < (unsigned)n_det) ? 1.f - w : 0.f;
      const float g1 = ((unsigned)(j0 + 1) < (unsigned)n_det) ? w : 0.f;
      const int ja = min(max(j0, 0), n_det - 1), jb = min(max(j0 + 1, 0), n_det - 1);
      const float val = fmaf(g0, __ldg(row + ja), g1 * __ldg(row + jb));
      acc = WEIGHTED ? fmaf(q, val, acc) : acc + val;
    }
  }
  if (active) out[(long long)iy * nx + ix] = acc;
}

// Exact transposes B^T of the voxel-driven gathers above: one CTA per angle;
// every pixel scatters its value times the two interpolation weights it gathers
// with (times the fan distance weight) into the angle's detector row, accumulated
// with shared-memory atomics (rows up to kBt2Max detectors) or global atomics.
// fp32 atomics: summation order is not deterministic.
constexpr int kBt2Max = 12288;
template <bool FAN, bool WEIGHTED, bool SMEM>
__global__ void __launch_bounds__(256)
    bp2d_adjoint_kernel(const float *__restrict__ img, int n_det, const Bp2View *__restrict__ views, float hfrac,
                        int hint, float sdd_over_ds, float sid, int nx, int ny, float sx, float sy,
                        float *__restrict__ sino) {
  extern __shared__ float row_acc[];
  const int a = blockIdx.x;
  const Bp2View V = views[a];
  float *row = SMEM ? row_acc : sino + (long long)a * n_det;
  if (SMEM) {
    for (int j = threadIdx.x; j < n_det; j += blockDim.x) row[j] = 0.f;
    __syncthreads();
  }
  const long long npix = (long long)nx * ny;
  for (long long i = threadIdx.x; i < npix; i += blockDim.x) {
    const float g = __ldg(img + i);
    if (g == 0.f) continue;
    const int ix = (int)(i % nx), iy = (int)(i / nx);
    const float x = ((float)ix - (nx - 1) * 0.5f) * sx;
    const float y = ((float)iy - (ny - 1) * 0.5f) * sy;
    float t, q = 1.f;
    if (!FAN) {
      t = fmaf(x, V.c, y * V.s);
    } else {
      const float w = sid - x * V.c - y * V.s;
      if (!(w > 1e-12f)) continue;
      const float rw = 1.f / w;
      t = sdd_over_ds * (y * V.c - x * V.s) * rw;
      if (WEIGHTED) {
        q = sid * rw;
        q *= q;
      }
    }
    const float tt = t + hfrac, fl = floorf(tt);
    const int j0 = (int)fl + hint;
    const float w = tt - fl, gq = g * q;
    if ((unsigned)j0 < (unsigned)n_det) atomicAdd(row + j0, (1.f - w) * gq);
    if ((unsigned)(j0 + 1) < (unsigned)n_det) atomicAdd(row + j0 + 1, w * gq);
  }
  if (SMEM) {
    __syncthreads();
    for (int j = threadIdx.x; j < n_det; j += blockDim.x) sino[(long long)a * n_det + j] = row[j];
  }
}

static int upload_angles(Scratch &d, const double *cos_a, const double *sin_a, int n,
                         cudaStream_t st) {
  std::vector<double2> h(n);
  for (int i = 0; i < n; ++i) h[i] = make_double2(cos_a[i], sin_a[i]);
  TK_TRY_CUDA(upload(d, h.data(), sizeof(double2) * n, st));
  return TK_OK;
}

static int fp2d(bool fan, bool adj, const float *in, int ny, int nx, double sy, double sx,
                const double *cos_a, const double *sin_a, int n_ang, double sdd, double sid,
                int n_det, double ds, double step, float *out, void *stream) {
  clear_error();
  if (!in || !out || !cos_a || !sin_a) return fail_arg("2D projector: null pointer");
  if (ny < 1 || nx < 1 || n_ang < 1 || n_det < 1) return fail_arg("2D projector: non-positive extent");
  if (!(sx > 0 && sy > 0 && ds > 0 && step > 0)) return fail_arg("2D projector: spacing/step must be > 0");
  if (fan && !(sid > 0 && sid < sdd)) return fail_arg("fan projector requires 0 < sid < sdd");
  cudaStream_t st = as_stream(stream);
  Scratch d;
  int rc = upload_angles(d, cos_a, sin_a, n_ang, st);
  if (rc) return rc;
  const long long n = (long long)n_ang * n_det;
  const unsigned grid = ceil_div(n, 256);
  if (adj) TK_TRY_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)nx * ny, st));
  if (fan && adj)
    fp2d_kernel<true, true><<<grid, 256, 0, st>>>(in, nx, ny, sx, sy, d.as<double2>(), n_ang, n_det, ds, sdd, sid, step, out);
  else if (fan)
    fp2d_kernel<true, false><<<grid, 256, 0, st>>>(in, nx, ny, sx, sy, d.as<double2>(), n_ang, n_det, ds, sdd, sid, step, out);
  else if (adj)
    fp2d_kernel<false, true><<<grid, 256, 0, st>>>(in, nx, ny, sx, sy, d.as<double2>(), n_ang, n_det, ds, sdd, sid, step, out);
  else
    fp2d_kernel<false, false><<<grid, 256, 0, st>>>(in, nx, ny, sx, sy, d.as<double2>(), n_ang, n_det, ds, sdd, sid, step, out);
  TK_LAUNCHED("fp2d_kernel");
  return TK_OK;
}

static int bp2d(bool fan, const float *sino, int n_ang, int n_det, const double *cos_a,
                const double *sin_a, double sdd, double sid, double ds, int ny, int nx,
                double sy, double sx, bool weighted, float *out, void *stream) {
  clear_error();
  if (!sino || !out || !cos_a || !sin_a) return fail_arg("2D back projector: null pointer");
  if (ny < 1 || nx < 1 || n_ang < 1 || n_det < 1) return fail_arg("2D back projector: non-positive extent");
  if (!(sx > 0 && sy > 0 && ds > 0)) return fail_arg("2D back projector: spacing must be > 0");
  if (fan && !(sid > 0 && sid < sdd)) return fail_arg("fan back projector requires 0 < sid < sdd");
  cudaStream_t st = as_stream(stream);
  std::vector<Bp2View> h(n_ang);
  for (int i = 0; i < n_ang; ++i) {
    if (fan) {
      h[i].c = (float)cos_a[i];
      h[i].s = (float)sin_a[i];
    } else {
      h[i].c = (float)(cos_a[i] / ds);
      h[i].s = (float)(sin_a[i] / ds);
    }
  }
  Scratch d;
  TK_TRY_CUDA(upload(d, h.data(), sizeof(Bp2View) * n_ang, st));
  dim3 grid(ceil_div(nx, 32), ceil_div(ny, 8));
  const int hint = (n_det - 1) / 2;  // detector centre (n_det - 1) / 2 = hint + hfrac, hfrac in {0, 1/2}
  const float hfrac = (n_det - 1) % 2 ? 0.5f : 0.f;
  const float sdd_ds = (float)(sdd / ds);
  if (!fan)
    bp2d_kernel<false, false><<<grid, 256, 0, st>>>(sino, n_ang, n_det, d.as<Bp2View>(), hfrac, hint, 0.f, 0.f, nx, ny,
                                                    (float)sx, (float)sy, out);
  else if (weighted)
    bp2d_kernel<true, true><<<grid, 256, 0, st>>>(sino, n_ang, n_det, d.as<Bp2View>(), hfrac, hint, sdd_ds, (float)sid,
                                                  nx, ny, (float)sx, (float)sy, out);
  else
    bp2d_kernel<true, false><<<grid, 256, 0, st>>>(sino, n_ang, n_det, d.as<Bp2View>(), hfrac, hint, sdd_ds, (float)sid,
                                                   nx, ny, (float)sx, (float)sy, out);
  TK_LAUNCHED("bp2d_kernel");
  return TK_OK;
}

static int bp2d_adjoint(bool fan, const float *img, int ny, int nx, double sy, double sx, const double *cos_a,
                        const double *sin_a, int n_ang, double sdd, double sid, int n_det, double ds, bool weighted,
                        float *sino, void *stream) {
  clear_error();
  if (!img || !sino || !cos_a || !sin_a) return fail_arg("2D back-projection transpose: null pointer");
  if (ny < 1 || nx < 1 || n_ang < 1 || n_det < 1) return fail_arg("2D back-projection transpose: non-positive extent");
  if (!(sx > 0 && sy > 0 && ds > 0)) return fail_arg("2D back-projection transpose: spacing must be > 0");
  if (fan && !(sid > 0 && sid < sdd)) return fail_arg("fan back projector requires 0 < sid < sdd");
  if (!fan && weighted) return fail_arg("parallel backprojection has no distance weighting");
  cudaStream_t st = as_stream(stream);
  std::vector<Bp2View> h(n_ang);
  for (int i = 0; i < n_ang; ++i) {
    h[i].c = (float)(fan ? cos_a[i] : cos_a[i] / ds);
    h[i].s = (float)(fan ? sin_a[i] : sin_a[i] / ds);
  }
  Scratch d;
  TK_TRY_CUDA(upload(d, h.data(), sizeof(Bp2View) * n_ang, st));
  const int hint = (n_det - 1) / 2;  // detector centre (n_det - 1) / 2 = hint + hfrac, hfrac in {0, 1/2}
  const float hfrac = (n_det - 1) % 2 ? 0.5f : 0.f, sdd_ds = (float)(sdd / ds);
  const bool smem = n_det <= kBt2Max;
  const size_t sb = smem ? sizeof(float) * n_det : 0;
  if (!smem) TK_TRY_CUDA(cudaMemsetAsync(sino, 0, sizeof(float) * (size_t)n_ang * n_det, st));
  auto kern = fan ? (weighted ? (smem ? bp2d_adjoint_kernel<true, true, true> : bp2d_adjoint_kernel<true, true, false>)
                              : (smem ? bp2d_adjoint_kernel<true, false, true> : bp2d_adjoint_kernel<true, false, false>))
                  : (smem ? bp2d_adjoint_kernel<false, false, true> : bp2d_adjoint_kernel<false, false, false>);
  if (sb > 48 * 1024) TK_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
  kern<<<n_ang, 256, sb, st>>>(img, n_det, d.as<Bp2View>(), hfrac, hint, sdd_ds, (float)sid, nx, ny, (float)sx, (float)sy,
                               sino);
  TK_LAUNCHED("bp2d_adjoint_kernel");
  return TK_OK;
}

}  // namespace tk

using namespace tk;

extern "C" {

int tk_back_parallel_2d_adjoint(const float *img, int ny, int nx, double sy, double sx, const double *cos_a,
                                const double *sin_a, int n_ang, int n_det, double ds, float *sino_out, void *stream) {
  return bp2d_adjoint(false, img, ny, nx, sy, sx, cos_a, sin_a, n_ang, 0.0, 0.0, n_det, ds, false, sino_out, stream);
}

int tk_back_fan_2d_adjoint(const float *img, int ny, int nx, double sy, double sx, const double *cos_a,
                           const double *sin_a, int n_ang, double sdd, double sid, int n_det, double ds, int weighted,
                           float *sino_out, void *stream) {
  return bp2d_adjoint(true, img, ny, nx, sy, sx, cos_a, sin_a, n_ang, sdd, sid, n_det, ds, weighted != 0, sino_out,
                      stream);
}

int tk_forward_parallel_2d(const float *vol, int ny, int nx, double sy, double sx,
                           const double *cos_a, const double *sin_a, int n_ang, int n_det,
                           double ds, double step, float *out, void *stream) {
  return fp2d(false, false, vol, ny, nx, sy, sx, cos_a, sin_a, n_ang, 0.0, 0.0, n_det, ds, step,
              out, stream);
}

int tk_back_parallel_2d(const float *sino, int n_ang, int n_det, const double *cos_a,
                        const double *sin_a, double ds, int ny, int nx, double sy, double sx,
                        float *out, void *stream) {
  return bp2d(false, sino, n_ang, n_det, cos_a, sin_a, 0.0, 0.0, ds, ny, nx, sy, sx, false, out,
              stream);
}

int tk_forward_fan_2d(const float *vol, int ny, int nx, double sy, double sx,
                      const double *cos_a, const double *sin_a, int n_ang, double sdd,
                      double sid, int n_det, double ds, double step, float *out, void *stream) {
  return fp2d(true, false, vol, ny, nx, sy, sx, cos_a, sin_a, n_ang, sdd, sid, n_det, ds, step,
              out, stream);
}

int tk_back_fan_2d(const float *sino, int n_ang, int n_det, const double *cos_a,
                   const double *sin_a, double sdd, double sid, double ds, int ny, int nx,
                   double sy, double sx, int weighted, float *out, void *stream) {
  return bp2d(true, sino, n_ang, n_det, cos_a, sin_a, sdd, sid, ds, ny, nx, sy, sx,
              weighted != 0, out, stream);
}

int tk_forward_parallel_2d_adjoint(const float *sino, int n_ang, int n_det,
                                   const double *cos_a, const double *sin_a, double ds,
                                   double step, int ny, int nx, double sy, double sx,
                                   float *vol_out, void *stream) {
  return fp2d(false, true, sino, ny, nx, sy, sx, cos_a, sin_a, n_ang, 0.0, 0.0, n_det, ds, step,
              vol_out, stream);
}

int tk_forward_fan_2d_adjoint(const float *sino, int n_ang, int n_det, const double *cos_a,
                              const double *sin_a, double sdd, double sid, double ds,
                              double step, int ny, int nx, double sy, double sx,
                              float *vol_out, void *stream) {
  return fp2d(true, true, sino, ny, nx, sy, sx, cos_a, sin_a, n_ang, sdd, sid, n_det, ds, step,
              vol_out, stream);
}

}  // extern "C"
