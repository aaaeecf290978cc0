// tk_fp_tex.cu -- texture-unit forward projectors, kept as the benchmark
// comparison the north star asks for (hardware texture path vs the hand-written
// fp32 gathers of tk_fp.cu; DESIGN.md 4.2 table).  Selected with
// TK_FP_ALGO=tex (TLD4 gathers of exact fp32 texels, fp32 weights) or
// TK_FP_ALGO=hwtex (hardware trilinear filtering: 8-bit weights, not a parity
// path).  Same ray set-up and midpoint march as the reference
// (_kernels.py:254-278, 117-157).
#include <algorithm>
#include <vector>

#include "tk_cone_fp.cuh"
#include "tk_tex.cuh"

namespace tk {

constexpr int kFtBX = 8, kFtBY = 16;  // an 8 x 16 detector tile per CTA (one view)

// Texture-gather variant: the volume lives in a layered CUDA array (layer =
// z slice, block-linear (x, y) tiles), each sample fetches its two 2x2 tap
// quads with TLD4 (exact fp32 texels; the interpolation weights stay fp32 in
// registers).  x/y zero-extension comes from border addressing; only the
// layer index needs an explicit range check (layers clamp).
__device__ __forceinline__ float trilinear_tex(cudaTextureObject_t tex, int nz, float fx, float fy,
                                               float fz) {
  const float flx = floorf(fx), fly = floorf(fy), flz = floorf(fz);
  const float wx = fx - flx, wy = fy - fly, wz = fz - flz;
  const int lz = (int)flz - 1;  // unpadded index of the lower slice
  float lo = 0.f, hi = 0.f;
  // gather centre (flx, fly) in unpadded texel units = (ix_u + 1, iy_u + 1)
  if ((unsigned)lz < (unsigned)nz) {
    const float4 g = gather_a2d(tex, lz, flx, fly);
    lo = lerpf(lerpf(g.w, g.z, wx), lerpf(g.x, g.y, wx), wy);
  }
  if ((unsigned)(lz + 1) < (unsigned)nz) {
    const float4 g = gather_a2d(tex, lz + 1, flx, fly);
    hi = lerpf(lerpf(g.w, g.z, wx), lerpf(g.x, g.y, wx), wy);
  }
  return lerpf(lo, hi, wz);
}

__global__ void __launch_bounds__(kFtBX *kFtBY)
    cone_fp_tex_kernel(cudaTextureObject_t tex, int nx, int ny, int nz, double sx, double sy,
                       double sz, const ConeRayView *__restrict__ views, int rows, int cols,
                       double step, float *__restrict__ out) {
  const int c = blockIdx.x * kFtBX + threadIdx.x;
  const int r = blockIdx.y * kFtBY + threadIdx.y;
  const int v = blockIdx.z;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const ConeRayView V = views[v];
  RaySetup rs;
  if (!cone_ray_setup(V, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  float acc = 0.f;
  const int nfull = rs.n - 1;
#pragma unroll 4
  for (int k = 0; k < nfull; ++k) {
    const float kf = (float)k + 0.5f;
    acc += trilinear_tex(tex, nz, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey),
                         fmaf(kf, rs.gz, rs.ez));
  }
  const float kf = (float)nfull + 0.5f * rs.last;
  acc += rs.last * trilinear_tex(tex, nz, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey),
                                 fmaf(kf, rs.gz, rs.ez));
  *dst = acc * (float)step;
}

// Hardware-trilinear variant (benchmark comparison only: the texture unit's
// 8-bit fractional weights cost accuracy).  3D array, border 0.
__global__ void __launch_bounds__(kFtBX *kFtBY)
    cone_fp_hwtex_kernel(cudaTextureObject_t tex, int nx, int ny, int nz, double sx, double sy,
                         double sz, const ConeRayView *__restrict__ views, int rows, int cols,
                         double step, float *__restrict__ out) {
  const int c = blockIdx.x * kFtBX + threadIdx.x;
  const int r = blockIdx.y * kFtBY + threadIdx.y;
  const int v = blockIdx.z;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const ConeRayView V = views[v];
  RaySetup rs;
  if (!cone_ray_setup(V, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  // padded index p -> unpadded texel coordinate p - 1 + 0.5
  const float ex = rs.ex - 0.5f, ey = rs.ey - 0.5f, ez = rs.ez - 0.5f;
  float acc = 0.f;
  const int nfull = rs.n - 1;
#pragma unroll 4
  for (int k = 0; k < nfull; ++k) {
    const float kf = (float)k + 0.5f;
    acc += tex3D<float>(tex, fmaf(kf, rs.gx, ex), fmaf(kf, rs.gy, ey), fmaf(kf, rs.gz, ez));
  }
  const float kf = (float)nfull + 0.5f * rs.last;
  acc += rs.last * tex3D<float>(tex, fmaf(kf, rs.gx, ex), fmaf(kf, rs.gy, ey), fmaf(kf, rs.gz, ez));
  *dst = acc * (float)step;
}


int launch_fp_tex(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx, const double *sources,
                  const double *minv, int n_views, int rows, int cols, double step, bool hw, float *out,
                  cudaStream_t st) {
  std::vector<ConeRayView> hv(n_views);
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].minv[j] = minv[9 * i + j];
  }
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeRayView) * n_views, st));
  const dim3 block(kFtBX, kFtBY);
  TexLease lease;
  TK_TRY_CUDA(tex_acquire(vol, nx, ny, nz, hw ? TexKind::kVolumeLinear : TexKind::kLayeredPoint, st, lease));
  for (int v0 = 0; v0 < n_views; v0 += 65535) {  // views on gridDim.z
    const int nv = std::min(65535, n_views - v0);
    const dim3 grid(ceil_div(cols, kFtBX), ceil_div(rows, kFtBY), nv);
    float *o = out + (long long)v0 * rows * cols;
    if (hw)
      cone_fp_hwtex_kernel<<<grid, block, 0, st>>>(lease.tex, nx, ny, nz, sx, sy, sz,
                                                   dviews.as<ConeRayView>() + v0, rows, cols, step, o);
    else
      cone_fp_tex_kernel<<<grid, block, 0, st>>>(lease.tex, nx, ny, nz, sx, sy, sz, dviews.as<ConeRayView>() + v0,
                                                 rows, cols, step, o);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      tex_release(lease, st);
      return check_cuda(e, hw ? "cone_fp_hwtex_kernel" : "cone_fp_tex_kernel");
    }
    count_launch();
  }
  tex_release(lease, st);
  return TK_OK;
}

}  // namespace tk
