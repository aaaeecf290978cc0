// tk_cone.cu -- cone-beam voxel-driven back projection B y and its exact
// transpose B^T, for sm_100a.
//
// Reference semantics: /root/reference/pkg/src/tomokit/_kernels.py:281-322
// (back_cone_3d: per voxel and view, u = P (x, y, z, 1), behind-source test,
// bilinear detector taps with zero outside, optional (sid / w)^2 FDK weight).
// Projection-matrix rows are pre-multiplied by the voxel spacing and shifted by
// the detector centre (principal-point shift keeps fp32 well conditioned), and
// evaluated on centred integer voxel coordinates.  For trajectories whose
// detector column / depth rows have no z component (circular, helical,
// sinusoidal orbits with v = +z: "z-invariant") the column, depth and distance
// weight are computed once per (x, y, view) and reused along z.
//
// Kernels: cone_bp_tma_kernel (tk_bp_tma.cu; default for z-invariant
// trajectories), cone_bp_quad_kernel (any trajectory), cone_bp_tex_kernel
// (texture-unit comparison: TLD4 gathers, or hardware bilinear filtering),
// cone_bp_adjoint4_kernel + unquad_det_kernel (B^T).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tk_common.cuh"
#include "tk_cone_bp.cuh"
#include "tk_tex.cuh"

namespace tk {

constexpr int kBpBX = 32, kBpBY = 8, kBpChunk = 128;  // texture kernels: 32 x 8 (x, y) columns per CTA

// ---------------------------------------------------------------------------
// Quad-layout back projector ("quad", default).
//
// The (band) sinogram is first rewritten as tap quads: for every detector cell
// (r0, c0) with r0 in [-2, R], c0 in [-2, C] the float4
//   Q[v][r0+2][c0+2] = (S[r0][c0], S[r0][c0+1], S[r0+1][c0], S[r0+1][c0+1]),
// S = 0 outside the detector.  One 16-byte load then yields all four bilinear
// taps of an update, the zero border replaces every per-tap range test
// (reference _kernels.py:308-317), and an out-of-range row index is simply
// clamped onto the all-zero quads of rows -2 / R.  A warp covers an 8x4 (x, y)
// voxel tile (compact detector footprint) and each thread ZB voxels along z.
// ---------------------------------------------------------------------------
constexpr int kQuadPad = 2;
constexpr int kBqBX = 8, kBqBY = 32;

__global__ void quadify_kernel(const float *__restrict__ sino, int n_views, int rows, int cols,
                               float4 *__restrict__ quads) {
  const int qc = cols + 1 + kQuadPad, qr = rows + 1 + kQuadPad;
  const long long total = (long long)n_views * qr * qc;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % qc) - kQuadPad;
    const long long t = i / qc;
    const int r0 = (int)(t % qr) - kQuadPad;
    const int v = (int)(t / qr);
    const float *s = sino + (long long)v * rows * cols;
    const bool ca = (unsigned)c0 < (unsigned)cols, cb = (unsigned)(c0 + 1) < (unsigned)cols;
    const bool ra = (unsigned)r0 < (unsigned)rows, rb = (unsigned)(r0 + 1) < (unsigned)rows;
    float4 q;
    q.x = (ra && ca) ? __ldg(s + (long long)r0 * cols + c0) : 0.f;
    q.y = (ra && cb) ? __ldg(s + (long long)r0 * cols + c0 + 1) : 0.f;
    q.z = (rb && ca) ? __ldg(s + (long long)(r0 + 1) * cols + c0) : 0.f;
    q.w = (rb && cb) ? __ldg(s + (long long)(r0 + 1) * cols + c0 + 1) : 0.f;
    quads[i] = q;
  }
}

// Q42: a quarter-warp (the 8 lanes whose 16-byte loads share one L1 data
// wavefront per 128-byte line) covers 4 x 2 (x, y) voxels instead of 8 x 1, a
// tighter detector footprint (fewer lines per quarter).
template <int ZB, bool ZINV, bool WEIGHTED, bool Q42 = true>
__global__ void __launch_bounds__(kBqBX *kBqBY, 2) cone_bp_quad_kernel(const BpParams p,
                                                                   const float4 *__restrict__ quads) {
  __shared__ ConeVoxView sv[kBpChunk];
  int ix, iy;
  if (Q42) {
    const int t = threadIdx.y * kBqBX + threadIdx.x, w = t >> 5, l = t & 31;
    ix = blockIdx.x * kBqBX + (l & 3) + 4 * ((l >> 3) & 1);
    iy = blockIdx.y * kBqBY + 4 * w + ((l >> 2) & 1) + 2 * (l >> 4);
  } else {
    ix = blockIdx.x * kBqBX + threadIdx.x;
    iy = blockIdx.y * kBqBY + threadIdx.y;
  }
  const int zl0 = blockIdx.z * ZB;
  const bool active = ix < p.nx && iy < p.ny;
  const float xc = (float)ix - p.cx;
  const float yc = (float)iy - p.cy;
  const float zc0 = (float)(p.z_begin + zl0) - p.cz;
  const int tid = threadIdx.y * kBqBX + threadIdx.x;
  const int qc = p.cols + 1 + kQuadPad;                 // quads per row
  const int rmax = p.band_rows;                          // last (all-zero) quad row index r0
  const long long qview = (long long)(p.band_rows + 1 + kQuadPad) * qc;
  const float colmax = (float)(p.cols - 1);

  float acc[ZB];
#pragma unroll
  for (int k = 0; k < ZB; ++k) acc[k] = 0.f;

  for (int v0 = 0; v0 < p.n_views; v0 += kBpChunk) {
    const int nch = min(kBpChunk, p.n_views - v0);
    __syncthreads();
    for (int i = tid; i < nch * 12; i += kBqBX * kBqBY)
      reinterpret_cast<float *>(sv)[i] = __ldg(reinterpret_cast<const float *>(p.views + v0) + i);
    __syncthreads();
    if (!active) continue;
    for (int j = 0; j < nch; ++j) {
      const ConeVoxView &V = sv[j];
      const float4 *qv = quads + (long long)(v0 + j) * qview;
      const float a0 = fmaf(V.a[0], xc, fmaf(V.a[1], yc, fmaf(V.a[2], zc0, V.a[3])));
      const float b0 = fmaf(V.b[0], xc, fmaf(V.b[1], yc, fmaf(V.b[2], zc0, V.b[3])));
      const float w0 = fmaf(V.w[0], xc, fmaf(V.w[1], yc, fmaf(V.w[2], zc0, V.w[3])));
      if (ZINV) {
        if (!(w0 > (float)kTiny)) continue;  // _kernels.py:297-298
        const float rw = 1.f / w0;
        const float fc = fmaf(a0, rw, p.cu);
        const float flc = floorf(fc);
        if (!(flc >= -1.f && flc <= colmax)) continue;  // both column taps off the detector
        const float wc = fc - flc;
        float q = 1.f;
        if (WEIGHTED) {  // (sid / w)^2, _kernels.py:318-320
          q = p.sid * rw;
          q *= q;
        }
        const float g0 = q * (1.f - wc), g1 = q * wc;
        const float4 *col = qv + ((int)flc + kQuadPad);
        const float fr0 = fmaf(b0, rw, p.cv);
        const float dr = V.b[2] * rw;
        // batches of 8 independent 16-byte loads in flight per thread
#pragma unroll
        for (int k0 = 0; k0 < ZB; k0 += 8) {
          unsigned off[8];
          float wr[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float fr = fmaf((float)(k0 + i), dr, fr0);
            const float flr = floorf(fr);
            off[i] = (unsigned)((min(max((int)flr, -kQuadPad), rmax) + kQuadPad) * qc);
            wr[i] = fr - flr;
          }
          float4 t[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = __ldg(col + off[i]);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float top = fmaf(g1, t[i].y, g0 * t[i].x);
            const float bot = fmaf(g1, t[i].w, g0 * t[i].z);
            acc[k0 + i] += fmaf(wr[i], bot - top, top);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < ZB; ++k) {
          const float kf = (float)k;
          const float w = fmaf(kf, V.w[2], w0);
          if (!(w > (float)kTiny)) continue;
          const float rw = 1.f / w;
          const float fc = fmaf(fmaf(kf, V.a[2], a0), rw, p.cu);
          const float fr = fmaf(fmaf(kf, V.b[2], b0), rw, p.cv);
          const float flc = floorf(fc), flr = floorf(fr);
          const int c0 = min(max((int)flc, -kQuadPad), p.cols);
          const int r0 = min(max((int)flr, -kQuadPad), rmax);
          const float4 t = __ldg(qv + (long long)(r0 + kQuadPad) * qc + (c0 + kQuadPad));
          const float wc = fc - flc;
          const float top = lerpf(t.x, t.y, wc), bot = lerpf(t.z, t.w, wc);
          float val = lerpf(top, bot, fr - flr);
          if (WEIGHTED) {
            const float q = p.sid * rw;
            val *= q * q;
          }
          acc[k] += val;
        }
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < ZB; ++k) {
    const int zl = zl0 + k;
    if (zl < p.z_count) {
      float *o = p.out + ((long long)zl * p.ny + iy) * p.nx + ix;
      *o = p.accumulate ? *o + acc[k] : acc[k];
    }
  }
}

// ---------------------------------------------------------------------------
// Texture-gather variant: the (band) sinogram lives in a layered CUDA array
// (layer = view); each update fetches its 2x2 tap quad with one TLD4, the
// zero outside the detector comes from border addressing, and the bilinear
// weights stay exact fp32.  HW = true uses the texture unit's own bilinear
// filter instead (8-bit weights; benchmark comparison only).
template <int ZB, bool ZINV, bool WEIGHTED, bool HW>
__global__ void __launch_bounds__(kBpBX *kBpBY) cone_bp_tex_kernel(const BpParams p) {
  __shared__ ConeVoxView sv[kBpChunk];
  const int ix = blockIdx.x * kBpBX + threadIdx.x;
  const int iy = blockIdx.y * kBpBY + threadIdx.y;
  const int zl0 = blockIdx.z * ZB;
  const bool active = ix < p.nx && iy < p.ny;
  const float xc = (float)ix - p.cx;
  const float yc = (float)iy - p.cy;
  const float zc0 = (float)(p.z_begin + zl0) - p.cz;
  const int tid = threadIdx.y * kBpBX + threadIdx.x;
  const float colmax = (float)(p.cols - 1);

  float acc[ZB];
#pragma unroll
  for (int k = 0; k < ZB; ++k) acc[k] = 0.f;

  for (int v0 = 0; v0 < p.n_views; v0 += kBpChunk) {
    const int nch = min(kBpChunk, p.n_views - v0);
    __syncthreads();
    for (int i = tid; i < nch * 12; i += kBpBX * kBpBY)
      reinterpret_cast<float *>(sv)[i] = __ldg(reinterpret_cast<const float *>(p.views + v0) + i);
    __syncthreads();
    if (!active) continue;
    for (int j = 0; j < nch; ++j) {
      const ConeVoxView &V = sv[j];
      const int layer = v0 + j;
      const float a0 = fmaf(V.a[0], xc, fmaf(V.a[1], yc, fmaf(V.a[2], zc0, V.a[3])));
      const float b0 = fmaf(V.b[0], xc, fmaf(V.b[1], yc, fmaf(V.b[2], zc0, V.b[3])));
      const float w0 = fmaf(V.w[0], xc, fmaf(V.w[1], yc, fmaf(V.w[2], zc0, V.w[3])));
      if (ZINV) {
        if (!(w0 > (float)kTiny)) continue;
        const float rw = 1.f / w0;
        const float fc = fmaf(a0, rw, p.cu);
        const float flc = floorf(fc);
        if (!(flc >= -1.f && flc <= colmax)) continue;  // both column taps off the detector
        const float wc = fc - flc;
        float q = 1.f;
        if (WEIGHTED) {
          q = p.sid * rw;
          q *= q;
        }
        const float g0 = q * (1.f - wc), g1 = q * wc;
        const float fr0 = fmaf(b0, rw, p.cv);
        const float dr = V.b[2] * rw;
#pragma unroll
        for (int k = 0; k < ZB; ++k) {
          const float fr = fmaf((float)k, dr, fr0);
          if (HW) {
            acc[k] = fmaf(q, tex2DLayered<float>(p.tex, fc + 0.5f, fr + 0.5f, layer), acc[k]);
          } else {
            const float flr = floorf(fr);
            const float wr = fr - flr;
            const float4 t = gather_a2d(p.tex, layer, flc + 1.f, flr + 1.f);
            const float top = fmaf(g1, t.z, g0 * t.w);  // detector row r0: (c0, c0 + 1)
            const float bot = fmaf(g1, t.y, g0 * t.x);  // detector row r0 + 1
            acc[k] += fmaf(wr, bot - top, top);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < ZB; ++k) {
          const float kf = (float)k;
          const float w = fmaf(kf, V.w[2], w0);
          if (!(w > (float)kTiny)) continue;
          const float rw = 1.f / w;
          const float fc = fmaf(fmaf(kf, V.a[2], a0), rw, p.cu);
          const float fr = fmaf(fmaf(kf, V.b[2], b0), rw, p.cv);
          float q = 1.f;
          if (WEIGHTED) {
            q = p.sid * rw;
            q *= q;
          }
          float val;
          if (HW) {
            val = tex2DLayered<float>(p.tex, fc + 0.5f, fr + 0.5f, layer);
          } else {
            const float flc = floorf(fc), flr = floorf(fr);
            const float wc = fc - flc, wr = fr - flr;
            const float4 t = gather_a2d(p.tex, layer, flc + 1.f, flr + 1.f);
            const float top = lerpf(t.w, t.z, wc), bot = lerpf(t.x, t.y, wc);
            val = lerpf(top, bot, wr);
          }
          acc[k] = fmaf(q, val, acc[k]);
        }
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < ZB; ++k) {
    const int zl = zl0 + k;
    if (zl < p.z_count) {
      float *o = p.out + ((long long)zl * p.ny + iy) * p.nx + ix;
      *o = p.accumulate ? *o + acc[k] : acc[k];
    }
  }
}

// Quad form ("red4", default): one REDG.F32x4 per voxel-view update into a
// detector quad buffer Qs[v][r0+1][c0+1] += (w00, w01, w10, w11) (one-texel
// margin so partially covered cells keep their in-detector taps), folded back
// into the sinogram by unquad_det_kernel.  Weights and products of the
// reference's bilinear taps (_kernels.py:308-320).
__global__ void __launch_bounds__(256)
    cone_bp_adjoint4_kernel(const float *__restrict__ vol, int nx, int ny, int nz, float cx, float cy, float cz,
                            const ConeVoxView *__restrict__ views, int rows, int cols, float cu, float cv,
                            float sid, int weighted, float4 *__restrict__ qs) {
  const long long nvox = (long long)nx * ny * nz;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (i >= nvox) return;
  const float g = __ldg(vol + i);
  if (g == 0.f) return;
  const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / ((long long)nx * ny));
  const float xc = (float)ix - cx, yc = (float)iy - cy, zc = (float)iz - cz;
  const ConeVoxView V = views[v];
  const float w = fmaf(V.w[0], xc, fmaf(V.w[1], yc, fmaf(V.w[2], zc, V.w[3])));
  if (!(w > (float)kTiny)) return;
  const float rw = 1.f / w;
  const float fc = fmaf(fmaf(V.a[0], xc, fmaf(V.a[1], yc, fmaf(V.a[2], zc, V.a[3]))), rw, cu);
  const float fr = fmaf(fmaf(V.b[0], xc, fmaf(V.b[1], yc, fmaf(V.b[2], zc, V.b[3]))), rw, cv);
  float gg = g;
  if (weighted) {
    const float q = sid * rw;
    gg *= q * q;
  }
  const float flc = floorf(fc), flr = floorf(fr);
  const int c0 = (int)flc, r0 = (int)flr;
  if (r0 < -1 || r0 >= rows || c0 < -1 || c0 >= cols) return;  // all four taps off the detector
  const float wc = fc - flc, wr = fr - flr;
  float4 *e = qs + ((long long)v * (rows + 1) + (r0 + 1)) * (cols + 1) + (c0 + 1);
  red_add_v4(e, make_float4(gg * (1.f - wr) * (1.f - wc), gg * (1.f - wr) * wc, gg * wr * (1.f - wc), gg * wr * wc));
}

// sino[v][r][c] = Qs[r+1][c+1].x + Qs[r+1][c].y + Qs[r][c+1].z + Qs[r][c].w
__global__ void __launch_bounds__(256) unquad_det_kernel(const float4 *__restrict__ qs, int n_views, int rows,
                                                         int cols, float *__restrict__ sino) {
  const long long n = (long long)n_views * rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cols);
    const long long t = i / cols;
    const int r = (int)(t % rows);
    const long long v = t / rows;
    const float4 *row1 = qs + (v * (rows + 1) + (r + 1)) * (cols + 1), *row0 = row1 - (cols + 1);
    sino[i] = __ldg(row1 + c + 1).x + __ldg(row1 + c).y + __ldg(row0 + c + 1).z + __ldg(row0 + c).w;
  }
}

// ---------------------------------------------------------------------------
// host-side packing
// ---------------------------------------------------------------------------

// Fold voxel spacing into P and shift the column/row rows by the detector
// centre: a' = (P0 - cu P2) . (s * (i - c), 1) etc., so fc = cu + a'/w.
static void pack_bp_views(const double *mats, int n_views, double sx, double sy, double sz,
                          double cu, double cv, std::vector<ConeVoxView> &out, bool &zinv) {
  out.resize(n_views);
  zinv = true;
  for (int i = 0; i < n_views; ++i) {
    const double *P = mats + 12 * i;
    const double s[3] = {sx, sy, sz};
    ConeVoxView &V = out[i];
    for (int j = 0; j < 3; ++j) {
      V.a[j] = (float)((P[j] - cu * P[8 + j]) * s[j]);
      V.b[j] = (float)((P[4 + j] - cv * P[8 + j]) * s[j]);
      V.w[j] = (float)(P[8 + j] * s[j]);
    }
    V.a[3] = (float)(P[3] - cu * P[11]);
    V.b[3] = (float)(P[7] - cv * P[11]);
    V.w[3] = (float)P[11];
    if (V.a[2] != 0.f || V.w[2] != 0.f) zinv = false;
  }
}

// Back-projector algorithm: TK_BP_ALGO = tma (default) | quad | tex | hwtex.
// tma needs a z-invariant trajectory and a detector width that is a multiple of
// 4 (16-byte TMA row pitch); otherwise quad runs.
enum class BpAlgo { kTma, kQuad, kTex, kHwTex };

static BpAlgo bp_algo() {
  const char *e = getenv("TK_BP_ALGO");
  if (e && !strcmp(e, "quad")) return BpAlgo::kQuad;
  if (e && !strcmp(e, "tex")) return BpAlgo::kTex;
  if (e && !strcmp(e, "hwtex")) return BpAlgo::kHwTex;
  return BpAlgo::kTma;
}

constexpr int kBqZB = 16;

static int launch_bp_quad(BpParams p, bool weighted, bool zinv, cudaStream_t st) {
  const long long qview = (long long)(p.band_rows + 1 + kQuadPad) * (p.cols + 1 + kQuadPad);
  const long long nq = qview * p.n_views;
  Scratch quads;
  TK_TRY_CUDA(quads.alloc(sizeof(float4) * nq, st));
  const unsigned qgrid = (unsigned)std::min<long long>(ceil_div(nq, 256), (long long)sm_count() * 32);
  quadify_kernel<<<qgrid, 256, 0, st>>>(p.sino, p.n_views, p.band_rows, p.cols, quads.as<float4>());
  TK_LAUNCHED("quadify_kernel");
  dim3 block(kBqBX, kBqBY);
  dim3 grid(ceil_div(p.nx, kBqBX), ceil_div(p.ny, kBqBY), ceil_div(p.z_count, kBqZB));
  const float4 *q = quads.as<float4>();
  const int sel = (zinv ? 2 : 0) + (weighted ? 1 : 0);
  if (sel == 3) cone_bp_quad_kernel<kBqZB, true, true><<<grid, block, 0, st>>>(p, q);
  else if (sel == 2) cone_bp_quad_kernel<kBqZB, true, false><<<grid, block, 0, st>>>(p, q);
  else if (sel == 1) cone_bp_quad_kernel<kBqZB, false, true><<<grid, block, 0, st>>>(p, q);
  else cone_bp_quad_kernel<kBqZB, false, false><<<grid, block, 0, st>>>(p, q);
  TK_LAUNCHED("cone_bp_quad_kernel");
  return TK_OK;
}

template <int ZB, bool ZINV>
static void launch_bp_tex_t(const BpParams &p, bool weighted, bool hw, dim3 grid, dim3 block, cudaStream_t st) {
  if (hw) {
    if (weighted)
      cone_bp_tex_kernel<ZB, ZINV, true, true><<<grid, block, 0, st>>>(p);
    else
      cone_bp_tex_kernel<ZB, ZINV, false, true><<<grid, block, 0, st>>>(p);
  } else if (weighted) {
    cone_bp_tex_kernel<ZB, ZINV, true, false><<<grid, block, 0, st>>>(p);
  } else {
    cone_bp_tex_kernel<ZB, ZINV, false, false><<<grid, block, 0, st>>>(p);
  }
}

}  // namespace tk

using namespace tk;

extern "C" {

int tk_back_cone_3d_ex(const float *sino, int n_views, int rows, int cols, int row_begin,
                       int band_rows, const double *mats, double sid, int weighted, int nz,
                       int ny, int nx, double sz, double sy, double sx, int z_begin,
                       int z_count, int accumulate, float *out, void *stream) {
  clear_error();
  if (!sino || !out || !mats) return fail_arg("tk_back_cone_3d: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_back_cone_3d: non-positive extent");
  if (band_rows < 1 || row_begin < 0 || row_begin + band_rows > rows)
    return fail_arg("tk_back_cone_3d: row band outside the detector");
  if (z_count < 1 || z_begin < 0 || z_begin + z_count > nz)
    return fail_arg("tk_back_cone_3d: z range outside the volume");
  if (!(sx > 0 && sy > 0 && sz > 0)) return fail_arg("tk_back_cone_3d: spacing must be > 0");
  cudaStream_t st = as_stream(stream);
  const double cu = (cols - 1) / 2.0, cv = (rows - 1) / 2.0;
  std::vector<ConeVoxView> hv;
  bool zinv = true;
  pack_bp_views(mats, n_views, sx, sy, sz, cu, cv, hv, zinv);
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeVoxView) * n_views, st));
  BpParams p;
  p.sino = sino;
  p.view_stride = (long long)band_rows * cols;
  p.n_views = n_views;
  p.band_rows = band_rows;
  p.cols = cols;
  p.views = dviews.as<ConeVoxView>();
  p.cu = (float)cu;
  p.cv = (float)(cv - row_begin);
  p.sid = (float)sid;
  p.nx = nx;
  p.ny = ny;
  p.z_begin = z_begin;
  p.z_count = z_count;
  p.cx = (float)((nx - 1) / 2.0);
  p.cy = (float)((ny - 1) / 2.0);
  p.cz = (float)((nz - 1) / 2.0);
  p.accumulate = accumulate;
  p.out = out;
  p.tex = 0;
  BpAlgo algo = bp_algo();
  if (algo == BpAlgo::kTma && zinv) {
    const int rc = launch_bp_tma(p, hv.data(), weighted != 0, st);
    if (rc != -1) return rc;
  }
  if (algo == BpAlgo::kTma || algo == BpAlgo::kQuad || n_views > 2048)  // layered arrays hold <= 2048 layers
    return launch_bp_quad(p, weighted != 0, zinv, st);
  constexpr int ZB = 8;
  dim3 block(kBpBX, kBpBY);
  dim3 grid(ceil_div(nx, kBpBX), ceil_div(ny, kBpBY), ceil_div(z_count, ZB));
  TexLease lease;
  const bool hw = algo == BpAlgo::kHwTex;
  TK_TRY_CUDA(tex_acquire(sino, cols, band_rows, n_views, hw ? TexKind::kLayeredLinear : TexKind::kLayeredPoint, st,
                          lease));
  p.tex = lease.tex;
  if (zinv)
    launch_bp_tex_t<ZB, true>(p, weighted != 0, hw, grid, block, st);
  else
    launch_bp_tex_t<ZB, false>(p, weighted != 0, hw, grid, block, st);
  tex_release(lease, st);
  TK_LAUNCHED("cone_bp_tex_kernel");
  return TK_OK;
}

int tk_back_cone_3d(const float *sino, int n_views, int rows, int cols, const double *mats,
                    double sid, int weighted, int nz, int ny, int nx, double sz, double sy,
                    double sx, float *out, void *stream) {
  return tk_back_cone_3d_ex(sino, n_views, rows, cols, 0, rows, mats, sid, weighted, nz, ny,
                            nx, sz, sy, sx, 0, nz, 0, out, stream);
}

int tk_back_cone_3d_adjoint(const float *vol, int nz, int ny, int nx, double sz, double sy,
                            double sx, const double *mats, double sid, int weighted,
                            int n_views, int rows, int cols, float *sino_out, void *stream) {
  clear_error();
  if (!vol || !sino_out || !mats) return fail_arg("tk_back_cone_3d_adjoint: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_back_cone_3d_adjoint: non-positive extent");
  cudaStream_t st = as_stream(stream);
  const double cu = (cols - 1) / 2.0, cv = (rows - 1) / 2.0;
  std::vector<ConeVoxView> hv;
  bool zinv = true;
  pack_bp_views(mats, n_views, sx, sy, sz, cu, cv, hv, zinv);
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeVoxView) * n_views, st));
  const long long nvox = (long long)nx * ny * nz;
  Scratch qs;
  const size_t nq = (size_t)n_views * (rows + 1) * (cols + 1);
  TK_TRY_CUDA(qs.alloc(sizeof(float4) * nq, st));
  TK_TRY_CUDA(cudaMemsetAsync(qs.ptr, 0, sizeof(float4) * nq, st));
  for (int v0 = 0; v0 < n_views; v0 += 65535) {  // views on gridDim.y
    const dim3 grid(ceil_div(nvox, 256), std::min(65535, n_views - v0));
    cone_bp_adjoint4_kernel<<<grid, 256, 0, st>>>(vol, nx, ny, nz, (float)((nx - 1) / 2.0), (float)((ny - 1) / 2.0),
                                                  (float)((nz - 1) / 2.0), dviews.as<ConeVoxView>() + v0, rows, cols,
                                                  (float)cu, (float)cv, (float)sid, weighted,
                                                  qs.as<float4>() + (size_t)v0 * (rows + 1) * (cols + 1));
    TK_LAUNCHED("cone_bp_adjoint4_kernel");
  }
  const long long npix = (long long)n_views * rows * cols;
  unquad_det_kernel<<<(unsigned)std::min<long long>(ceil_div(npix, 256), (long long)sm_count() * 16), 256, 0, st>>>(
      qs.as<float4>(), n_views, rows, cols, sino_out);
  TK_LAUNCHED("unquad_det_kernel");
  return TK_OK;
}

}  // extern "C"
