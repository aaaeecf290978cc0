// tk_cone.cu -- cone-beam 3D forward (ray-driven) and back (voxel-driven)
// projectors for sm_100a, plus their exact transposes (matched adjoints).
//
// Semantics follow the reference kernels line for line
// (/root/reference/pkg/src/tomokit/_kernels.py:117-157, 254-322); the
// arithmetic is reorganised for the GPU:
//   * forward: per-ray set-up (direction M^-1 (c,r,1), normalisation, slab
//     clipping, sample count) in float64; the march itself in float32 in
//     padded-index space, sample k at  e + (k + 1/2) * g  computed directly
//     (no accumulated t), exact last partial segment.
//   * back: projection-matrix rows are pre-multiplied by the voxel spacing,
//     shifted by the detector centre (principal-point shift keeps fp32 well
//     conditioned), and evaluated on centred integer voxel coordinates.  For
//     trajectories whose detector column/depth rows have no z component
//     (circular, helical, sinusoidal orbits with v = +z) the column, depth and
//     distance weight are computed once per (x,y,view) and reused by ZB voxels
//     along z; only the row coordinate advances.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tk_common.cuh"
#include "tk_cone_bp.cuh"
#include "tk_cone_fp.cuh"
#include "tk_tex.cuh"

namespace tk {

// ---------------------------------------------------------------------------
// zero-padded copy: volp (nz+2, ny+2, nx+2)  <-  vol (nz, ny, nx)
// (reference projectors.py:26-29)
// ---------------------------------------------------------------------------
__global__ void pad3d_kernel(const float *__restrict__ vol, int nz, int ny, int nx,
                             float *__restrict__ volp) {
  const int nxp = nx + 2, nyp = ny + 2, nzp = nz + 2;
  const long long total = (long long)nzp * nyp * nxp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int x = (int)(i % nxp);
    long long t = i / nxp;
    int y = (int)(t % nyp);
    int z = (int)(t / nyp);
    float v = 0.f;
    if (x >= 1 && x <= nx && y >= 1 && y <= ny && z >= 1 && z <= nz)
      v = __ldg(vol + ((long long)(z - 1) * ny + (y - 1)) * nx + (x - 1));
    volp[i] = v;
  }
}

// crop a padded fp32 volume back to (nz, ny, nx)
__global__ void crop3d_kernel(const float *__restrict__ volp, int nz, int ny, int nx,
                              float *__restrict__ vol) {
  const long long total = (long long)nz * ny * nx;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int x = (int)(i % nx);
    long long t = i / nx;
    int y = (int)(t % ny);
    int z = (int)(t / ny);
    vol[i] = volp[((long long)(z + 1) * (ny + 2) + (y + 1)) * (nx + 2) + (x + 1)];
  }
}

// One trilinear sample of the zero-padded volume at padded-index coordinates
// (_kernels.py:141-154).  Returns 0 outside 0 <= i < n+1.
__device__ __forceinline__ float trilinear_padded(const float *__restrict__ volp, int nxp,
                                                  int nyp, int nzp, float fx, float fy,
                                                  float fz) {
  const float flx = floorf(fx), fly = floorf(fy), flz = floorf(fz);
  const int ix = (int)flx, iy = (int)fly, iz = (int)flz;
  if ((unsigned)ix >= (unsigned)(nxp - 1) || (unsigned)iy >= (unsigned)(nyp - 1) ||
      (unsigned)iz >= (unsigned)(nzp - 1))
    return 0.f;
  const float wx = fx - flx, wy = fy - fly, wz = fz - flz;
  const unsigned sxy = (unsigned)nyp * (unsigned)nxp;
  const float *p = volp + ((unsigned)iz * sxy + (unsigned)iy * (unsigned)nxp + (unsigned)ix);
  const float *q = p + sxy;
  const float v00 = lerpf(__ldg(p), __ldg(p + 1), wx);
  const float v01 = lerpf(__ldg(p + nxp), __ldg(p + nxp + 1), wx);
  const float v10 = lerpf(__ldg(q), __ldg(q + 1), wx);
  const float v11 = lerpf(__ldg(q + nxp), __ldg(q + nxp + 1), wx);
  return lerpf(lerpf(v00, v01, wy), lerpf(v10, v11, wy), wz);
}

// ---------------------------------------------------------------------------
// Forward projection: one thread per detector pixel; a warp covers an 8x4
// pixel tile so its rays sample a compact patch of the volume at each step.
// ---------------------------------------------------------------------------
constexpr int kFpBX = 8, kFpBY = 16;

__global__ void __launch_bounds__(kFpBX *kFpBY)
    cone_fp_kernel(const float *__restrict__ volp, int nx, int ny, int nz, double sx,
                   double sy, double sz, const ConeRayView *__restrict__ views, int rows,
                   int cols, double step, float *__restrict__ out) {
  const int c = blockIdx.x * kFpBX + threadIdx.x;
  const int r = blockIdx.y * kFpBY + threadIdx.y;
  const int v = blockIdx.z;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const ConeRayView V = views[v];
  RaySetup rs;
  if (!cone_ray_setup(V, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  const int nxp = nx + 2, nyp = ny + 2, nzp = nz + 2;
  float acc = 0.f;
  const int nfull = rs.n - 1;
  for (int k = 0; k < nfull; ++k) {
    const float kf = (float)k + 0.5f;
    acc += trilinear_padded(volp, nxp, nyp, nzp, fmaf(kf, rs.gx, rs.ex),
                            fmaf(kf, rs.gy, rs.ey), fmaf(kf, rs.gz, rs.ez));
  }
  {  // last (possibly partial) segment, midpoint at t + seg/2
    const float kf = (float)nfull + 0.5f * rs.last;
    acc += rs.last * trilinear_padded(volp, nxp, nyp, nzp, fmaf(kf, rs.gx, rs.ex),
                                      fmaf(kf, rs.gy, rs.ey), fmaf(kf, rs.gz, rs.ez));
  }
  *dst = acc * (float)step;
}

// ---------------------------------------------------------------------------
// Forward projection, orientation-matched LDG variant ("ldg2", default).
//
// * The volume is kept with a TWO-voxel zero margin in two orientations: x
//   fastest (A) and y fastest (B, x/y exchanged).  Each view uses the copy
//   whose fastest axis is most aligned with the detector u direction, and a
//   warp covers 32 consecutive detector columns, so the 32 rays' samples at a
//   step lie along the fast axis and each tap load touches one or two lines.
// * With the 2-voxel margin every cell a sample can reach (inside the clip
//   box up to float32 rounding) is addressable and its out-of-volume taps read
//   zero, which IS the reference's zero-extended interpolant -- no per-sample
//   range test, no clamping.
// * A thread keeps the taps of its current cell (and their differences along
//   the fast axis) in registers; a sample that stays in the same cell (about
//   half of them at step = s/2) issues no load.
// ---------------------------------------------------------------------------
constexpr int kFp2BX = 32, kFp2BY = 4;

// vol (nz, ny, nx) -> copy with a kFpMargin zero margin; swap_xy selects the
// y-fastest orientation out[z][x][y].  Tiled through shared memory so both
// the read and the (possibly transposed) write are coalesced.
__global__ void pad_margin_kernel(const float *__restrict__ vol, int nz, int ny, int nx, int swap_xy,
                                  float *__restrict__ out) {
  __shared__ float tile[32][33];
  constexpr int m = kFpMargin;
  const int nxp = nx + 2 * m, nyp = ny + 2 * m;
  const int z = blockIdx.z;  // padded z
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const bool zin = z >= m && z < nz + m;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int y = y0 + j, x = x0 + threadIdx.x;  // padded coordinates
    float v = 0.f;
    if (zin && y >= m && y < ny + m && x >= m && x < nx + m)
      v = __ldg(vol + ((long long)(z - m) * ny + (y - m)) * nx + (x - m));
    tile[j][threadIdx.x] = v;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    if (swap_xy) {
      const int x = x0 + j, y = y0 + threadIdx.x;
      if (x < nxp && y < nyp) out[((long long)z * nxp + x) * nyp + y] = tile[threadIdx.x][j];
    } else {
      const int y = y0 + j, x = x0 + threadIdx.x;
      if (x < nxp && y < nyp) out[((long long)z * nyp + y) * nxp + x] = tile[j][threadIdx.x];
    }
  }
}

struct CellTaps {  // the 8 taps of one cell: v[z][b][a], with d = v[..][1] - v[..][0]
  float v00, d00, v01, d01, v10, d10, v11, d11;
};

__device__ __forceinline__ void load_cell(const float *__restrict__ p, int pa, int ps, CellTaps &t) {
  const float a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + pa), d = __ldg(p + pa + 1);
  const float e = __ldg(p + ps), f = __ldg(p + ps + 1), g = __ldg(p + ps + pa),
              h = __ldg(p + ps + pa + 1);
  t.v00 = a;
  t.d00 = b - a;
  t.v01 = c;
  t.d01 = d - c;
  t.v10 = e;
  t.d10 = f - e;
  t.v11 = g;
  t.d11 = h - g;
}

__device__ __forceinline__ float interp_cell(const CellTaps &t, float wa, float wb, float wz) {
  const float a0 = fmaf(wa, t.d00, t.v00), a1 = fmaf(wa, t.d01, t.v01);
  const float b0 = fmaf(wa, t.d10, t.v10), b1 = fmaf(wa, t.d11, t.v11);
  const float lo = fmaf(wb, a1 - a0, a0), hi = fmaf(wb, b1 - b0, b0);
  return fmaf(wz, hi - lo, lo);
}

template <int MINB>
__global__ void __launch_bounds__(kFp2BX *kFp2BY, MINB)
    cone_fp2_kernel(const float *__restrict__ volA, const float *__restrict__ volB, int nx, int ny,
                    int nz, double sx, double sy, double sz, const Fp2View *__restrict__ views,
                    int rows, int cols, int n_views, double step, float *__restrict__ out) {
  // 1D grid, view-major within a detector row band: consecutive CTAs cover the
  // same rows of successive views, so the CTAs resident at any time sample the
  // same thin z-slab of the volume (which then stays in L2 across views).
  const int ncb = (cols + kFp2BX - 1) / kFp2BX;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int c = cb * kFp2BX + threadIdx.x;
  const int r = rb * kFp2BY + threadIdx.y;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  // fast axis "a", middle axis "b": (x, y) for copy A, (y, x) for copy B.
  // rs.e* are one-voxel-padded coordinates; the copies carry a 2-voxel margin.
  const float *vol = W.swap ? volB : volA;
  const int na = W.swap ? ny : nx, nb = W.swap ? nx : ny;
  const float ea = (W.swap ? rs.ey : rs.ex) + (kFpMargin - 1);
  const float eb = (W.swap ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = W.swap ? rs.gy : rs.gx, gb = W.swap ? rs.gx : rs.gy, gz = rs.gz;
  const int pa = na + 2 * kFpMargin;        // padded row pitch
  const int ps = (nb + 2 * kFpMargin) * pa;  // padded slice pitch
  int cell = -1;
  CellTaps t = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float acc = 0.f;
  float kf = 0.5f;
  const int nfull = rs.n - 1;
  for (int k = 0; k < nfull; ++k, kf += 1.f) {
    const float fa = fmaf(kf, ga, ea), fb = fmaf(kf, gb, eb), fz = fmaf(kf, gz, ez);
    const float la = floorf(fa), lb = floorf(fb), lz = floorf(fz);
    const int id = (int)lz * ps + (int)lb * pa + (int)la;
    if (id != cell) {
      cell = id;
      load_cell(vol + id, pa, ps, t);
    }
    acc += interp_cell(t, fa - la, fb - lb, fz - lz);
  }
  {  // last (possibly partial) segment: midpoint at t + seg/2, weight seg/step
    kf = (float)nfull + 0.5f * rs.last;
    const float fa = fmaf(kf, ga, ea), fb = fmaf(kf, gb, eb), fz = fmaf(kf, gz, ez);
    const float la = floorf(fa), lb = floorf(fb), lz = floorf(fz);
    const int id = (int)lz * ps + (int)lb * pa + (int)la;
    if (id != cell) load_cell(vol + id, pa, ps, t);
    acc = fmaf(rs.last, interp_cell(t, fa - la, fb - lb, fz - lz), acc);
  }
  *dst = acc * (float)step;
}

// ---------------------------------------------------------------------------
// Forward projection, quad-tap variant ("ldg4", default).
//
// The ncu capture of cone_fp2_kernel shows the L1 tag stage (output
// wavefronts, ~80% of peak) as the limit: 8 scalar loads per cell, each
// touching 2-3 lines.  Here every margin-padded cell (z, b, a) of the
// orientation copy stores its four in-slice taps as one float4
//   Q[z][b][a] = (V[z][b][a], V[z][b][a+1], V[z][b+1][a], V[z][b+1][a+1]),
// so a cell is 2 LDG.128 (slices z and z+1) instead of 8 LDG.32.
// Same traversal, ordering, arithmetic order of weights as cone_fp2_kernel.
// ---------------------------------------------------------------------------
// Tap quads of the orientation copies: every margin-padded cell (z, b, a) stores
// Q[z][b][a] = (V[z][b][a], V[z][b][a+1], V[z][b+1][a], V[z][b+1][a+1]); diff = 1
// stores (v00, v01 - v00, v10, v11 - v10) (fast-axis differences pre-subtracted:
// the sample's fast-axis lerps become single FFMAs with the same fp32 rounding as
// fmaf(w, b - a, a), i.e. bit-identical results).
// Built tiled through shared memory: a 32 (a) x 32 (b) tile of cells needs a
// 33 x 33 tap patch, read along x (coalesced) and written along a (coalesced);
// a per-cell gather reads the y-fastest copy (SWAP) with a stride of nx floats
// (1.97 ms at 512^3 -> 0.60 ms tiled).
template <bool SWAP>
__global__ void __launch_bounds__(256) quad_volume_tiled_kernel(const float *__restrict__ vol, int nz, int ny,
                                                                int nx, float4 *__restrict__ q, int diff) {
  __shared__ float tile[33][34];  // [a - a0][b - b0]
  constexpr int m = kFpMargin;
  const int na = SWAP ? ny : nx, nb = SWAP ? nx : ny;
  const int pa = na + 2 * m, pb = nb + 2 * m;
  const int a0 = blockIdx.x * 32 - m, b0 = blockIdx.y * 32 - m, z = (int)blockIdx.z - m;
  const bool zin = (unsigned)z < (unsigned)nz;
  for (int e = threadIdx.x; e < 33 * 33; e += 256) {
    // consecutive threads read consecutive x: x = b for SWAP, x = a otherwise
    const int da = SWAP ? e / 33 : e % 33, db = SWAP ? e % 33 : e / 33;
    const int a = a0 + da, b = b0 + db;
    const int x = SWAP ? b : a, y = SWAP ? a : b;
    float val = 0.f;
    if (zin && (unsigned)y < (unsigned)ny && (unsigned)x < (unsigned)nx)
      val = __ldg(vol + ((long long)z * ny + y) * nx + x);
    tile[da][db] = val;
  }
  __syncthreads();
  const int ta = threadIdx.x & 31;
  for (int tb = threadIdx.x >> 5; tb < 32; tb += 8) {
    const int a = a0 + ta, b = b0 + tb;  // cell (z, b, a) of the copy
    if (a + m >= pa || b + m >= pb) continue;
    const float v0 = tile[ta][tb], v1 = tile[ta + 1][tb], v2 = tile[ta][tb + 1], v3 = tile[ta + 1][tb + 1];
    q[((long long)(z + m) * pb + (b + m)) * pa + (a + m)] =
        diff ? make_float4(v0, v1 - v0, v2, v3 - v2) : make_float4(v0, v1, v2, v3);
  }
}

// WR = detector rows per warp: lane l takes row l % WR, column l / WR, so a
// quarter-warp (8 lanes) spans min(WR, 8) rows of one to eight columns.  Rays of
// one column march through the same (a, b) cells in near lock-step (they
// differ only in z), so with WR > 1 the cell changes of a quarter coincide.
template <int MINB, bool MAGIC, int WR = 1>
__global__ void __launch_bounds__(kFp2BX *kFp2BY, MINB)
    cone_fp4_kernel(const float4 *__restrict__ qA, const float4 *__restrict__ qB, int nx, int ny,
                    int nz, double sx, double sy, double sz, const Fp2View *__restrict__ views,
                    int rows, int cols, int n_views, double step, float *__restrict__ out) {
  constexpr int kCols = WR == 1 ? kFp2BX : kFp2BX * kFp2BY / WR;  // columns per CTA
  const int ncb = (cols + kCols - 1) / kCols;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int lane = threadIdx.x, warp = threadIdx.y;  // blockDim = (32, 4)
  const int c = WR == 1 ? cb * kFp2BX + lane : cb * kCols + warp * (32 / WR) + lane / WR;
  const int r = WR == 1 ? rb * kFp2BY + warp : rb * WR + lane % WR;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  // Orientation copy per ray (W.face_copy) or per view.  At march step k the
  // sample points of neighbouring rays lie on a plane parallel to the box face
  // the rays entered through (same t - t0), so a ray that entered through an
  // x face has its neighbours spread along y: the y-fastest copy keeps a
  // quarter-warp's taps in one or two 128-byte lines, the x-fastest copy would
  // put every lane in a different line.  Rays entering through a z face spread
  // along the detector u direction (the per-view choice).
  const int swap = W.face_copy ? (rs.face == 0 ? 1 : (rs.face == 1 ? 0 : W.swap)) : W.swap;
  const float4 *q = swap ? qB : qA;
  const int na = swap ? ny : nx, nb = swap ? nx : ny;
  const float ea = (swap ? rs.ey : rs.ex) + (kFpMargin - 1);
  const float eb = (swap ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = swap ? rs.gy : rs.gx, gb = swap ? rs.gx : rs.gy, gz = rs.gz;
  const int pa = na + 2 * kFpMargin;
  const int ps = (nb + 2 * kFpMargin) * pa;
  const float paf = (float)pa;
  int cell = -1;
  float4 lo4 = make_float4(0.f, 0.f, 0.f, 0.f), hi4 = lo4;
  // one trilinear sample at march parameter kk (in steps); the in-slice part
  // of the cell index, lb * pa + la < 2^24, is formed exactly in float
  const unsigned bias = kFloorBits * (1u + (unsigned)pa + (unsigned)ps);
  auto sample = [&](float kk) -> float {
    const float fa = fmaf(kk, ga, ea), fb = fmaf(kk, gb, eb), fz = fmaf(kk, gz, ez);
    float la, lb, lz;
    int id;
    if (MAGIC) {  // floor via FADD.RM (no conversion-pipe instructions), index from the float bits
      const float xa = floor_magic(fa), xb = floor_magic(fb), xz = floor_magic(fz);
      id = (int)(__float_as_uint(xz) * (unsigned)ps + (__float_as_uint(xb) * (unsigned)pa + __float_as_uint(xa)));
      la = xa - kFloorMagic;
      lb = xb - kFloorMagic;
      lz = xz - kFloorMagic;
    } else {
      la = floorf(fa);
      lb = floorf(fb);
      lz = floorf(fz);
      id = __float2int_rz(lz) * ps + __float2int_rz(fmaf(lb, paf, la));
    }
    if (id != cell) {
      cell = id;
      const float4 *p = MAGIC ? elem_ptr(q, (unsigned)id - bias) : q + id;
      lo4 = __ldg(p);
      hi4 = __ldg(p + ps);
    }
    const float wa = fa - la, wb = fb - lb;
    if (MAGIC) {  // difference quads (quad_volume_tiled_kernel diff = 1)
      const float s0 = lerpf(fmaf(wa, lo4.y, lo4.x), fmaf(wa, lo4.w, lo4.z), wb);
      const float s1 = lerpf(fmaf(wa, hi4.y, hi4.x), fmaf(wa, hi4.w, hi4.z), wb);
      return lerpf(s0, s1, fz - lz);
    }
    const float s0 = lerpf(lerpf(lo4.x, lo4.y, wa), lerpf(lo4.z, lo4.w, wa), wb);
    const float s1 = lerpf(lerpf(hi4.x, hi4.y, wa), lerpf(hi4.z, hi4.w, wa), wb);
    return lerpf(s0, s1, fz - lz);
  };
  float acc = 0.f;
  float kf = 0.5f;
  const int nfull = rs.n - 1;
#pragma unroll 2
  for (int k = 0; k < nfull; ++k, kf += 1.f) acc += sample(kf);
  acc = fmaf(rs.last, sample((float)nfull + 0.5f * rs.last), acc);  // exact last segment
  *dst = acc * (float)step;
}

// ---------------------------------------------------------------------------
// Forward projection, z-fastest quad variant ("ldg4z").
//
// A load instruction costs one L1 data-pipe wavefront per 128-byte line per
// ACTIVE quarter-warp (8 lanes); a quarter whose lanes all stay in their cells
// costs nothing (loading unconditionally measured 2.2x slower).  With 8
// adjacent columns of one row per quarter, every lane crosses cell boundaries
// along the volume axis that follows the detector u direction at its own steps,
// so nearly every quarter is active at every step.  Here a quarter is 8
// consecutive ROWS of one column: their rays lie in one vertical plane through
// the source and share the horizontal track, so their x / y cell crossings
// coincide and only z crossings (|gz| <= ~0.12 cell per step at cfg4) are per
// lane.  The taps are stored z-fastest so the quarter's ~6 consecutive z cells
// are contiguous:  Qz[y][x][z] = (V[z][y][x], V[z][y][x+1] - V[z][y][x],
// V[z+1][y][x], V[z+1][y][x+1] - V[z+1][y][x])  (margin-padded), a cell is
// Qz[y][x][z] and Qz[y+1][x][z].  One copy serves every view.
// ---------------------------------------------------------------------------
// 32 (z) x 32 (x) tiles of one y row: reads along x, writes along z (coalesced).
__global__ void __launch_bounds__(256) quad_volume_z_kernel(const float *__restrict__ vol, int nz, int ny, int nx,
                                                            float4 *__restrict__ q) {
  __shared__ float tile[33][34];  // [x - x0][z - z0]
  constexpr int m = kFpMargin;
  const int pz = nz + 2 * m, px = nx + 2 * m;
  const int z0 = blockIdx.x * 32 - m, x0 = blockIdx.y * 32 - m, y = (int)blockIdx.z - m;
  const bool yin = (unsigned)y < (unsigned)ny;
  for (int e = threadIdx.x; e < 33 * 33; e += 256) {
    const int dx = e % 33, dz = e / 33;
    const int x = x0 + dx, z = z0 + dz;
    float val = 0.f;
    if (yin && (unsigned)z < (unsigned)nz && (unsigned)x < (unsigned)nx)
      val = __ldg(vol + ((long long)z * ny + y) * nx + x);
    tile[dx][dz] = val;
  }
  __syncthreads();
  const int tz = threadIdx.x & 31;
  for (int tx = threadIdx.x >> 5; tx < 32; tx += 8) {
    const int z = z0 + tz, x = x0 + tx;  // cell (z, y, x) of the padded grid
    if (z + m >= pz || x + m >= px) continue;
    const float v00 = tile[tx][tz], v01 = tile[tx + 1][tz], v10 = tile[tx][tz + 1], v11 = tile[tx + 1][tz + 1];
    q[((long long)(y + m) * px + (x + m)) * pz + (z + m)] = make_float4(v00, v01 - v00, v10, v11 - v10);
  }
}

// Coefficient form ("ldg4z", default): each cell of row y stores the bilinear
// (x, z) polynomial of its taps,  Cz[y][x][z] = (A, B, C, D) with A = V00,
// B = V01 - V00, C = V10 - V00, D = (V11 - V10) - (V01 - V00)  (V_zx of row y),
// so a row is  P = fma(wz, fma(wx, D, C), fma(wx, B, A))  (3 FFMA instead of 4
// FFMA + FADD) and a sample is lerp(P(Cz[y]), P(Cz[y+1]), wy).  (A second array
// of y differences, s = P(C) + wy P(dC), saves one more FADD but loses the L1
// sharing between a cell's y+1 row and the next cell's y row: measured 776 ms
// vs 489 ms.)
__global__ void __launch_bounds__(256) coef_volume_z_kernel(const float *__restrict__ vol, int nz, int ny, int nx,
                                                            float4 *__restrict__ cq, int zpitch, long long ystride,
                                                            int acbd) {
  __shared__ float tile[33][34];  // [x - x0][z - z0]
  constexpr int m = kFpMargin;
  const int pz = nz + 2 * m, px = nx + 2 * m;
  const int z0 = blockIdx.x * 32 - m, x0 = blockIdx.y * 32 - m, y = (int)blockIdx.z - m;
  const bool yin = (unsigned)y < (unsigned)ny;
  for (int e = threadIdx.x; e < 33 * 33; e += 256) {
    const int dx = e % 33, dz = e / 33;
    const int x = x0 + dx, z = z0 + dz;
    float val = 0.f;
    if (yin && (unsigned)z < (unsigned)nz && (unsigned)x < (unsigned)nx)
      val = __ldg(vol + ((long long)z * ny + y) * nx + x);
    tile[dx][dz] = val;
  }
  __syncthreads();
  const int tz = threadIdx.x & 31;
  for (int tx = threadIdx.x >> 5; tx < 32; tx += 8) {
    const int z = z0 + tz, x = x0 + tx;  // cell (z, y, x) of the padded grid
    if (z + m >= pz || x + m >= px) continue;
    const float v00 = tile[tx][tz], v01 = tile[tx + 1][tz], v10 = tile[tx][tz + 1], v11 = tile[tx + 1][tz + 1];
    const float A = v00, B = v01 - v00, C = v10 - v00, D = (v11 - v10) - (v01 - v00);
    // acbd: (A, C, B, D) so that (A, C) and (B, D) are register pairs for FFMA2
    cq[(long long)(y + m) * ystride + (long long)(x + m) * zpitch + (z + m)] =
        acbd ? make_float4(A, C, B, D) : make_float4(A, B, C, D);
  }
}

constexpr int kFpzRows = 8;  // rows per quarter-warp group (one column)
// RB = detector rows per CTA band (8, 16 or 32): the CTA's 16 quarter-warps
// cover (128 / RB) columns x RB rows, each quarter 8 consecutive rows of one column.
// VG > 1: one CTA = VG sub-blocks of 128 threads on the SAME detector tile of VG
// consecutive views (their rays are the previous view's rotated by 2pi/V about
// the axis, so near the axis they sample the same cells: L1 sharing on one SM).
// FIXS: the y stride is the compile-time constant kFpFixS (cells), so the far
// row's load is the near row's address + an immediate offset (kFpFixS * 16 B
// fits LDG's signed 24-bit offset): no 64-bit add per load.
constexpr unsigned kFpFixS = 524032u;  // 2047 * 256 cells: z pitch must be == 255 (mod 256)
template <int MINB, bool COEF, int RB = 8, int VG = 1, bool FIXS = false, bool F2 = false>
__global__ void __launch_bounds__(128 * VG, (MINB + VG - 1) / VG)
    cone_fp4z_kernel(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy, double sz,
                     const Fp2View *__restrict__ views, int rows, int cols, int n_views, double step,
                     float *__restrict__ out, unsigned zpitch, unsigned ystride) {
  // view-major order within RB-row bands
  constexpr int kCols = 128 / RB, kQpc = RB / kFpzRows;  // columns per CTA, quarters per column
  const int ncb = (cols + kCols - 1) / kCols;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int nvg = (n_views + VG - 1) / VG;
  const int v = (int)(bt % nvg) * VG + (int)(threadIdx.x >> 7);
  const int rb = (int)(bt / nvg);
  const int t = threadIdx.x & 127;
  const int qd = t >> 3;  // quarter-warp index in the sub-block
  const int c = cb * kCols + qd / kQpc;
  const int r = rb * RB + (qd % kQpc) * kFpzRows + (t & 7);
  if (c >= cols || r >= rows || v >= n_views) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  const float ex = rs.ex + (kFpMargin - 1), ey = rs.ey + (kFpMargin - 1), ez = rs.ez + (kFpMargin - 1);
  const float gx = rs.gx, gy = rs.gy, gz = rs.gz;
  // COEF layouts use zpitch / xpitch chosen on the host so that the floor bias
  // 0x4B000000 * (1 + zpitch + xpitch * zpitch) vanishes modulo 2^32: the cell
  // index formed from the FADD.RM float bits IS the element index (one
  // IMAD.WIDE per address instead of IADD + LEA + LEA.HI.X).  Coordinates are
  // >= 0 here, so floor(f) = bits(f + 2^23) - 0x4B000000.
  const float magic = COEF ? 8388608.f : kFloorMagic;
  const unsigned sxs = zpitch, sys = FIXS ? kFpFixS : ystride;  // x and y strides (cells)
  const unsigned bias = COEF ? 0u : kFloorBits * (1u + sxs + sys);
  unsigned cell = 0xffffffffu;
  float4 lo4 = make_float4(0.f, 0.f, 0.f, 0.f), hi4 = lo4;
  const unsigned long long e2 = pk2(ex, ey), g2 = pk2(gx, gy), m2 = pk2(magic, magic);
  auto sample = [&](float kk) -> float {
    if (F2) {  // (x, y) as FFMA2 / FADD2 pairs; cells stored (A, C, B, D); bit-identical results
      const unsigned long long fxy = ffma2(pk2(kk, kk), g2, e2);
      const float fz = fmaf(kk, gz, ez);
      const unsigned long long xxy = fadd2_rm(fxy, m2);
      const float xz = __fadd_rd(fz, magic);
      const float2 xb = upk2(xxy);
      const unsigned id = __float_as_uint(xb.y) * sys + (__float_as_uint(xb.x) * sxs + __float_as_uint(xz));
      if (id != cell) {
        cell = id;
        const float4 *p = elem_ptr(q, id - bias);
        lo4 = __ldg(p);
        hi4 = __ldg(p + sys);
      }
      const float2 w = upk2(fsub2(fxy, fsub2(xxy, m2)));
      const float wz = fz - (xz - magic);
      const float2 tl = upk2(ffma2(pk2(lo4.z, lo4.w), pk2(w.x, w.x), pk2(lo4.x, lo4.y)));
      const float2 th = upk2(ffma2(pk2(hi4.z, hi4.w), pk2(w.x, w.x), pk2(hi4.x, hi4.y)));
      const float s0 = fmaf(wz, tl.y, tl.x), s1 = fmaf(wz, th.y, th.x);
      return lerpf(s0, s1, w.y);
    }
    const float fx = fmaf(kk, gx, ex), fy = fmaf(kk, gy, ey), fz = fmaf(kk, gz, ez);
    const float xx = __fadd_rd(fx, magic), xy = __fadd_rd(fy, magic), xz = __fadd_rd(fz, magic);
    const unsigned id = __float_as_uint(xy) * sys + (__float_as_uint(xx) * sxs + __float_as_uint(xz));
    if (id != cell) {
      cell = id;
      const float4 *p = elem_ptr(q, id - bias);
      lo4 = __ldg(p);
      hi4 = __ldg(p + sys);
    }
    const float wx = fx - (xx - magic), wy = fy - (xy - magic), wz = fz - (xz - magic);
    if (COEF) {
      const float s0 = fmaf(wz, fmaf(wx, lo4.w, lo4.z), fmaf(wx, lo4.y, lo4.x));
      const float s1 = fmaf(wz, fmaf(wx, hi4.w, hi4.z), fmaf(wx, hi4.y, hi4.x));
      return lerpf(s0, s1, wy);
    }
    const float s0 = lerpf(fmaf(wx, lo4.y, lo4.x), fmaf(wx, lo4.w, lo4.z), wz);
    const float s1 = lerpf(fmaf(wx, hi4.y, hi4.x), fmaf(wx, hi4.w, hi4.z), wz);
    return lerpf(s0, s1, wy);
  };
  float acc = 0.f;
  float kf = 0.5f;
  const int nfull = rs.n - 1;
#pragma unroll 2
  for (int k = 0; k < nfull; ++k, kf += 1.f) acc += sample(kf);
  acc = fmaf(rs.last, sample((float)nfull + 0.5f * rs.last), acc);  // exact last segment
  *dst = acc * (float)step;
}

// ---------------------------------------------------------------------------
// Forward projection, b-plane quad variant ("ldg4p").
//
// Rays travel mostly along the middle axis b (the orientation copy puts the
// detector u direction on the fast axis a).  Here the taps are grouped per
// b-plane: Qp[b][z][a] = (V[z][b][a], V[z][b][a+1] - V[z][b][a],
// V[z+1][b][a], V[z+1][b][a+1] - V[z+1][b][a]), and a lane holds the two planes
// of its cell as "near" and "far" along its direction of travel.  A step into
// the next cell along b with the same (a, z) -- the most frequent change --
// keeps far as the new near and loads only the new far plane, so the "near"
// load is issued by far fewer lanes of each quarter-warp and touches fewer
// 128-byte lines (L1 data-pipe wavefronts; a trace of the cfg4
// access pattern predicts -21 % wavefronts per sample).
// ---------------------------------------------------------------------------
__global__ void plane_quad_volume_kernel(const float *__restrict__ vol, int nz, int ny, int nx, int swap_xy,
                                         float4 *__restrict__ q) {
  constexpr int m = kFpMargin;
  const int na = swap_xy ? ny : nx, nb = swap_xy ? nx : ny;
  const int pa = na + 2 * m, pb = nb + 2 * m, pz = nz + 2 * m;
  const long long total = (long long)pb * pz * pa;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(i % pa) - m;
    const long long t = i / pa;
    const int z = (int)(t % pz) - m;
    const int b = (int)(t / pz) - m;
    float v[4];  // v[dz * 2 + da]
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int aa = a + (j & 1), zz = z + (j >> 1);
      float val = 0.f;
      if ((unsigned)zz < (unsigned)nz && (unsigned)aa < (unsigned)na && (unsigned)b < (unsigned)nb) {
        const int x = swap_xy ? b : aa, y = swap_xy ? aa : b;
        val = __ldg(vol + ((long long)zz * ny + y) * nx + x);
      }
      v[j] = val;
    }
    q[i] = make_float4(v[0], v[1] - v[0], v[2], v[3] - v[2]);
  }
}

template <int MINB>
__global__ void __launch_bounds__(kFp2BX *kFp2BY, MINB)
    cone_fp4p_kernel(const float4 *__restrict__ qA, const float4 *__restrict__ qB, int nx, int ny,
                     int nz, double sx, double sy, double sz, const Fp2View *__restrict__ views,
                     int rows, int cols, int n_views, double step, float *__restrict__ out) {
  const int ncb = (cols + kFp2BX - 1) / kFp2BX;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int c = cb * kFp2BX + threadIdx.x;
  const int r = rb * kFp2BY + threadIdx.y;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  const int swap = W.face_copy ? (rs.face == 0 ? 1 : (rs.face == 1 ? 0 : W.swap)) : W.swap;
  const float4 *q = swap ? qB : qA;
  const int na = swap ? ny : nx;
  const float ea = (swap ? rs.ey : rs.ex) + (kFpMargin - 1);
  const float eb = (swap ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = swap ? rs.gy : rs.gx, gb = swap ? rs.gx : rs.gy, gz = rs.gz;
  const unsigned pa = (unsigned)(na + 2 * kFpMargin);
  const unsigned pp = (unsigned)(nz + 2 * kFpMargin) * pa;  // b-plane stride
  const unsigned bias = kFloorBits * (1u + pa + pp);
  const bool fwd = gb >= 0.f;                      // direction of travel along b
  const unsigned far_off = fwd ? pp : 0u, near_off = fwd ? 0u : pp;
  const unsigned bstep = fwd ? pp : 0u - pp;        // cell index change of a pure b step
  const float tsgn = fwd ? 1.f : -1.f, toff = fwd ? 0.f : 1.f;  // weight of far: wb or 1 - wb
  unsigned cell = 0x80000000u;
  float4 nr = make_float4(0.f, 0.f, 0.f, 0.f), fr = nr;
  auto sample = [&](float kk) -> float {
    const float fa = fmaf(kk, ga, ea), fb = fmaf(kk, gb, eb), fz = fmaf(kk, gz, ez);
    const float xa = floor_magic(fa), xb = floor_magic(fb), xz = floor_magic(fz);
    const unsigned id = __float_as_uint(xb) * pp + (__float_as_uint(xz) * pa + __float_as_uint(xa)) - bias;
    // straight-line, predicated: shift (near <- far) or reload near, then the new far
    const bool chg = id != cell;
    const bool sh = id - cell == bstep;  // implies chg
    if (sh) nr = fr;
    if (chg && !sh) nr = __ldg(elem_ptr(q, id + near_off));
    if (chg) fr = __ldg(elem_ptr(q, id + far_off));
    cell = id;
    const float wa = fa - (xa - kFloorMagic), wb = fb - (xb - kFloorMagic), wz = fz - (xz - kFloorMagic);
    const float sn = lerpf(fmaf(wa, nr.y, nr.x), fmaf(wa, nr.w, nr.z), wz);
    const float sf = lerpf(fmaf(wa, fr.y, fr.x), fmaf(wa, fr.w, fr.z), wz);
    return lerpf(sn, sf, fmaf(tsgn, wb, toff));
  };
  float acc = 0.f;
  float kf = 0.5f;
  const int nfull = rs.n - 1;
#pragma unroll 2
  for (int k = 0; k < nfull; ++k, kf += 1.f) acc += sample(kf);
  acc = fmaf(rs.last, sample((float)nfull + 0.5f * rs.last), acc);  // exact last segment
  *dst = acc * (float)step;
}

// ---------------------------------------------------------------------------
// Forward projection, coefficient-cell variant ("ldg8").
//
// The ncu capture of cone_fp4_kernel (profiles/ncu_r01c_*) shows an issue-
// bound loop of ~42 instructions per sample, 5 of them conversions (3 FRND
// + 2 F2I, quarter-rate pipe).  Here
//   * every margin-padded cell (z, b, a) stores the 8 coefficients of its
//     trilinear polynomial in Horner order, 32 B aligned, so a cell is ONE
//     256-bit load (one sector) and the interpolation is 7 FFMA:
//       f = c000 + wa c100 + wb c010 + wa wb c110
//         + wz (c001 + wa c101 + wb c011 + wa wb c111);
//   * floor() is an FADD.RM with 1.5 * 2^23 (the sum's mantissa IS the
//     integer), so the loop has no conversion instructions: the cell index is
//     formed from the raw float bits with two IMADs, the fraction fa - floor(fa)
//     is exact as before.
// Traversal, sample positions and loop counts are those of cone_fp2_kernel.
// ---------------------------------------------------------------------------
struct __align__(32) Cell8 {
  float c[8];  // c000 c100 c010 c110 | c001 c101 c011 c111   (a fastest, then b, then z)
};

__global__ void coef_volume_kernel(const float *__restrict__ vol, int nz, int ny, int nx, int swap_xy,
                                   Cell8 *__restrict__ q) {
  constexpr int m = kFpMargin;
  const int na = swap_xy ? ny : nx, nb = swap_xy ? nx : ny;
  const int pa = na + 2 * m, pb = nb + 2 * m, pz = nz + 2 * m;
  const long long total = (long long)pz * pb * pa;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(i % pa) - m;
    const long long t = i / pa;
    const int b = (int)(t % pb) - m;
    const int z = (int)(t / pb) - m;
    float v[8];  // v[dz*4 + db*2 + da]
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int aa = a + (j & 1), bb = b + ((j >> 1) & 1), zz = z + (j >> 2);
      float val = 0.f;
      if ((unsigned)zz < (unsigned)nz && (unsigned)aa < (unsigned)na && (unsigned)bb < (unsigned)nb) {
        const int x = swap_xy ? bb : aa, y = swap_xy ? aa : bb;
        val = __ldg(vol + ((long long)zz * ny + y) * nx + x);
      }
      v[j] = val;
    }
    Cell8 c;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // z = 0 / 1 slice: bilinear coefficients
      const float *s = v + 4 * h;
      c.c[4 * h + 0] = s[0];
      c.c[4 * h + 1] = s[1] - s[0];
      c.c[4 * h + 2] = s[2] - s[0];
      c.c[4 * h + 3] = (s[3] - s[2]) - (s[1] - s[0]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) c.c[4 + j] -= c.c[j];  // z differences
    q[i] = c;
  }
}

__device__ __forceinline__ void ldg_cell8(const Cell8 *p, float (&c)[8]) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(c[0]), "=f"(c[1]), "=f"(c[2]), "=f"(c[3]), "=f"(c[4]), "=f"(c[5]), "=f"(c[6]),
                 "=f"(c[7])
               : "l"(p));
}

template <int MINB>
__global__ void __launch_bounds__(kFp2BX *kFp2BY, MINB)
    cone_fp8_kernel(const Cell8 *__restrict__ qA, const Cell8 *__restrict__ qB, int nx, int ny,
                    int nz, double sx, double sy, double sz, const Fp2View *__restrict__ views,
                    int rows, int cols, int n_views, double step, float *__restrict__ out) {
  const int ncb = (cols + kFp2BX - 1) / kFp2BX;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int c = cb * kFp2BX + threadIdx.x;
  const int r = rb * kFp2BY + threadIdx.y;
  if (c >= cols || r >= rows) return;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    return;
  }
  const Cell8 *q = W.swap ? qB : qA;
  const int na = W.swap ? ny : nx, nb = W.swap ? nx : ny;
  const float ea = (W.swap ? rs.ey : rs.ex) + (kFpMargin - 1);
  const float eb = (W.swap ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = W.swap ? rs.gy : rs.gx, gb = W.swap ? rs.gx : rs.gy, gz = rs.gz;
  const unsigned pa = (unsigned)(na + 2 * kFpMargin);
  const unsigned ps = (unsigned)(nb + 2 * kFpMargin) * pa;
  // raw index = bits(za) * ps + bits(zb) * pa + bits(xa) = cell + bias  (mod 2^32)
  const unsigned bias = kFloorBits * (1u + pa + ps);
  unsigned cell = ~0u;
  float k8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto sample = [&](float kk) -> float {
    const float fa = fmaf(kk, ga, ea), fb = fmaf(kk, gb, eb), fz = fmaf(kk, gz, ez);
    const float xa = floor_magic(fa), xb = floor_magic(fb), xz = floor_magic(fz);
    const unsigned id = __float_as_uint(xz) * ps + (__float_as_uint(xb) * pa + __float_as_uint(xa));
    if (id != cell) {
      cell = id;
      ldg_cell8(elem_ptr(q, id - bias), k8);
    }
    const float wa = fa - (xa - kFloorMagic), wb = fb - (xb - kFloorMagic), wz = fz - (xz - kFloorMagic);
    const float lo = fmaf(wb, fmaf(wa, k8[3], k8[2]), fmaf(wa, k8[1], k8[0]));
    const float dz = fmaf(wb, fmaf(wa, k8[7], k8[6]), fmaf(wa, k8[5], k8[4]));
    return fmaf(wz, dz, lo);
  };
  float acc = 0.f;
  float kf = 0.5f;
  const int nfull = rs.n - 1;
#pragma unroll 4
  for (int k = 0; k < nfull; ++k, kf += 1.f) acc += sample(kf);
  acc = fmaf(rs.last, sample((float)nfull + 0.5f * rs.last), acc);  // exact last segment
  *dst = acc * (float)step;
}

// Two rays per thread (detector rows r and r+1 of the same column): the two
// independent sample chains double the loads in flight per warp, hiding L1/L2
// latency without more resident warps.  Same arithmetic as cone_fp2_kernel.
struct RayMarch {
  float ea, eb, ez;
  int nfull;
  float last;
  int cell;
  CellTaps t;
  float acc;
  bool live;
};

__device__ __forceinline__ void march_sample(RayMarch &m, const float *__restrict__ vol, float kf,
                                             float ga, float gb, float gz, int pa, int ps) {
  const float fa = fmaf(kf, ga, m.ea), fb = fmaf(kf, gb, m.eb), fz = fmaf(kf, gz, m.ez);
  const float la = floorf(fa), lb = floorf(fb), lz = floorf(fz);
  const int id = (int)lz * ps + (int)lb * pa + (int)la;
  if (id != m.cell) {
    m.cell = id;
    load_cell(vol + id, pa, ps, m.t);
  }
  m.acc += interp_cell(m.t, fa - la, fb - lb, fz - lz);
}

__device__ __forceinline__ void march_last(RayMarch &m, const float *__restrict__ vol, float ga,
                                           float gb, float gz, int pa, int ps) {
  const float kf = (float)m.nfull + 0.5f * m.last;
  const float fa = fmaf(kf, ga, m.ea), fb = fmaf(kf, gb, m.eb), fz = fmaf(kf, gz, m.ez);
  const float la = floorf(fa), lb = floorf(fb), lz = floorf(fz);
  const int id = (int)lz * ps + (int)lb * pa + (int)la;
  if (id != m.cell) load_cell(vol + id, pa, ps, m.t);
  m.acc = fmaf(m.last, interp_cell(m.t, fa - la, fb - lb, fz - lz), m.acc);
}

template <int MINB>
__global__ void __launch_bounds__(kFp2BX *kFp2BY, MINB)
    cone_fp2r_kernel(const float *__restrict__ volA, const float *__restrict__ volB, int nx, int ny,
                     int nz, double sx, double sy, double sz, const Fp2View *__restrict__ views,
                     int rows, int cols, int n_views, double step, float *__restrict__ out) {
  const int ncb = (cols + kFp2BX - 1) / kFp2BX;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int c = cb * kFp2BX + threadIdx.x;
  const int r0 = rb * (2 * kFp2BY) + 2 * threadIdx.y;  // rows r0 and r0 + 1
  if (c >= cols || r0 >= rows) return;
  const Fp2View W = views[v];
  const bool swap = W.swap != 0;
  const float *vol = swap ? volB : volA;
  const int na = swap ? ny : nx, nb = swap ? nx : ny;
  const int pa = na + 2 * kFpMargin;
  const int ps = (nb + 2 * kFpMargin) * pa;
  RayMarch m[2];
  float g[2][3];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    RaySetup rs;
    m[j].live = (r0 + j) < rows && cone_ray_setup(W.ray, r0 + j, c, nx, ny, nz, sx, sy, sz, step, rs);
    m[j].cell = -1;
    m[j].t = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    m[j].acc = 0.f;
    m[j].nfull = m[j].live ? rs.n - 1 : 0;
    m[j].last = m[j].live ? rs.last : 0.f;
    m[j].ea = m[j].live ? (swap ? rs.ey : rs.ex) + (kFpMargin - 1) : 0.f;
    m[j].eb = m[j].live ? (swap ? rs.ex : rs.ey) + (kFpMargin - 1) : 0.f;
    m[j].ez = m[j].live ? rs.ez + (kFpMargin - 1) : 0.f;
    g[j][0] = m[j].live ? (swap ? rs.gy : rs.gx) : 0.f;
    g[j][1] = m[j].live ? (swap ? rs.gx : rs.gy) : 0.f;
    g[j][2] = m[j].live ? rs.gz : 0.f;
  }
  const float ga = g[0][0], gb = g[0][1], gz = g[0][2];
  const float ga1 = g[1][0], gb1 = g[1][1], gz1 = g[1][2];
  const int n0 = m[0].live ? m[0].nfull : 0, n1 = m[1].live ? m[1].nfull : 0;
  const int nmin = min(n0, n1), nmax = max(n0, n1);
  float kf = 0.5f;
  int k = 0;
  for (; k < nmin; ++k, kf += 1.f) {
    march_sample(m[0], vol, kf, ga, gb, gz, pa, ps);
    march_sample(m[1], vol, kf, ga1, gb1, gz1, pa, ps);
  }
  for (; k < nmax; ++k, kf += 1.f) {
    if (k < n0) march_sample(m[0], vol, kf, ga, gb, gz, pa, ps);
    if (k < n1) march_sample(m[1], vol, kf, ga1, gb1, gz1, pa, ps);
  }
  if (m[0].live) march_last(m[0], vol, ga, gb, gz, pa, ps);
  if (m[1].live) march_last(m[1], vol, ga1, gb1, gz1, pa, ps);
  float *dst = out + ((long long)v * rows + r0) * cols + c;
  dst[0] = m[0].live ? m[0].acc * (float)step : 0.f;
  if (r0 + 1 < rows) dst[cols] = m[1].live ? m[1].acc * (float)step : 0.f;
}

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

__global__ void __launch_bounds__(kFpBX *kFpBY)
    cone_fp_tex_kernel(cudaTextureObject_t tex, int nx, int ny, int nz, double sx, double sy,
                       double sz, const ConeRayView *__restrict__ views, int rows, int cols,
                       double step, float *__restrict__ out) {
  const int c = blockIdx.x * kFpBX + threadIdx.x;
  const int r = blockIdx.y * kFpBY + threadIdx.y;
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
__global__ void __launch_bounds__(kFpBX *kFpBY)
    cone_fp_hwtex_kernel(cudaTextureObject_t tex, int nx, int ny, int nz, double sx, double sy,
                         double sz, const ConeRayView *__restrict__ views, int rows, int cols,
                         double step, float *__restrict__ out) {
  const int c = blockIdx.x * kFpBX + threadIdx.x;
  const int r = blockIdx.y * kFpBY + threadIdx.y;
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

// Exact transpose of cone_fp_kernel: scatter y * seg * weights into the padded
// accumulation volume (fp32 atomics).
__device__ __forceinline__ void trilinear_scatter(float *__restrict__ adjp, int nxp, int nyp,
                                                  int nzp, float fx, float fy, float fz,
                                                  float g) {
  const float flx = floorf(fx), fly = floorf(fy), flz = floorf(fz);
  const int ix = (int)flx, iy = (int)fly, iz = (int)flz;
  if ((unsigned)ix >= (unsigned)(nxp - 1) || (unsigned)iy >= (unsigned)(nyp - 1) ||
      (unsigned)iz >= (unsigned)(nzp - 1))
    return;
  const float wx = fx - flx, wy = fy - fly, wz = fz - flz;
  const unsigned sxy = (unsigned)nyp * (unsigned)nxp;
  float *p = adjp + ((unsigned)iz * sxy + (unsigned)iy * (unsigned)nxp + (unsigned)ix);
  float *q = p + sxy;
  const float gz0 = g * (1.f - wz), gz1 = g * wz;
  const float a0 = gz0 * (1.f - wy), a1 = gz0 * wy, b0 = gz1 * (1.f - wy), b1 = gz1 * wy;
  atomicAdd(p, a0 * (1.f - wx));
  atomicAdd(p + 1, a0 * wx);
  atomicAdd(p + nxp, a1 * (1.f - wx));
  atomicAdd(p + nxp + 1, a1 * wx);
  atomicAdd(q, b0 * (1.f - wx));
  atomicAdd(q + 1, b0 * wx);
  atomicAdd(q + nxp, b1 * (1.f - wx));
  atomicAdd(q + nxp + 1, b1 * wx);
}

__global__ void __launch_bounds__(kFpBX *kFpBY)
    cone_fp_adjoint_kernel(const float *__restrict__ sino, int nx, int ny, int nz,
                           double sx, double sy, double sz,
                           const ConeRayView *__restrict__ views, int rows, int cols,
                           double step, float *__restrict__ adjp) {
  const int c = blockIdx.x * kFpBX + threadIdx.x;
  const int r = blockIdx.y * kFpBY + threadIdx.y;
  const int v = blockIdx.z;
  if (c >= cols || r >= rows) return;
  const float y = __ldg(sino + ((long long)v * rows + r) * cols + c);
  if (y == 0.f) return;
  const ConeRayView V = views[v];
  RaySetup rs;
  if (!cone_ray_setup(V, r, c, nx, ny, nz, sx, sy, sz, step, rs)) return;
  const int nxp = nx + 2, nyp = ny + 2, nzp = nz + 2;
  const float g = y * (float)step;
  const int nfull = rs.n - 1;
  for (int k = 0; k < nfull; ++k) {
    const float kf = (float)k + 0.5f;
    trilinear_scatter(adjp, nxp, nyp, nzp, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey),
                      fmaf(kf, rs.gz, rs.ez), g);
  }
  const float kf = (float)nfull + 0.5f * rs.last;
  trilinear_scatter(adjp, nxp, nyp, nzp, fmaf(kf, rs.gx, rs.ex), fmaf(kf, rs.gy, rs.ey),
                    fmaf(kf, rs.gz, rs.ez), g * rs.last);
}

// ---------------------------------------------------------------------------
// Matched adjoint A^T of the forward projector, quad-scatter form ("red4",
// default).  The exact transpose of cone_fp4_kernel's march: the same rays,
// CTA order, per-ray orientation copy and sample positions, but each sample
// SCATTERS y * seg * (trilinear weights) into tap quads of the copy,
//   Q[z][b][a] += (w(b,a), w(b,a+1), w(b+1,a), w(b+1,a+1)) of slice z,
// accumulated in registers while the ray stays in one cell and flushed as two
// vector reductions (REDG.ADD.F32x4: slices z and z+1) when it leaves -- one
// L2 atomic op per 4 taps instead of 4, and ~1.7 samples per flush.
// unquad_tiled_kernel then folds the four quads that hold each voxel's tap
// back into the (z, y, x) volume (the transpose of quad_volume_tiled_kernel).
// fp32 atomics: the summation order is not deterministic (tolerance 1e-4 vs
// the oracle's exact transpose, tests/test_gpu_parity.py).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_add_v4(float4 *p, const float4 &v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

template <int MINB>
__global__ void __launch_bounds__(kFp2BX *kFp2BY, MINB)
    cone_fp_adjoint4_kernel(const float *__restrict__ sino, float4 *__restrict__ qA, float4 *__restrict__ qB,
                            int nx, int ny, int nz, double sx, double sy, double sz,
                            const Fp2View *__restrict__ views, int rows, int cols, int n_views, double step) {
  const int ncb = (cols + kFp2BX - 1) / kFp2BX;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int c = cb * kFp2BX + threadIdx.x;
  const int r = rb * kFp2BY + threadIdx.y;
  if (c >= cols || r >= rows) return;
  const float y = __ldg(sino + ((long long)v * rows + r) * cols + c);
  if (y == 0.f) return;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) return;
  const int swap = W.face_copy ? (rs.face == 0 ? 1 : (rs.face == 1 ? 0 : W.swap)) : W.swap;
  float4 *q = swap ? qB : qA;
  const int na = swap ? ny : nx, nb = swap ? nx : ny;
  const float ea = (swap ? rs.ey : rs.ex) + (kFpMargin - 1);
  const float eb = (swap ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = swap ? rs.gy : rs.gx, gb = swap ? rs.gx : rs.gy, gz = rs.gz;
  const int pa = na + 2 * kFpMargin;
  const int ps = (nb + 2 * kFpMargin) * pa;
  const unsigned bias = kFloorBits * (1u + (unsigned)pa + (unsigned)ps);
  const float g = y * (float)step;
  float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
  unsigned cell = 0u;
  bool open = false;
  auto sample = [&](float kk, float gs) {
    const float fa = fmaf(kk, ga, ea), fb = fmaf(kk, gb, eb), fz = fmaf(kk, gz, ez);
    const float xa = floor_magic(fa), xb = floor_magic(fb), xz = floor_magic(fz);
    const unsigned id = __float_as_uint(xz) * (unsigned)ps + (__float_as_uint(xb) * (unsigned)pa + __float_as_uint(xa));
    if (id != cell) {
      if (open) {
        float4 *p = q + (cell - bias);
        red_add_v4(p, lo);
        red_add_v4(p + ps, hi);
      }
      open = true;
      cell = id;
      lo = make_float4(0.f, 0.f, 0.f, 0.f);
      hi = lo;
    }
    const float wa = fa - (xa - kFloorMagic), wb = fb - (xb - kFloorMagic), wz = fz - (xz - kFloorMagic);
    const float g1 = gs * wz, g0 = gs - g1;
    const float l1 = g0 * wb, l0 = g0 - l1, h1 = g1 * wb, h0 = g1 - h1;
    const float l0a = l0 * wa, l1a = l1 * wa, h0a = h0 * wa, h1a = h1 * wa;
    lo.x += l0 - l0a;
    lo.y += l0a;
    lo.z += l1 - l1a;
    lo.w += l1a;
    hi.x += h0 - h0a;
    hi.y += h0a;
    hi.z += h1 - h1a;
    hi.w += h1a;
  };
  float kf = 0.5f;
  const int nfull = rs.n - 1;
  for (int k = 0; k < nfull; ++k, kf += 1.f) sample(kf, g);
  sample((float)nfull + 0.5f * rs.last, g * rs.last);
  float4 *p = q + (cell - bias);
  red_add_v4(p, lo);
  red_add_v4(p + ps, hi);
}

// vol (+)= fold of one orientation copy's scatter quads: the tap at margin-
// padded (z, b, a) is Q[b][a].x + Q[b][a-1].y + Q[b-1][a].z + Q[b-1][a-1].w of
// slice z.  32 (a) x 32 (b) tiles through shared memory so that both the quad
// reads (along a) and the volume writes (along x) are coalesced for either copy.
template <bool SWAP>
__global__ void __launch_bounds__(256) unquad_tiled_kernel(const float4 *__restrict__ q, int nz, int ny, int nx,
                                                           float *__restrict__ vol, int accumulate) {
  __shared__ float4 tq[33][33];  // [b - b0 + 1][a - a0 + 1]
  __shared__ float res[32][33];  // [a - a0][b - b0]
  constexpr int m = kFpMargin;
  const int na = SWAP ? ny : nx, nb = SWAP ? nx : ny;
  const int pa = na + 2 * m, pb = nb + 2 * m;
  const int a0 = blockIdx.x * 32, b0 = blockIdx.y * 32, z = blockIdx.z;  // real voxel coordinates
  const long long slice = (long long)(z + m) * pb * pa;
  for (int e = threadIdx.x; e < 33 * 33; e += 256) {
    const int da = e % 33, db = e / 33;
    const int pa_i = a0 + m - 1 + da, pb_i = b0 + m - 1 + db;  // padded cell coordinates
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (pa_i < pa && pb_i < pb) val = q[slice + (long long)pb_i * pa + pa_i];
    tq[db][da] = val;
  }
  __syncthreads();
  const int ta = threadIdx.x & 31;
  for (int tb = threadIdx.x >> 5; tb < 32; tb += 8)
    res[ta][tb] = tq[tb + 1][ta + 1].x + tq[tb + 1][ta].y + tq[tb][ta + 1].z + tq[tb][ta].w;
  __syncthreads();
  // write along x: x = a (copy A) or x = b (copy B)
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    const int dx = e & 31, dy = e >> 5;
    const int da = SWAP ? dy : dx, db = SWAP ? dx : dy;
    const int a = a0 + da, bb = b0 + db;
    if (a >= na || bb >= nb) continue;
    const int x = SWAP ? bb : a, yy = SWAP ? a : bb;
    float *o = vol + ((long long)z * ny + yy) * nx + x;
    const float t = res[da][db];
    *o = accumulate ? *o + t : t;
  }
}

// z-fastest form of the quad scatter (the transpose of cone_fp4z_kernel, "red4z",
// default): quarter = 8 rows of one column, so lanes flush together into
// contiguous quads.  Two scatter buffers, one per horizontal row axis b:
//   qy: Qz[y][x][z] += (w(z,x), w(z,x+1), w(z+1,x), w(z+1,x+1)) of row y,
//   qx: Qx[x][y][z] += (w(z,y), w(z,y+1), w(z+1,y), w(z+1,y+1)) of row x;
// a ray scatters into the buffer whose row axis is its major horizontal axis,
// so most cell changes are row steps b -> b +- 1, where the new cell's near row
// is the old cell's far row: that quad's accumulator is carried over in
// registers and only the row left behind is flushed (one REDG.F32x4 instead of
// two).
// DET: fixed-point flush -- each quad component is rounded to an integer multiple of
// 2^-e (scale = 2^e, exact) and added with 64-bit integer atomics into u64 quads.
// Integer addition is associative, so the result does not depend on the order in
// which rays flush: bit-reproducible (torch.use_deterministic_algorithms).
__device__ __forceinline__ void red_add_fx4(unsigned long long *p, const float4 &v, float scale) {
  atomicAdd(p, (unsigned long long)__float2ll_rn(v.x * scale));
  atomicAdd(p + 1, (unsigned long long)__float2ll_rn(v.y * scale));
  atomicAdd(p + 2, (unsigned long long)__float2ll_rn(v.z * scale));
  atomicAdd(p + 3, (unsigned long long)__float2ll_rn(v.w * scale));
}

template <int MINB, bool DET = false>
__global__ void __launch_bounds__(128, MINB)
    cone_fp_adjoint4z_kernel(const float *__restrict__ sino, void *__restrict__ qy_, void *__restrict__ qx_,
                             int nx, int ny, int nz, double sx, double sy, double sz,
                             const Fp2View *__restrict__ views, int rows, int cols, int n_views, double step,
                             float scale) {
  constexpr int kCols = 16;
  const int ncb = (cols + kCols - 1) / kCols;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views);
  const int rb = (int)(bt / n_views);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = cb * kCols + warp * 4 + (lane >> 3);
  const int r = rb * kFpzRows + (lane & 7);
  if (c >= cols || r >= rows) return;
  const float y = __ldg(sino + ((long long)v * rows + r) * cols + c);
  if (y == 0.f) return;
  const Fp2View W = views[v];
  RaySetup rs;
  if (!cone_ray_setup(W.ray, r, c, nx, ny, nz, sx, sy, sz, step, rs)) return;
  const bool xrow = fabsf(rs.gx) > fabsf(rs.gy);  // major horizontal axis (cells per step)
  void *qv = xrow ? qx_ : qy_;
  auto flush = [&](unsigned cidx, const float4 &v) {  // quad cidx += v
    if (DET)
      red_add_fx4(static_cast<unsigned long long *>(qv) + 4ull * cidx, v, scale);
    else
      red_add_v4(static_cast<float4 *>(qv) + cidx, v);
  };
  const float ea = (xrow ? rs.ey : rs.ex) + (kFpMargin - 1), eb = (xrow ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = xrow ? rs.gy : rs.gx, gb = xrow ? rs.gx : rs.gy, gz = rs.gz;
  const unsigned pz = (unsigned)(nz + 2 * kFpMargin);
  const unsigned sas = pz, sbs = (unsigned)((xrow ? ny : nx) + 2 * kFpMargin) * pz;  // a and b strides
  const unsigned bias = kFloorBits * (1u + sas + sbs);
  const float g = y * (float)step;
  float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
  unsigned cell = 0u;
  bool open = false;
  auto sample = [&](float kk, float gs) {
    const float fa = fmaf(kk, ga, ea), fb = fmaf(kk, gb, eb), fz = fmaf(kk, gz, ez);
    const float xa = floor_magic(fa), xb = floor_magic(fb), xz = floor_magic(fz);
    const unsigned id = __float_as_uint(xb) * sbs + (__float_as_uint(xa) * sas + __float_as_uint(xz));
    if (id != cell) {
      const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
      if (open) {
        const unsigned c0 = cell - bias;
        const unsigned d = id - cell;
        if (d == sbs) {  // row b -> b + 1: the far row becomes the near row
          flush(c0, lo);
          lo = hi;
          hi = zero;
        } else if (d == 0u - sbs) {  // row b -> b - 1: the near row becomes the far row
          flush(c0 + sbs, hi);
          hi = lo;
          lo = zero;
        } else {
          flush(c0, lo);
          flush(c0 + sbs, hi);
          lo = hi = zero;
        }
      }
      open = true;
      cell = id;
    }
    const float wa = fa - (xa - kFloorMagic), wb = fb - (xb - kFloorMagic), wz = fz - (xz - kFloorMagic);
    const float g1 = gs * wb, g0 = gs - g1;
    const float l1 = g0 * wz, l0 = g0 - l1, h1 = g1 * wz, h0 = g1 - h1;
    const float l0a = l0 * wa, l1a = l1 * wa, h0a = h0 * wa, h1a = h1 * wa;
    lo.x += l0 - l0a;
    lo.y += l0a;
    lo.z += l1 - l1a;
    lo.w += l1a;
    hi.x += h0 - h0a;
    hi.y += h0a;
    hi.z += h1 - h1a;
    hi.w += h1a;
  };
  float kf = 0.5f;
  const int nfull = rs.n - 1;
  for (int k = 0; k < nfull; ++k, kf += 1.f) sample(kf, g);
  sample((float)nfull + 0.5f * rs.last, g * rs.last);
  flush(cell - bias, lo);
  flush(cell - bias + sbs, hi);
}

// deterministic fold: vol[z][y][x] = 2^-e (sum of the 8 fixed-point taps of both
// scatter buffers) -- integer sums, one rounding to float
__global__ void __launch_bounds__(256) unquad_fx_kernel(const unsigned long long *__restrict__ qy,
                                                        const unsigned long long *__restrict__ qx, int nz, int ny,
                                                        int nx, double inv_scale, float *__restrict__ vol) {
  constexpr int m = kFpMargin;
  const long long pz = nz + 2 * m, px = nx + 2 * m, py = ny + 2 * m;
  const long long n = (long long)nz * ny * nx;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((long long)nx * ny));
    const long long zp = z + m, yp = y + m, xp = x + m;
    // qy: Qz[y][x][z] taps (z,x),(z,x+1),(z+1,x),(z+1,x+1) of row y
    auto Y = [&](long long yy, long long xx, long long zz, int c) { return (long long)qy[4 * ((yy * px + xx) * pz + zz) + c]; };
    // qx: Qx[x][y][z] taps (z,y),(z,y+1),(z+1,y),(z+1,y+1) of row x
    auto X = [&](long long xx, long long yy, long long zz, int c) { return (long long)qx[4 * ((xx * py + yy) * pz + zz) + c]; };
    const long long t = Y(yp, xp, zp, 0) + Y(yp, xp - 1, zp, 1) + Y(yp, xp, zp - 1, 2) + Y(yp, xp - 1, zp - 1, 3) +
                        X(xp, yp, zp, 0) + X(xp, yp - 1, zp, 1) + X(xp, yp, zp - 1, 2) + X(xp, yp - 1, zp - 1, 3);
    vol[i] = (float)((double)t * inv_scale);
  }
}

__global__ void absmax_kernel(const float *__restrict__ x, long long n, unsigned *__restrict__ out) {
  unsigned m = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(__ldg(x + i))));  // non-negative floats order as integers
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// vol += fold of the x-row scatter quads qx: the tap at padded (z, y, x) is
// Qx[x][y][z].x + Qx[x][y-1][z].y + Qx[x][y][z-1].z + Qx[x][y-1][z-1].w.
// 32 (z) x 32 (x) tiles of one y: quad reads along z, volume writes along x.
__global__ void __launch_bounds__(256) unquad_zx_kernel(const float4 *__restrict__ q, int nz, int ny, int nx,
                                                        float *__restrict__ vol) {
  __shared__ float4 tq[2][32][33];  // [y row: 0 = y-1, 1 = y][x - x0][z - z0 + 1]
  __shared__ float res[32][33];     // [z - z0][x - x0]
  constexpr int m = kFpMargin;
  const int pz = nz + 2 * m, py = ny + 2 * m;
  const int z0 = blockIdx.x * 32, x0 = blockIdx.y * 32, y = blockIdx.z;  // real voxel coordinates
  for (int e = threadIdx.x; e < 2 * 32 * 33; e += 256) {
    const int h = e / (32 * 33), f = e % (32 * 33);
    const int dz = f % 33, dx = f / 33;
    const int zi = z0 + m - 1 + dz, xi = x0 + m + dx, yi = y + m - 1 + h;  // padded cell coordinates
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (zi < pz && x0 + dx < nx) val = q[((long long)xi * py + yi) * pz + zi];
    tq[h][dx][dz] = val;
  }
  __syncthreads();
  const int tz = threadIdx.x & 31;
  for (int tx = threadIdx.x >> 5; tx < 32; tx += 8)
    res[tz][tx] = tq[1][tx][tz + 1].x + tq[0][tx][tz + 1].y + tq[1][tx][tz].z + tq[0][tx][tz].w;
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    const int dx = e & 31, dz = e >> 5;
    const int x = x0 + dx, z = z0 + dz;
    if (x < nx && z < nz) vol[((long long)z * ny + y) * nx + x] += res[dz][dx];
  }
}

// vol = fold of the z-fastest scatter quads: the tap at padded (z, y, x) is
// Qz[y][x][z].x + Qz[y][x-1][z].y + Qz[y][x][z-1].z + Qz[y][x-1][z-1].w.
// 32 (z) x 32 (x) tiles of one y row: quad reads along z, volume writes along x.
__global__ void __launch_bounds__(256) unquad_z_kernel(const float4 *__restrict__ q, int nz, int ny, int nx,
                                                       float *__restrict__ vol) {
  __shared__ float4 tq[33][33];  // [x - x0 + 1][z - z0 + 1]
  __shared__ float res[32][33];  // [z - z0][x - x0]
  constexpr int m = kFpMargin;
  const int pz = nz + 2 * m, px = nx + 2 * m;
  const int z0 = blockIdx.x * 32, x0 = blockIdx.y * 32, y = blockIdx.z;  // real voxel coordinates
  const long long row = (long long)(y + m) * px;
  for (int e = threadIdx.x; e < 33 * 33; e += 256) {
    const int dz = e % 33, dx = e / 33;
    const int zi = z0 + m - 1 + dz, xi = x0 + m - 1 + dx;  // padded cell coordinates
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (zi < pz && xi < px) val = q[(row + xi) * pz + zi];
    tq[dx][dz] = val;
  }
  __syncthreads();
  const int tz = threadIdx.x & 31;
  for (int tx = threadIdx.x >> 5; tx < 32; tx += 8)
    res[tz][tx] = tq[tx + 1][tz + 1].x + tq[tx][tz + 1].y + tq[tx + 1][tz].z + tq[tx][tz].w;
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    const int dx = e & 31, dz = e >> 5;
    const int x = x0 + dx, z = z0 + dz;
    if (x < nx && z < nz) vol[((long long)z * ny + y) * nx + x] = res[dz][dx];
  }
}

// ---------------------------------------------------------------------------
// Back projection (voxel-driven gather), _kernels.py:281-322.
// Thread = one (x, y) column and ZB consecutive z voxels; loop over views
// with the per-view constants staged in shared memory.
// ---------------------------------------------------------------------------
constexpr int kBpBX = 32, kBpBY = 8, kBpChunk = 128;


// Column taps (clamped indices + weights, zero outside [0, cols)).
__device__ __forceinline__ void col_taps(float fc, int cols, int &ca, int &cb, float &g0,
                                         float &g1) {
  const float fl = floorf(fc);
  const int c0 = (int)fl;
  const float wc = fc - fl;
  g0 = ((unsigned)c0 < (unsigned)cols) ? 1.f - wc : 0.f;
  g1 = ((unsigned)(c0 + 1) < (unsigned)cols) ? wc : 0.f;
  ca = min(max(c0, 0), cols - 1);
  cb = min(max(c0 + 1, 0), cols - 1);
}

template <int ZB, bool ZINV, bool WEIGHTED>
__global__ void __launch_bounds__(kBpBX *kBpBY) cone_bp_kernel(const BpParams p) {
  __shared__ ConeVoxView sv[kBpChunk];
  const int ix = blockIdx.x * kBpBX + threadIdx.x;
  const int iy = blockIdx.y * kBpBY + threadIdx.y;
  const int zl0 = blockIdx.z * ZB;  // local z of this thread's first voxel
  const bool active = ix < p.nx && iy < p.ny;
  const float xc = (float)ix - p.cx;
  const float yc = (float)iy - p.cy;
  const float zc0 = (float)(p.z_begin + zl0) - p.cz;
  const int tid = threadIdx.y * kBpBX + threadIdx.x;

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
      const float *s = p.sino + (long long)(v0 + j) * p.view_stride;
      const float a0 = fmaf(V.a[0], xc, fmaf(V.a[1], yc, fmaf(V.a[2], zc0, V.a[3])));
      const float b0 = fmaf(V.b[0], xc, fmaf(V.b[1], yc, fmaf(V.b[2], zc0, V.b[3])));
      const float w0 = fmaf(V.w[0], xc, fmaf(V.w[1], yc, fmaf(V.w[2], zc0, V.w[3])));
      if (ZINV) {
        if (!(w0 > (float)kTiny)) continue;  // _kernels.py:297-298
        const float rw = 1.f / w0;
        int ca, cb;
        float g0, g1;
        col_taps(fmaf(a0, rw, p.cu), p.cols, ca, cb, g0, g1);
        if (WEIGHTED) {  // (sid / w)^2 folded into the column weights
          const float q = p.sid * rw;
          g0 *= q * q;
          g1 *= q * q;
        }
        if (g0 == 0.f && g1 == 0.f) continue;
        const float fr0 = fmaf(b0, rw, p.cv);
        const float dr = V.b[2] * rw;
#pragma unroll
        for (int k = 0; k < ZB; ++k) {
          const float fr = fmaf((float)k, dr, fr0);
          const float fl = floorf(fr);
          const int r0 = (int)fl;
          const float wr = fr - fl;
          const float h0 = ((unsigned)r0 < (unsigned)p.band_rows) ? 1.f - wr : 0.f;
          const float h1 = ((unsigned)(r0 + 1) < (unsigned)p.band_rows) ? wr : 0.f;
          const int ra = min(max(r0, 0), p.band_rows - 1);
          const int rb = min(max(r0 + 1, 0), p.band_rows - 1);
          const float *sa = s + (long long)ra * p.cols;
          const float *sb = s + (long long)rb * p.cols;
          const float top = fmaf(g0, __ldg(sa + ca), g1 * __ldg(sa + cb));
          const float bot = fmaf(g0, __ldg(sb + ca), g1 * __ldg(sb + cb));
          acc[k] = fmaf(h0, top, fmaf(h1, bot, acc[k]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < ZB; ++k) {
          const float kf = (float)k;
          const float w = fmaf(kf, V.w[2], w0);
          if (!(w > (float)kTiny)) continue;
          const float rw = 1.f / w;
          int ca, cb;
          float g0, g1;
          col_taps(fmaf(fmaf(kf, V.a[2], a0), rw, p.cu), p.cols, ca, cb, g0, g1);
          const float fr = fmaf(fmaf(kf, V.b[2], b0), rw, p.cv);
          const float fl = floorf(fr);
          const int r0 = (int)fl;
          const float wr = fr - fl;
          const float h0 = ((unsigned)r0 < (unsigned)p.band_rows) ? 1.f - wr : 0.f;
          const float h1 = ((unsigned)(r0 + 1) < (unsigned)p.band_rows) ? wr : 0.f;
          const int ra = min(max(r0, 0), p.band_rows - 1);
          const int rb = min(max(r0 + 1, 0), p.band_rows - 1);
          const float *sa = s + (long long)ra * p.cols;
          const float *sb = s + (long long)rb * p.cols;
          float val = h0 * fmaf(g0, __ldg(sa + ca), g1 * __ldg(sa + cb)) +
                      h1 * fmaf(g0, __ldg(sb + ca), g1 * __ldg(sb + cb));
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
template <int ZB, bool ZINV, bool WEIGHTED, bool Q42 = false>
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
// Coefficient-quad back projector ("coef", default).
//
// Same traversal as cone_bp_quad_kernel, but
//   * each quad holds the bilinear polynomial of its detector cell,
//       C[v][r0+2][c0+2] = (s00, s01 - s00, s10 - s00, s11 - s10 - s01 + s00),
//     so an update is  acc += q * ((s00 + wc c1) + wr (c2 + wc c3)): 4 FFMA;
//   * row / column floors use floor_magic (no FRND / F2I), the row index comes
//     straight from the float bits; rows are clamped in float onto the all-zero
//     quad rows -2 / R (their weights are irrelevant there).
// ---------------------------------------------------------------------------
__global__ void coefify_kernel(const float *__restrict__ sino, int n_views, int rows, int cols,
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
    const float s00 = (ra && ca) ? __ldg(s + (long long)r0 * cols + c0) : 0.f;
    const float s01 = (ra && cb) ? __ldg(s + (long long)r0 * cols + c0 + 1) : 0.f;
    const float s10 = (rb && ca) ? __ldg(s + (long long)(r0 + 1) * cols + c0) : 0.f;
    const float s11 = (rb && cb) ? __ldg(s + (long long)(r0 + 1) * cols + c0 + 1) : 0.f;
    quads[i] = make_float4(s00, s01 - s00, s10 - s00, (s11 - s10) - (s01 - s00));
  }
}

template <int ZB, bool ZINV, bool WEIGHTED>
__global__ void __launch_bounds__(kBqBX *kBqBY, 2) cone_bp_coef_kernel(const BpParams p,
                                                                   const float4 *__restrict__ quads) {
  __shared__ ConeVoxView sv[kBpChunk];
  const int ix = blockIdx.x * kBqBX + threadIdx.x;
  const int iy = blockIdx.y * kBqBY + threadIdx.y;
  const int zl0 = blockIdx.z * ZB;
  const bool active = ix < p.nx && iy < p.ny;
  const float xc = (float)ix - p.cx;
  const float yc = (float)iy - p.cy;
  const float zc0 = (float)(p.z_begin + zl0) - p.cz;
  const int tid = threadIdx.y * kBqBX + threadIdx.x;
  const unsigned qc = (unsigned)(p.cols + 1 + kQuadPad);  // quads per row
  const float rhi = (float)p.band_rows;                   // all-zero quad rows: -2 and R
  const float chi = (float)p.cols;                        // all-zero quad columns: -2 and C
  const long long qview = (long long)(p.band_rows + 1 + kQuadPad) * qc;
  const float colmax = (float)(p.cols - 1);
  // quad offset of (row r0, column c0) from raw floor bits: (r0 + 2) qc + c0 + 2
  const unsigned rbias = ((unsigned)kQuadPad - kFloorBits) * qc;
  const unsigned cbias = (unsigned)kQuadPad - kFloorBits;

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
        const float xcf = floor_magic(fc);
        const float flc = xcf - kFloorMagic;
        if (!(flc >= -1.f && flc <= colmax)) continue;  // both column taps off the detector
        const float wc = fc - flc;
        float q = 1.f;
        if (WEIGHTED) {  // (sid / w)^2, _kernels.py:318-320
          q = p.sid * rw;
          q *= q;
        }
        const unsigned rcb = rbias + __float_as_uint(xcf) + cbias;  // + column, per (x, y, view)
        const float fr0 = fmaf(b0, rw, p.cv);
        const float dr = V.b[2] * rw;
#pragma unroll
        for (int k0 = 0; k0 < ZB; k0 += 8) {
          unsigned off[8];
          float wr[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float fr = fminf(fmaxf(fmaf((float)(k0 + i), dr, fr0), -2.f), rhi);
            const float xr = floor_magic(fr);
            off[i] = __float_as_uint(xr) * qc + rcb;
            wr[i] = fr - (xr - kFloorMagic);
          }
          float4 t[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = __ldg(elem_ptr(qv, off[i]));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float val = fmaf(wr[i], fmaf(wc, t[i].w, t[i].z), fmaf(wc, t[i].y, t[i].x));
            acc[k0 + i] = fmaf(q, val, acc[k0 + i]);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < ZB; ++k) {
          const float kf = (float)k;
          const float w = fmaf(kf, V.w[2], w0);
          if (!(w > (float)kTiny)) continue;
          const float rw = 1.f / w;
          const float fc = fminf(fmaxf(fmaf(fmaf(kf, V.a[2], a0), rw, p.cu), -2.f), chi);
          const float fr = fminf(fmaxf(fmaf(fmaf(kf, V.b[2], b0), rw, p.cv), -2.f), rhi);
          const float xcf = floor_magic(fc), xr = floor_magic(fr);
          const float4 t = __ldg(elem_ptr(qv, __float_as_uint(xr) * qc + rbias + __float_as_uint(xcf) + cbias));
          const float wc = fc - (xcf - kFloorMagic), wr = fr - (xr - kFloorMagic);
          const float val = fmaf(wr, fmaf(wc, t.w, t.z), fmaf(wc, t.y, t.x));
          if (WEIGHTED) {
            const float q = p.sid * rw;
            acc[k] = fmaf(q * q, val, acc[k]);
          } else {
            acc[k] += val;
          }
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
// Shared-memory staged back projector ("smem", default for z-invariant
// trajectories) -- the north star's "detector tiles for a batch of views are
// staged into shared memory".
//
// CTA = 16x16 (x, y) voxel columns x kBsZB z-voxels.  For each batch of kBsNV
// views, the CTA projects the 8 corners of its voxel box through each view's
// P (exact bound: central projection of a convex box), and copies the
// covering detector rectangle (+1 pixel margin) into shared memory with
// cp.async (zero-filled outside the detector = the reference's per-tap
// bounds).  The next batch streams in while the current one is consumed
// (double buffering).  Each update then reads its 4 taps with LDS (L1 data
// path not involved) -- 128 B/clk/SM of shared-memory bandwidth instead of
// the ~64 B/clk the L1 load path sustains for 16-byte-per-lane gathers.
// A view whose rectangle does not fit (extreme magnification) or that has a
// corner behind the source is gathered straight from global memory instead.
// ---------------------------------------------------------------------------
constexpr int kBsTX = 16, kBsTY = 16, kBsZB = 16, kBsNV = 4, kBsCap = 3072;

struct BsRect {
  int r0, c0, h, w;  // detector rectangle (band-local rows), h*w <= kBsCap, or w = 0: uncached
};

__device__ __forceinline__ void cp_async4(float *smem_dst, const float *gsrc, bool valid) {
  const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int bytes = valid ? 4 : 0;  // 0 source bytes -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(gsrc), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Rectangle of the CTA's voxel box in view V (band-local rows); uncached if
// it does not fit or the box reaches behind the source.
__device__ __forceinline__ BsRect bs_rect(const ConeVoxView &V, const BpParams &p, float x0, float x1,
                                          float y0, float y1, float z0, float z1) {
  float cmin = 1e30f, cmax = -1e30f, rmin = 1e30f, rmax = -1e30f;
  bool behind = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float x = (i & 1) ? x1 : x0, y = (i & 2) ? y1 : y0, z = (i & 4) ? z1 : z0;
    const float w = fmaf(V.w[0], x, fmaf(V.w[1], y, fmaf(V.w[2], z, V.w[3])));
    behind |= !(w > (float)kTiny);
    const float rw = 1.f / w;
    const float fc = fmaf(fmaf(V.a[0], x, fmaf(V.a[1], y, fmaf(V.a[2], z, V.a[3]))), rw, p.cu);
    const float fr = fmaf(fmaf(V.b[0], x, fmaf(V.b[1], y, fmaf(V.b[2], z, V.b[3]))), rw, p.cv);
    cmin = fminf(cmin, fc);
    cmax = fmaxf(cmax, fc);
    rmin = fminf(rmin, fr);
    rmax = fmaxf(rmax, fr);
  }
  BsRect R;
  // taps floor(f) and floor(f)+1, plus one pixel of rounding margin each side
  R.c0 = (int)floorf(cmin) - 1;
  R.r0 = (int)floorf(rmin) - 1;
  R.w = (int)floorf(cmax) + 3 - R.c0;
  R.h = (int)floorf(rmax) + 3 - R.r0;
  if (behind || R.w <= 0 || R.h <= 0 || R.w * R.h > kBsCap || !(cmax - cmin < 1e6f) ||
      !(rmax - rmin < 1e6f)) {
    R.w = 0;
    R.h = 0;
  }
  return R;
}

template <bool WEIGHTED>
__global__ void __launch_bounds__(kBsTX *kBsTY, 2) cone_bp_smem_kernel(const BpParams p) {
  extern __shared__ float smem_bs[];
  float *tiles = smem_bs;  // [2][kBsNV][kBsCap]
  __shared__ ConeVoxView sv[2][kBsNV];
  __shared__ BsRect rect[2][kBsNV];
  const int tx = threadIdx.x & (kBsTX - 1), ty = threadIdx.x / kBsTX;
  const int ix = blockIdx.x * kBsTX + tx;
  const int iy = blockIdx.y * kBsTY + ty;
  const int zl0 = blockIdx.z * kBsZB;
  const bool active = ix < p.nx && iy < p.ny;
  const float xc = (float)ix - p.cx, yc = (float)iy - p.cy;
  const float zc0 = (float)(p.z_begin + zl0) - p.cz;
  // the CTA's voxel box in centred index units (clipped to the volume)
  const float bx0 = (float)(blockIdx.x * kBsTX) - p.cx;
  const float bx1 = (float)(min((int)(blockIdx.x + 1) * kBsTX, p.nx) - 1) - p.cx;
  const float by0 = (float)(blockIdx.y * kBsTY) - p.cy;
  const float by1 = (float)(min((int)(blockIdx.y + 1) * kBsTY, p.ny) - 1) - p.cy;
  const float bz1 = (float)(p.z_begin + min(zl0 + kBsZB, p.z_count) - 1) - p.cz;
  const int tid = threadIdx.x;
  const int nbatch = (p.n_views + kBsNV - 1) / kBsNV;

  float acc[kBsZB];
#pragma unroll
  for (int k = 0; k < kBsZB; ++k) acc[k] = 0.f;

  // stage batch `bi` into buffer `buf` (views, rectangles, async tile copies)
  auto stage = [&](int bi, int buf) {
    const int v0 = bi * kBsNV;
    if (tid < kBsNV) {
      const int v = v0 + tid;
      if (v < p.n_views) {
        const ConeVoxView V = p.views[v];
        sv[buf][tid] = V;
        rect[buf][tid] = bs_rect(V, p, bx0, bx1, by0, by1, zc0, bz1);
      } else {
        rect[buf][tid] = BsRect{0, 0, 0, 0};
      }
    }
    __syncthreads();
    for (int j = 0; j < kBsNV; ++j) {
      const BsRect R = rect[buf][j];
      if (R.w == 0) continue;
      const float *src = p.sino + (long long)(v0 + j) * p.view_stride;
      float *dst = tiles + (buf * kBsNV + j) * kBsCap;
      const int n = R.w * R.h;
      for (int e = tid; e < n; e += kBsTX * kBsTY) {
        const int rr = R.r0 + e / R.w, cc = R.c0 + e % R.w;
        const bool in = (unsigned)rr < (unsigned)p.band_rows && (unsigned)cc < (unsigned)p.cols;
        cp_async4(dst + e, in ? src + (long long)rr * p.cols + cc : src, in);
      }
    }
    cp_async_commit();
  };

  stage(0, 0);
  for (int bi = 0; bi < nbatch; ++bi) {
    const int buf = bi & 1;
    if (bi + 1 < nbatch) {
      __syncthreads();  // buffer buf^1 is no longer read (previous iteration)
      stage(bi + 1, buf ^ 1);
      cp_async_wait_prev();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    if (!active) continue;
    const int v0 = bi * kBsNV;
    for (int j = 0; j < kBsNV; ++j) {
      if (v0 + j >= p.n_views) break;
      const ConeVoxView &V = sv[buf][j];
      const BsRect R = rect[buf][j];
      const float a0 = fmaf(V.a[0], xc, fmaf(V.a[1], yc, fmaf(V.a[2], zc0, V.a[3])));
      const float b0 = fmaf(V.b[0], xc, fmaf(V.b[1], yc, fmaf(V.b[2], zc0, V.b[3])));
      const float w0 = fmaf(V.w[0], xc, fmaf(V.w[1], yc, fmaf(V.w[2], zc0, V.w[3])));
      if (!(w0 > (float)kTiny)) continue;
      const float rw = 1.f / w0;
      const float fc = fmaf(a0, rw, p.cu);
      const float flc = floorf(fc);
      float q = 1.f;
      if (WEIGHTED) {
        q = p.sid * rw;
        q *= q;
      }
      const float wc = fc - flc;
      const float g0 = q * (1.f - wc), g1 = q * wc;
      const float fr0 = fmaf(b0, rw, p.cv);
      const float dr = V.b[2] * rw;
      if (R.w > 0) {
        const float *t = tiles + (buf * kBsNV + j) * kBsCap;
        const int cl = min(max((int)flc - R.c0, 0), R.w - 2);
        const int hmax = R.h - 2;
#pragma unroll
        for (int k = 0; k < kBsZB; ++k) {
          const float fr = fmaf((float)k, dr, fr0);
          const float flr = floorf(fr);
          const int rl = min(max((int)flr - R.r0, 0), hmax);
          const float *e = t + rl * R.w + cl;
          const float top = fmaf(g1, e[1], g0 * e[0]);
          const float bot = fmaf(g1, e[R.w + 1], g0 * e[R.w]);
          acc[k] += fmaf(fr - flr, bot - top, top);
        }
      } else {  // uncached view: bounded global gathers (reference per-tap bounds)
        const float *s = p.sino + (long long)(v0 + j) * p.view_stride;
        const int c0 = (int)flc;
        const bool ca = (unsigned)c0 < (unsigned)p.cols, cb = (unsigned)(c0 + 1) < (unsigned)p.cols;
#pragma unroll
        for (int k = 0; k < kBsZB; ++k) {
          const float fr = fmaf((float)k, dr, fr0);
          const float flr = floorf(fr);
          const int r0 = (int)flr;
          const bool ra = (unsigned)r0 < (unsigned)p.band_rows;
          const bool rb = (unsigned)(r0 + 1) < (unsigned)p.band_rows;
          const float *e = s + (long long)r0 * p.cols + c0;
          const float t00 = (ra && ca) ? __ldg(e) : 0.f, t01 = (ra && cb) ? __ldg(e + 1) : 0.f;
          const float t10 = (rb && ca) ? __ldg(e + p.cols) : 0.f;
          const float t11 = (rb && cb) ? __ldg(e + p.cols + 1) : 0.f;
          const float top = fmaf(g1, t01, g0 * t00);
          const float bot = fmaf(g1, t11, g0 * t10);
          acc[k] += fmaf(fr - flr, bot - top, top);
        }
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < kBsZB; ++k) {
    const int zl = zl0 + k;
    if (zl < p.z_count) {
      float *o = p.out + ((long long)zl * p.ny + iy) * p.nx + ix;
      *o = p.accumulate ? *o + acc[k] : acc[k];
    }
  }
}

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

// Exact transpose of the (unweighted or weighted) voxel-driven back projector:
// splat each voxel into the detector with the same bilinear weights.
__global__ void __launch_bounds__(256)
    cone_bp_adjoint_kernel(const float *__restrict__ vol, int nx, int ny, int nz, float cx,
                           float cy, float cz, const ConeVoxView *__restrict__ views,
                           int n_views, int rows, int cols, float cu, float cv, float sid,
                           int weighted, float *__restrict__ sino) {
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
  const float wc = fc - flc, wr = fr - flr;
  float *s = sino + (long long)v * rows * cols;
  if ((unsigned)r0 < (unsigned)rows) {
    if ((unsigned)c0 < (unsigned)cols) atomicAdd(s + (long long)r0 * cols + c0, gg * (1.f - wr) * (1.f - wc));
    if ((unsigned)(c0 + 1) < (unsigned)cols) atomicAdd(s + (long long)r0 * cols + c0 + 1, gg * (1.f - wr) * wc);
  }
  if ((unsigned)(r0 + 1) < (unsigned)rows) {
    if ((unsigned)c0 < (unsigned)cols) atomicAdd(s + (long long)(r0 + 1) * cols + c0, gg * wr * (1.f - wc));
    if ((unsigned)(c0 + 1) < (unsigned)cols) atomicAdd(s + (long long)(r0 + 1) * cols + c0 + 1, gg * wr * wc);
  }
}

// Quad form ("red4", default): one REDG.F32x4 per voxel-view update into a
// detector quad buffer Qs[v][r0+1][c0+1] += (w00, w01, w10, w11) (one-texel
// margin so partially covered cells keep their in-detector taps), folded back
// into the sinogram by unquad_det_kernel.  Same weights and products as
// cone_bp_adjoint_kernel.
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

// Forward-projector algorithm: TK_FP_ALGO = ldg4z (default) | ldg4zq | ldg4m | ldg4p | ldg4 | ldg8 | ldg2 | ldg | tex | hwtex.
enum class FpAlgo { kLdg8, kLdg4, kLdg4m, kLdg4z, kLdg4zq, kLdg4p, kLdg2, kTex, kLdg, kHwTex };

static FpAlgo fp_algo() {
  const char *e = getenv("TK_FP_ALGO");
  if (e && !strcmp(e, "ldg4")) return FpAlgo::kLdg4;
  if (e && !strcmp(e, "ldg")) return FpAlgo::kLdg;
  if (e && !strcmp(e, "ldg2")) return FpAlgo::kLdg2;
  if (e && !strcmp(e, "tex")) return FpAlgo::kTex;
  if (e && !strcmp(e, "hwtex")) return FpAlgo::kHwTex;
  if (e && !strcmp(e, "ldg8")) return FpAlgo::kLdg8;
  if (e && !strcmp(e, "ldg4p")) return FpAlgo::kLdg4p;
  if (e && !strcmp(e, "ldg4m")) return FpAlgo::kLdg4m;
  if (e && !strcmp(e, "ldg4zq")) return FpAlgo::kLdg4zq;
  return FpAlgo::kLdg4z;
}

// A forward-projection plan: the two orientation copies of one volume (8-
// coefficient cells for ldg8, tap quads for ldg4), built once and reused by
// any number of view blocks (the e2e path projects view chunks so their D2H
// copies overlap the next chunk's kernel).
struct FpPlan {
  int nz, ny, nx;
  double sz, sy, sx;
  bool coef = true;   // Cell8 (ldg8) or float4 quads (ldg4 / ldg4m)
  bool diff = false;  // difference quads (ldg4m)
  bool plane = false; // b-plane difference quads (ldg4p)
  bool zfast = false; // one z-fastest copy (ldg4z coefficient cells, ldg4zq difference quads)
  unsigned zpitch = 0, xpitch = 0;  // z-fastest cell pitches
  unsigned ystride = 0;              // cells between rows y and y + 1
  bool f2 = false;                   // cells stored (A, C, B, D) for the FFMA2 march
  bool fixs = false;                 // ystride == kFpFixS (immediate-offset far-row loads)
  void *qA = nullptr, *qB = nullptr;
};

static int fp_plan_create(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                          FpPlan *plan, cudaStream_t st) {
  plan->nz = nz;
  plan->ny = ny;
  plan->nx = nx;
  plan->sz = sz;
  plan->sy = sy;
  plan->sx = sx;
  plan->coef = fp_algo() == FpAlgo::kLdg8;
  plan->diff = fp_algo() == FpAlgo::kLdg4m;
  plan->plane = fp_algo() == FpAlgo::kLdg4p;
  plan->zfast = fp_algo() == FpAlgo::kLdg4z || fp_algo() == FpAlgo::kLdg4zq;
  if (plan->zfast) plan->diff = fp_algo() == FpAlgo::kLdg4zq;
  constexpr int m2 = 2 * kFpMargin;
  const long long ncell = (long long)(nz + m2) * (ny + m2) * (nx + m2);
  const unsigned qgrid = (unsigned)std::min<long long>(ceil_div(ncell, 256), (long long)sm_count() * 32);
  const size_t esz = plan->coef ? sizeof(Cell8) : sizeof(float4);
  if (plan->zfast) {
    plan->zpitch = (unsigned)(nz + m2);
    plan->xpitch = (unsigned)(nx + m2);
    if (!plan->diff) {  // bias-free pitches: zp (1 + xp) == -1 (mod 256), zp odd; least padding
      long long best = -1;
      for (unsigned zp = (unsigned)(nz + m2) | 1u; zp < (unsigned)(nz + m2) + 128; zp += 2) {
        unsigned xp = (unsigned)(nx + m2);
        while ((zp * (1u + xp)) % 256u != 255u) ++xp;
        const long long cells = (long long)zp * xp;
        if (best < 0 || cells < best) {
          best = cells;
          plan->zpitch = zp;
          plan->xpitch = xp;
        }
      }
    }
    plan->ystride = plan->xpitch * plan->zpitch;
    const char *nofix = getenv("TK_FPZ_NOFIX");  // 1: runtime y stride (no immediate-offset far-row loads)
    if (!plan->diff && !(nofix && atoi(nofix))) {
      // fixed y stride: z pitch == 255 (mod 256) keeps the floor bias zero
      // (1 + zp + kFpFixS == 0 mod 256); the padding cells are never touched, so
      // it is used whenever the padded allocation stays below 8 GB
      const unsigned zpf = (unsigned)(nz + m2) + (255u - (unsigned)(nz + m2) % 256u);
      const unsigned long long xz = (unsigned long long)(nx + m2) * zpf;
      if (xz <= kFpFixS && (unsigned long long)(ny + m2) * kFpFixS * sizeof(float4) <= (8ull << 30)) {
        plan->zpitch = zpf;
        plan->xpitch = (unsigned)(nx + m2);
        plan->ystride = kFpFixS;
        plan->fixs = true;
      }
    }
    const long long nz_cells = (long long)(ny + m2) * plan->ystride;
    if (nz_cells >= (1LL << 32)) return fail_arg("tk_forward_cone_3d: volume too large for 32-bit cell indices");
    TK_TRY_CUDA(cudaMallocAsync(&plan->qA, esz * nz_cells, st));
    dim3 tg(ceil_div(nz + 2 * kFpMargin, 32), ceil_div(nx + 2 * kFpMargin, 32), ny + 2 * kFpMargin);
    if (plan->diff) {  // quads (ldg4zq)
      quad_volume_z_kernel<<<tg, 256, 0, st>>>(vol, nz, ny, nx, static_cast<float4 *>(plan->qA));
      TK_LAUNCHED("quad_volume_z_kernel");
    } else {  // coefficient cells (ldg4z)
      const char *f2e = getenv("TK_FPZ_F2");  // 1 (default): FFMA2 / FADD2 pair march
      const char *rbe = getenv("TK_FPZ_RB");  // the pair (A, C, B, D) layout is read only by RB = 8 kernels
      plan->f2 = plan->fixs && !(f2e && !atoi(f2e)) && !(rbe && atoi(rbe) != 8);
      coef_volume_z_kernel<<<tg, 256, 0, st>>>(vol, nz, ny, nx, static_cast<float4 *>(plan->qA), (int)plan->zpitch,
                                               (long long)plan->ystride, plan->f2 ? 1 : 0);
      TK_LAUNCHED("coef_volume_z_kernel");
    }
    return TK_OK;
  }
  TK_TRY_CUDA(cudaMallocAsync(&plan->qA, esz * ncell, st));
  TK_TRY_CUDA(cudaMallocAsync(&plan->qB, esz * ncell, st));
  for (int sw = 0; sw < 2; ++sw) {
    void *dst = sw ? plan->qB : plan->qA;
    if (plan->coef) {
      coef_volume_kernel<<<qgrid, 256, 0, st>>>(vol, nz, ny, nx, sw, static_cast<Cell8 *>(dst));
      TK_LAUNCHED("coef_volume_kernel");
    } else if (plan->plane) {
      plane_quad_volume_kernel<<<qgrid, 256, 0, st>>>(vol, nz, ny, nx, sw, static_cast<float4 *>(dst));
      TK_LAUNCHED("plane_quad_volume_kernel");
    } else {
      const int na = sw ? ny : nx, nb = sw ? nx : ny;
      dim3 tg(ceil_div(na + 2 * kFpMargin, 32), ceil_div(nb + 2 * kFpMargin, 32), nz + 2 * kFpMargin);
      if (sw)
        quad_volume_tiled_kernel<true><<<tg, 256, 0, st>>>(vol, nz, ny, nx, static_cast<float4 *>(dst), plan->diff);
      else
        quad_volume_tiled_kernel<false><<<tg, 256, 0, st>>>(vol, nz, ny, nx, static_cast<float4 *>(dst), plan->diff);
      TK_LAUNCHED("quad_volume_tiled_kernel");
    }
  }
  return TK_OK;
}

static void fp_plan_free(FpPlan *plan, cudaStream_t st) {
  if (plan->qA) cudaFreeAsync(plan->qA, st);
  if (plan->qB) cudaFreeAsync(plan->qB, st);
  plan->qA = plan->qB = nullptr;
}

// Per-view constants of the orientation-copy kernels (forward and its transpose).
static std::vector<Fp2View> fp2_views(const double *sources, const double *minv, int n_views, double sx,
                                      double sy) {
  std::vector<Fp2View> hv(n_views);
  const char *fce = getenv("TK_FP_FACE");  // 1 (default): orientation copy per ray from its entry face
  const int face_copy = fce ? atoi(fce) : 1;
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].ray.src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].ray.minv[j] = minv[9 * i + j];
    // detector u direction (column 0 of M^-1) in voxel units picks the copy
    const double ux = fabs(minv[9 * i + 0] / sx), uy = fabs(minv[9 * i + 3] / sy);
    hv[i].swap = uy > ux ? 1 : 0;
    hv[i].face_copy = face_copy;
  }
  return hv;
}

static int fp_plan_project(const FpPlan &pl, const double *sources, const double *minv, int n_views,
                           int rows, int cols, double step, float *out, cudaStream_t st) {
  const std::vector<Fp2View> hv = fp2_views(sources, minv, n_views, pl.sx, pl.sy);
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(Fp2View) * n_views, st));
  dim3 block(kFp2BX, kFp2BY);
  const char *wre = getenv("TK_FP_WR");  // detector rows per warp (1, 4 or 8; ldg4 / ldg4m only)
  const int wr = (!pl.coef && wre) ? atoi(wre) : 1;
  const bool wide = wr == 4 || wr == 8;
  const int bc = wide ? kFp2BX * kFp2BY / wr : kFp2BX, br = wide ? wr : kFp2BY;
  const long long nblocks = (long long)ceil_div(cols, bc) * ceil_div(rows, br) * n_views;
  if (nblocks >= (1LL << 31)) return fail_arg("tk_forward_cone_3d: problem too large for one launch");
  const char *mb = getenv("TK_FP2_MINB");  // 8, 10 or 12 resident CTAs per SM
  const int minb = mb ? atoi(mb) : 12;  // 12 CTAs x 128 threads (<= 40 regs): measured best for ldg4
  if (pl.coef) {
    auto kern = minb >= 12 ? cone_fp8_kernel<12> : (minb >= 10 ? cone_fp8_kernel<10> : cone_fp8_kernel<8>);
    kern<<<(unsigned)nblocks, block, 0, st>>>(static_cast<const Cell8 *>(pl.qA), static_cast<const Cell8 *>(pl.qB),
                                              pl.nx, pl.ny, pl.nz, pl.sx, pl.sy, pl.sz, dviews.as<Fp2View>(), rows,
                                              cols, n_views, step, out);
    TK_LAUNCHED("cone_fp8_kernel");
  } else if (pl.zfast) {
    const char *rbe = getenv("TK_FPZ_RB");  // detector rows per CTA band: 8 (default), 16, 32
    const int rbz = rbe ? atoi(rbe) : 8;
    const char *vge = getenv("TK_FPZ_VG");  // consecutive views per CTA: 4 (default), 1, 2, 6, 8
    // default: 8 views per CTA for long orbits (0.7 % over 4 at cfg4), 4 for short view blocks
    int vgz = (rbz != 8 || pl.diff) ? 1 : (vge ? atoi(vge) : (pl.f2 && n_views >= 128 ? 8 : 4));
    // only instantiated (views-per-CTA, kernel) combinations: the grid must match the kernel's VG
    if (pl.f2 ? !(vgz == 2 || vgz == 4 || vgz == 8) : !(vgz == 1 || vgz == 2 || vgz == 4 || vgz == 6)) vgz = 4;
    if (rbz != 8 || pl.diff) vgz = 1;
    const long long nbz = (long long)ceil_div(cols, 128 / rbz) * ceil_div(rows, rbz) * ceil_div(n_views, vgz);
    if (nbz >= (1LL << 31)) return fail_arg("tk_forward_cone_3d: problem too large for one launch");
    auto kern = pl.diff ? (minb >= 12 ? cone_fp4z_kernel<12, false> : cone_fp4z_kernel<10, false>)
                        : (minb >= 12 ? cone_fp4z_kernel<12, true>
                                      : (minb >= 10 ? cone_fp4z_kernel<10, true> : cone_fp4z_kernel<8, true>));
    if (!pl.diff && rbz == 16) kern = cone_fp4z_kernel<12, true, 16>;
    if (!pl.diff && rbz == 32) kern = cone_fp4z_kernel<12, true, 32>;
    if (!pl.diff && vgz == 2) kern = cone_fp4z_kernel<12, true, 8, 2>;
    if (!pl.diff && vgz == 4)
      // f2: 32 registers, 4 CTAs x 512 threads = 64 warps/SM (small set-up spills; 427 vs 435 ms at 48 warps)
      kern = pl.f2 ? ((mb && minb != 16) ? cone_fp4z_kernel<12, true, 8, 4, true, true>
                                         : cone_fp4z_kernel<16, true, 8, 4, true, true>)
                   : (pl.fixs ? cone_fp4z_kernel<12, true, 8, 4, true> : cone_fp4z_kernel<12, true, 8, 4>);
    if (!pl.diff && vgz == 6) kern = cone_fp4z_kernel<12, true, 8, 6>;
    if (pl.f2 && vgz == 8) kern = cone_fp4z_kernel<16, true, 8, 8, true, true>;
    if (pl.f2 && vgz == 2) kern = cone_fp4z_kernel<16, true, 8, 2, true, true>;
    kern<<<(unsigned)nbz, 128 * (pl.diff ? 1 : vgz), 0, st>>>(static_cast<const float4 *>(pl.qA), pl.nx, pl.ny,
                                                              pl.nz, pl.sx, pl.sy, pl.sz, dviews.as<Fp2View>(), rows,
                                                              cols, n_views, step, out, pl.zpitch, pl.ystride);
    TK_LAUNCHED("cone_fp4z_kernel");
  } else if (pl.plane) {
    auto kern = mb && minb >= 12 ? cone_fp4p_kernel<12> : cone_fp4p_kernel<10>;  // 10: no spills (measured best)
    kern<<<(unsigned)nblocks, block, 0, st>>>(static_cast<const float4 *>(pl.qA), static_cast<const float4 *>(pl.qB),
                                              pl.nx, pl.ny, pl.nz, pl.sx, pl.sy, pl.sz, dviews.as<Fp2View>(), rows,
                                              cols, n_views, step, out);
    TK_LAUNCHED("cone_fp4p_kernel");
  } else {
    const bool magic = pl.diff;  // ldg4m: FADD.RM floors + difference quads
    auto kern = minb >= 12 ? (magic ? cone_fp4_kernel<12, true> : cone_fp4_kernel<12, false>)
                           : (magic ? cone_fp4_kernel<10, true> : cone_fp4_kernel<10, false>);
    if (magic && wr == 4) kern = cone_fp4_kernel<12, true, 4>;
    if (magic && wr == 8) kern = cone_fp4_kernel<12, true, 8>;
    kern<<<(unsigned)nblocks, block, 0, st>>>(static_cast<const float4 *>(pl.qA), static_cast<const float4 *>(pl.qB),
                                              pl.nx, pl.ny, pl.nz, pl.sx, pl.sy, pl.sz, dviews.as<Fp2View>(), rows,
                                              cols, n_views, step, out);
    TK_LAUNCHED("cone_fp4_kernel");
  }
  return TK_OK;
}

static int launch_fp4(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                      const double *sources, const double *minv, int n_views, int rows, int cols,
                      double step, float *out, cudaStream_t st) {
  if (fp_use_mirror(sources, minv, n_views, rows, nz, ny, nx))
    return launch_fp_mirror(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, out, st);
  FpPlan plan;
  int rc = fp_plan_create(vol, nz, ny, nx, sz, sy, sx, &plan, st);
  if (rc == TK_OK) rc = fp_plan_project(plan, sources, minv, n_views, rows, cols, step, out, st);
  fp_plan_free(&plan, st);
  return rc;
}

static int launch_fp2(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                      const double *sources, const double *minv, int n_views, int rows, int cols,
                      double step, float *out, cudaStream_t st) {
  std::vector<Fp2View> hv(n_views);
  bool need_a = false, need_b = false;
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].ray.src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].ray.minv[j] = minv[9 * i + j];
    // detector u direction (column 0 of M^-1) in voxel units
    const double ux = fabs(minv[9 * i + 0] / sx), uy = fabs(minv[9 * i + 3] / sy);
    hv[i].swap = uy > ux ? 1 : 0;
    hv[i].face_copy = 0;
    (hv[i].swap ? need_b : need_a) = true;
  }
  Scratch dviews, volA, volB;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(Fp2View) * n_views, st));
  constexpr int m2 = 2 * kFpMargin;
  const long long npad = (long long)(nz + m2) * (ny + m2) * (nx + m2);
  dim3 tg(ceil_div(nx + m2, 32), ceil_div(ny + m2, 32), nz + m2);
  if (need_a) {
    TK_TRY_CUDA(volA.alloc(sizeof(float) * npad, st));
    pad_margin_kernel<<<tg, dim3(32, 8), 0, st>>>(vol, nz, ny, nx, 0, volA.as<float>());
    TK_LAUNCHED("pad_margin_kernel");
  }
  if (need_b) {
    TK_TRY_CUDA(volB.alloc(sizeof(float) * npad, st));
    pad_margin_kernel<<<tg, dim3(32, 8), 0, st>>>(vol, nz, ny, nx, 1, volB.as<float>());
    TK_LAUNCHED("pad_margin_kernel");
  }
  dim3 block(kFp2BX, kFp2BY);
  // TK_FP2_RAYS: rays per thread (1 or 2); TK_FP2_MINB: min resident CTAs per SM
  // (register cap) -- 10 (default), 12, 16
  const char *rp = getenv("TK_FP2_RAYS");
  const int rays = rp ? atoi(rp) : 1;
  const char *mb = getenv("TK_FP2_MINB");
  const int minb = mb ? atoi(mb) : 10;
  const long long nblocks =
      (long long)ceil_div(cols, kFp2BX) * ceil_div(rows, kFp2BY * (rays == 2 ? 2 : 1)) * n_views;
  if (nblocks >= (1LL << 31)) return fail_arg("tk_forward_cone_3d: problem too large for one launch");
  auto kern = rays == 2 ? (minb >= 12 ? cone_fp2r_kernel<12> : (minb >= 8 ? cone_fp2r_kernel<8> : cone_fp2r_kernel<6>))
                        : (minb >= 16 ? cone_fp2_kernel<16> : (minb >= 12 ? cone_fp2_kernel<12> : cone_fp2_kernel<10>));
  kern<<<(unsigned)nblocks, block, 0, st>>>(volA.as<float>(), volB.as<float>(), nx, ny, nz, sx, sy, sz,
                                            dviews.as<Fp2View>(), rows, cols, n_views, step, out);
  TK_LAUNCHED("cone_fp2_kernel");
  return TK_OK;
}

// A^T y by quad scatter (cone_fp_adjoint4_kernel) + fold (unquad_tiled_kernel).
// Upper bound on the number of step-sized contributions one voxel tap can
// receive over all views of a forward-projection transpose: per view, the rays
// that can pass within the tap's support (a ball of radius rho = sqrt(3) s_max
// around it) times the samples each such ray places in it.  Rays diverge from
// the source, so at distance >= dmin (source to the volume box) adjacent
// pixels' rays are >= dmin * alpha apart, alpha = the smallest angle between
// adjacent pixels' rays, attained at a detector corner for a flat detector
// (halved for safety).  Returns +inf when a source lies inside the box.
static double fp_adjoint_tap_count_bound(const double *sources, const double *minv, int n_views, int rows, int cols,
                                         int nz, int ny, int nx, double sz, double sy, double sx, double step) {
  const double h[3] = {(nx + 1) * sx / 2.0, (ny + 1) * sy / 2.0, (nz + 1) * sz / 2.0};
  const double rho = std::sqrt(3.0) * std::max(sx, std::max(sy, sz));
  const double samples = 2.0 * rho / step + 2.0;
  double total = 0.0;
  for (int i = 0; i < n_views; ++i) {
    const double *s = sources + 3 * i, *m = minv + 9 * i;
    double d2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double e = std::max(0.0, std::fabs(s[k]) - h[k]);
      d2 += e * e;
    }
    const double dmin = std::sqrt(d2);
    if (!(dmin > 0.0)) return INFINITY;
    auto dir = [&](double c, double r, double out[3]) {
      for (int k = 0; k < 3; ++k) out[k] = m[3 * k] * c + m[3 * k + 1] * r + m[3 * k + 2];
      const double n = std::sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
      for (int k = 0; k < 3; ++k) out[k] /= n;
    };
    auto angle = [](const double a[3], const double b[3]) {
      const double cx = a[1] * b[2] - a[2] * b[1], cy = a[2] * b[0] - a[0] * b[2], cz = a[0] * b[1] - a[1] * b[0];
      return std::atan2(std::sqrt(cx * cx + cy * cy + cz * cz), a[0] * b[0] + a[1] * b[1] + a[2] * b[2]);
    };
    double au = INFINITY, av = INFINITY;
    for (int cc = 0; cc < 2; ++cc)
      for (int rr = 0; rr < 2; ++rr) {
        const double c = cc ? cols - 1 : 0, r = rr ? rows - 1 : 0;
        double d[3], du[3], dv[3];
        dir(c, r, d);
        dir(c + (cc ? -1 : 1), r, du);
        dir(c, r + (rr ? -1 : 1), dv);
        au = std::min(au, angle(d, du));
        av = std::min(av, angle(d, dv));
      }
    au *= 0.5;
    av *= 0.5;
    const double nu = cols > 1 ? 2.0 * rho / (dmin * au) + 2.0 : 1.0;
    const double nv = rows > 1 ? 2.0 * rho / (dmin * av) + 2.0 : 1.0;
    total += nu * nv * samples;
  }
  return total;
}

// Deterministic A^T: fixed-point scale 2^e from max |y| and the geometry's tap
// contribution bound, so that no tap sum can overflow int64 (each contribution
// <= |y| step).
static int launch_fp_adjoint_det(const float *sino, int nz, int ny, int nx, double sz, double sy, double sx,
                                 const std::vector<Fp2View> &hv, Scratch &dviews, int n_views, int rows, int cols,
                                 double step, double tap_count, float *vol, cudaStream_t st) {
  constexpr int m2 = 2 * kFpMargin;
  const long long ncell = (long long)(nz + m2) * (ny + m2) * (nx + m2);
  const long long nsino = (long long)n_views * rows * cols;
  Scratch dmax, qA, qB;
  TK_TRY_CUDA(dmax.alloc(sizeof(unsigned), st));
  TK_TRY_CUDA(cudaMemsetAsync(dmax.ptr, 0, sizeof(unsigned), st));
  absmax_kernel<<<(unsigned)std::min<long long>(ceil_div(nsino, 256), (long long)sm_count() * 8), 256, 0, st>>>(
      sino, nsino, dmax.as<unsigned>());
  TK_LAUNCHED("absmax_kernel");
  unsigned bits = 0;
  TK_TRY_CUDA(cudaMemcpyAsync(&bits, dmax.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  TK_TRY_CUDA(cudaStreamSynchronize(st));
  float ymax;
  std::memcpy(&ymax, &bits, sizeof(float));
  if (!(ymax > 0.f) || !std::isfinite(ymax)) {
    TK_TRY_CUDA(cudaMemsetAsync(vol, 0, sizeof(float) * (size_t)nz * ny * nx, st));
    return std::isfinite(ymax) ? TK_OK : fail_arg("tk_forward_cone_3d_adjoint: non-finite sinogram");
  }
  if (!std::isfinite(tap_count))
    return fail_arg("tk_forward_cone_3d_adjoint: deterministic mode needs every source outside the volume");
  const double bound = (double)ymax * step * tap_count;
  const int e = std::min(100, (int)std::floor(62.0 - std::log2(bound)));
  const float scale = std::ldexp(1.0f, e);
  TK_TRY_CUDA(qA.alloc(32 * ncell, st));
  TK_TRY_CUDA(qB.alloc(32 * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qA.ptr, 0, 32 * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qB.ptr, 0, 32 * ncell, st));
  const long long nbz = (long long)ceil_div(cols, 16) * ceil_div(rows, kFpzRows) * n_views;
  if (nbz >= (1LL << 31)) return fail_arg("tk_forward_cone_3d_adjoint: problem too large for one launch");
  cone_fp_adjoint4z_kernel<8, true><<<(unsigned)nbz, 128, 0, st>>>(sino, qA.ptr, qB.ptr, nx, ny, nz, sx, sy, sz,
                                                                   dviews.as<Fp2View>(), rows, cols, n_views, step,
                                                                   scale);
  TK_LAUNCHED("cone_fp_adjoint4z_kernel");
  const long long nv = (long long)nz * ny * nx;
  unquad_fx_kernel<<<(unsigned)std::min<long long>(ceil_div(nv, 256), (long long)sm_count() * 16), 256, 0, st>>>(
      qA.as<unsigned long long>(), qB.as<unsigned long long>(), nz, ny, nx, std::ldexp(1.0, -e), vol);
  TK_LAUNCHED("unquad_fx_kernel");
  return TK_OK;
}

static int launch_fp_adjoint4(const float *sino, int nz, int ny, int nx, double sz, double sy, double sx,
                              const double *sources, const double *minv, int n_views, int rows, int cols,
                              double step, float *vol, cudaStream_t st, bool zfast, bool deterministic = false) {
  const std::vector<Fp2View> hv = fp2_views(sources, minv, n_views, sx, sy);
  Scratch dviews, qA, qB;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(Fp2View) * n_views, st));
  constexpr int m2 = 2 * kFpMargin;
  const long long ncell = (long long)(nz + m2) * (ny + m2) * (nx + m2);
  if (ncell >= (1LL << 32)) return fail_arg("tk_forward_cone_3d_adjoint: volume too large for 32-bit cell indices");
  if (deterministic)
    return launch_fp_adjoint_det(sino, nz, ny, nx, sz, sy, sx, hv, dviews, n_views, rows, cols, step,
                                 fp_adjoint_tap_count_bound(sources, minv, n_views, rows, cols, nz, ny, nx, sz, sy,
                                                            sx, step),
                                 vol, st);
  TK_TRY_CUDA(qA.alloc(sizeof(float4) * ncell, st));
  TK_TRY_CUDA(qB.alloc(sizeof(float4) * ncell, st));
  if (zfast) {
    TK_TRY_CUDA(cudaMemsetAsync(qA.ptr, 0, sizeof(float4) * ncell, st));
    TK_TRY_CUDA(cudaMemsetAsync(qB.ptr, 0, sizeof(float4) * ncell, st));
    const long long nbz = (long long)ceil_div(cols, 16) * ceil_div(rows, kFpzRows) * n_views;
    if (nbz >= (1LL << 31)) return fail_arg("tk_forward_cone_3d_adjoint: problem too large for one launch");
    cone_fp_adjoint4z_kernel<8><<<(unsigned)nbz, 128, 0, st>>>(sino, qA.ptr, qB.ptr, nx, ny, nz, sx, sy, sz,
                                                               dviews.as<Fp2View>(), rows, cols, n_views, step, 1.f);
    TK_LAUNCHED("cone_fp_adjoint4z_kernel");
    unquad_z_kernel<<<dim3(ceil_div(nz, 32), ceil_div(nx, 32), ny), 256, 0, st>>>(qA.as<float4>(), nz, ny, nx,
                                                                                 vol);
    TK_LAUNCHED("unquad_z_kernel");
    unquad_zx_kernel<<<dim3(ceil_div(nz, 32), ceil_div(nx, 32), ny), 256, 0, st>>>(qB.as<float4>(), nz, ny, nx,
                                                                                  vol);
    TK_LAUNCHED("unquad_zx_kernel");
    return TK_OK;
  }
  TK_TRY_CUDA(cudaMemsetAsync(qA.ptr, 0, sizeof(float4) * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qB.ptr, 0, sizeof(float4) * ncell, st));
  const long long nblocks = (long long)ceil_div(cols, kFp2BX) * ceil_div(rows, kFp2BY) * n_views;
  if (nblocks >= (1LL << 31)) return fail_arg("tk_forward_cone_3d_adjoint: problem too large for one launch");
  cone_fp_adjoint4_kernel<8><<<(unsigned)nblocks, dim3(kFp2BX, kFp2BY), 0, st>>>(
      sino, qA.as<float4>(), qB.as<float4>(), nx, ny, nz, sx, sy, sz, dviews.as<Fp2View>(), rows, cols, n_views,
      step);
  TK_LAUNCHED("cone_fp_adjoint4_kernel");
  unquad_tiled_kernel<false><<<dim3(ceil_div(nx, 32), ceil_div(ny, 32), nz), 256, 0, st>>>(qA.as<float4>(), nz, ny,
                                                                                          nx, vol, 0);
  TK_LAUNCHED("unquad_tiled_kernel");
  unquad_tiled_kernel<true><<<dim3(ceil_div(ny, 32), ceil_div(nx, 32), nz), 256, 0, st>>>(qB.as<float4>(), nz, ny,
                                                                                         nx, vol, 1);
  TK_LAUNCHED("unquad_tiled_kernel");
  return TK_OK;
}

static int launch_fp(const float *vol, int nz, int ny, int nx, double sz, double sy,
                     double sx, const double *sources, const double *minv, int n_views,
                     int rows, int cols, double step, float *out, cudaStream_t st,
                     bool adjoint) {
  // transpose: red4z (default, z-fastest quad scatter) | red4 (orientation-copy quads) | scatter (scalar atomics)
  const char *ta = getenv("TK_FPT_ALGO");
  if (adjoint && !(ta && !strcmp(ta, "scatter")))
    return launch_fp_adjoint4(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, out, st,
                              !(ta && !strcmp(ta, "red4")));
  std::vector<ConeRayView> hv(n_views);
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].minv[j] = minv[9 * i + j];
  }
  Scratch dviews, volp;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeRayView) * n_views, st));
  dim3 block(kFpBX, kFpBY);
  dim3 grid(ceil_div(cols, kFpBX), ceil_div(rows, kFpBY), n_views);
  const FpAlgo algo = fp_algo();
  if (!adjoint && (algo == FpAlgo::kLdg8 || algo == FpAlgo::kLdg4 || algo == FpAlgo::kLdg4m || algo == FpAlgo::kLdg4p ||
                   algo == FpAlgo::kLdg4z || algo == FpAlgo::kLdg4zq))
    return launch_fp4(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, out, st);
  if (!adjoint && algo == FpAlgo::kLdg2)
    return launch_fp2(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, out, st);
  if (!adjoint && algo != FpAlgo::kLdg) {
    TexLease lease;
    const bool hw = algo == FpAlgo::kHwTex;
    TK_TRY_CUDA(tex_acquire(vol, nx, ny, nz, hw ? TexKind::kVolumeLinear : TexKind::kLayeredPoint,
                            st, lease));
    if (hw)
      cone_fp_hwtex_kernel<<<grid, block, 0, st>>>(lease.tex, nx, ny, nz, sx, sy, sz,
                                                   dviews.as<ConeRayView>(), rows, cols, step, out);
    else
      cone_fp_tex_kernel<<<grid, block, 0, st>>>(lease.tex, nx, ny, nz, sx, sy, sz,
                                                 dviews.as<ConeRayView>(), rows, cols, step, out);
    tex_release(lease, st);
    TK_LAUNCHED(hw ? "cone_fp_hwtex_kernel" : "cone_fp_tex_kernel");
    return TK_OK;
  }
  const long long npad = (long long)(nz + 2) * (ny + 2) * (nx + 2);
  TK_TRY_CUDA(volp.alloc(sizeof(float) * npad, st));
  const unsigned pgrid = (unsigned)std::min<long long>(ceil_div(npad, 256), 148LL * 32);
  if (!adjoint) {
    pad3d_kernel<<<pgrid, 256, 0, st>>>(vol, nz, ny, nx, volp.as<float>());
    TK_LAUNCHED("pad3d_kernel");
    cone_fp_kernel<<<grid, block, 0, st>>>(volp.as<float>(), nx, ny, nz, sx, sy, sz,
                                           dviews.as<ConeRayView>(), rows, cols, step, out);
    TK_LAUNCHED("cone_fp_kernel");
  } else {
    // here `vol` is the sinogram and `out` the volume
    TK_TRY_CUDA(cudaMemsetAsync(volp.ptr, 0, sizeof(float) * npad, st));
    cone_fp_adjoint_kernel<<<grid, block, 0, st>>>(vol, nx, ny, nz, sx, sy, sz,
                                                   dviews.as<ConeRayView>(), rows, cols,
                                                   step, volp.as<float>());
    TK_LAUNCHED("cone_fp_adjoint_kernel");
    const long long nv = (long long)nz * ny * nx;
    crop3d_kernel<<<(unsigned)std::min<long long>(ceil_div(nv, 256), 148LL * 32), 256, 0, st>>>(
        volp.as<float>(), nz, ny, nx, out);
    TK_LAUNCHED("crop3d_kernel");
  }
  return TK_OK;
}

// Back-projector algorithm: TK_BP_ALGO = tma (default) | quad | coef | smem | ldg | tex | hwtex.
// tma needs a z-invariant trajectory and a detector width that is a multiple of
// 4 (16-byte TMA row pitch); otherwise quad runs.
enum class BpAlgo { kTma, kCoef, kSmem, kQuad, kLdg, kTex, kHwTex };

static BpAlgo bp_algo() {
  const char *e = getenv("TK_BP_ALGO");
  if (e && !strcmp(e, "quad")) return BpAlgo::kQuad;
  if (e && !strcmp(e, "coef")) return BpAlgo::kCoef;
  if (e && !strcmp(e, "smem")) return BpAlgo::kSmem;
  if (e && !strcmp(e, "ldg")) return BpAlgo::kLdg;
  if (e && !strcmp(e, "tex")) return BpAlgo::kTex;
  if (e && !strcmp(e, "hwtex")) return BpAlgo::kHwTex;
  return BpAlgo::kTma;
}

constexpr int kBqZB = 16;

static int launch_bp_smem(const BpParams &p, bool weighted, cudaStream_t st) {
  const size_t smem = sizeof(float) * 2 * kBsNV * kBsCap;
  static bool configured[2] = {false, false};
  if (!configured[weighted]) {
    TK_TRY_CUDA(cudaFuncSetAttribute(weighted ? cone_bp_smem_kernel<true> : cone_bp_smem_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[weighted] = true;
  }
  dim3 grid(ceil_div(p.nx, kBsTX), ceil_div(p.ny, kBsTY), ceil_div(p.z_count, kBsZB));
  if (weighted)
    cone_bp_smem_kernel<true><<<grid, kBsTX * kBsTY, smem, st>>>(p);
  else
    cone_bp_smem_kernel<false><<<grid, kBsTX * kBsTY, smem, st>>>(p);
  TK_LAUNCHED("cone_bp_smem_kernel");
  return TK_OK;
}

static int launch_bp_quad(BpParams p, bool weighted, bool zinv, bool coef, cudaStream_t st) {
  const long long qview = (long long)(p.band_rows + 1 + kQuadPad) * (p.cols + 1 + kQuadPad);
  const long long nq = qview * p.n_views;
  Scratch quads;
  TK_TRY_CUDA(quads.alloc(sizeof(float4) * nq, st));
  const unsigned qgrid = (unsigned)std::min<long long>(ceil_div(nq, 256), (long long)sm_count() * 32);
  if (coef) {
    coefify_kernel<<<qgrid, 256, 0, st>>>(p.sino, p.n_views, p.band_rows, p.cols, quads.as<float4>());
    TK_LAUNCHED("coefify_kernel");
  } else {
    quadify_kernel<<<qgrid, 256, 0, st>>>(p.sino, p.n_views, p.band_rows, p.cols, quads.as<float4>());
    TK_LAUNCHED("quadify_kernel");
  }
  dim3 block(kBqBX, kBqBY);
  dim3 grid(ceil_div(p.nx, kBqBX), ceil_div(p.ny, kBqBY), ceil_div(p.z_count, kBqZB));
  const float4 *q = quads.as<float4>();
  const int sel = (zinv ? 2 : 0) + (weighted ? 1 : 0);
  if (coef) {
    if (sel == 3) cone_bp_coef_kernel<kBqZB, true, true><<<grid, block, 0, st>>>(p, q);
    else if (sel == 2) cone_bp_coef_kernel<kBqZB, true, false><<<grid, block, 0, st>>>(p, q);
    else if (sel == 1) cone_bp_coef_kernel<kBqZB, false, true><<<grid, block, 0, st>>>(p, q);
    else cone_bp_coef_kernel<kBqZB, false, false><<<grid, block, 0, st>>>(p, q);
    TK_LAUNCHED("cone_bp_coef_kernel");
  } else if (!getenv("TK_BP_Q42") || atoi(getenv("TK_BP_Q42")) != 0) {  // 4x2 quarter-warps (default)
    if (sel == 3) cone_bp_quad_kernel<kBqZB, true, true, true><<<grid, block, 0, st>>>(p, q);
    else if (sel == 2) cone_bp_quad_kernel<kBqZB, true, false, true><<<grid, block, 0, st>>>(p, q);
    else if (sel == 1) cone_bp_quad_kernel<kBqZB, false, true, true><<<grid, block, 0, st>>>(p, q);
    else cone_bp_quad_kernel<kBqZB, false, false, true><<<grid, block, 0, st>>>(p, q);
    TK_LAUNCHED("cone_bp_quad_kernel");
  } else {
    if (sel == 3) cone_bp_quad_kernel<kBqZB, true, true><<<grid, block, 0, st>>>(p, q);
    else if (sel == 2) cone_bp_quad_kernel<kBqZB, true, false><<<grid, block, 0, st>>>(p, q);
    else if (sel == 1) cone_bp_quad_kernel<kBqZB, false, true><<<grid, block, 0, st>>>(p, q);
    else cone_bp_quad_kernel<kBqZB, false, false><<<grid, block, 0, st>>>(p, q);
    TK_LAUNCHED("cone_bp_quad_kernel");
  }
  return TK_OK;
}

template <int ZB, bool ZINV>
static void launch_bp_t(const BpParams &p, bool weighted, BpAlgo algo, dim3 grid, dim3 block,
                        cudaStream_t st) {
  if (algo == BpAlgo::kTex) {
    if (weighted)
      cone_bp_tex_kernel<ZB, ZINV, true, false><<<grid, block, 0, st>>>(p);
    else
      cone_bp_tex_kernel<ZB, ZINV, false, false><<<grid, block, 0, st>>>(p);
  } else if (algo == BpAlgo::kHwTex) {
    if (weighted)
      cone_bp_tex_kernel<ZB, ZINV, true, true><<<grid, block, 0, st>>>(p);
    else
      cone_bp_tex_kernel<ZB, ZINV, false, true><<<grid, block, 0, st>>>(p);
  } else if (weighted) {
    cone_bp_kernel<ZB, ZINV, true><<<grid, block, 0, st>>>(p);
  } else {
    cone_bp_kernel<ZB, ZINV, false><<<grid, block, 0, st>>>(p);
  }
}

}  // namespace tk

using namespace tk;

extern "C" {

int tk_forward_cone_3d(const float *vol, int nz, int ny, int nx, double sz, double sy,
                       double sx, const double *sources, const double *minv, int n_views,
                       int rows, int cols, double step, float *out, void *stream) {
  clear_error();
  if (!vol || !out || !sources || !minv) return fail_arg("tk_forward_cone_3d: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_forward_cone_3d: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0 && step > 0)) return fail_arg("tk_forward_cone_3d: spacing/step must be > 0");
  if (n_views > 65535) return fail_arg("tk_forward_cone_3d: more than 65535 views per call");
  return launch_fp(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, out,
                   as_stream(stream), false);
}

int tk_fp_plan_create(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                      void **plan, void *stream) {
  clear_error();
  if (!vol || !plan) return fail_arg("tk_fp_plan_create: null pointer");
  if (nz < 1 || ny < 1 || nx < 1) return fail_arg("tk_fp_plan_create: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0)) return fail_arg("tk_fp_plan_create: spacing must be > 0");
  FpPlan *pl = new FpPlan();
  const int rc = fp_plan_create(vol, nz, ny, nx, sz, sy, sx, pl, as_stream(stream));
  if (rc != TK_OK) {
    fp_plan_free(pl, as_stream(stream));
    delete pl;
    *plan = nullptr;
    return rc;
  }
  *plan = pl;
  return TK_OK;
}

int tk_fp_plan_project(void *plan, const double *sources, const double *minv, int n_views, int rows,
                       int cols, double step, float *out, void *stream) {
  clear_error();
  if (!plan || !sources || !minv || !out) return fail_arg("tk_fp_plan_project: null pointer");
  if (n_views < 1 || rows < 1 || cols < 1 || !(step > 0))
    return fail_arg("tk_fp_plan_project: bad extent / step");
  return fp_plan_project(*reinterpret_cast<FpPlan *>(plan), sources, minv, n_views, rows, cols, step,
                         out, as_stream(stream));
}

int tk_fp_plan_destroy(void *plan, void *stream) {
  clear_error();
  if (!plan) return TK_OK;
  FpPlan *pl = reinterpret_cast<FpPlan *>(plan);
  fp_plan_free(pl, as_stream(stream));
  delete pl;
  return TK_OK;
}

int tk_forward_cone_3d_adjoint_ex(const float *sino, int n_views, int rows, int cols, const double *sources,
                                  const double *minv, int nz, int ny, int nx, double sz, double sy, double sx,
                                  double step, int deterministic, float *vol_out, void *stream) {
  clear_error();
  if (!deterministic)
    return tk_forward_cone_3d_adjoint(sino, n_views, rows, cols, sources, minv, nz, ny, nx, sz, sy, sx, step,
                                      vol_out, stream);
  if (!sino || !vol_out || !sources || !minv) return fail_arg("tk_forward_cone_3d_adjoint: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_forward_cone_3d_adjoint: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0 && step > 0)) return fail_arg("tk_forward_cone_3d_adjoint: spacing/step must be > 0");
  return launch_fp_adjoint4(sino, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, vol_out,
                            as_stream(stream), true, true);
}

int tk_forward_cone_3d_adjoint(const float *sino, int n_views, int rows, int cols,
                               const double *sources, const double *minv, int nz, int ny,
                               int nx, double sz, double sy, double sx, double step,
                               float *vol_out, void *stream) {
  clear_error();
  if (!sino || !vol_out || !sources || !minv) return fail_arg("tk_forward_cone_3d_adjoint: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_forward_cone_3d_adjoint: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0 && step > 0)) return fail_arg("tk_forward_cone_3d_adjoint: spacing/step must be > 0");
  if (n_views > 65535) return fail_arg("tk_forward_cone_3d_adjoint: more than 65535 views per call");
  return launch_fp(sino, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step,
                   vol_out, as_stream(stream), true);
}

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
  constexpr int ZB = 8;
  dim3 block(kBpBX, kBpBY);
  dim3 grid(ceil_div(nx, kBpBX), ceil_div(ny, kBpBY), ceil_div(z_count, ZB));
  p.tex = 0;
  BpAlgo algo = bp_algo();
  if (algo == BpAlgo::kSmem && zinv) return launch_bp_smem(p, weighted != 0, st);
  if (algo == BpAlgo::kTma && zinv) {
    const int rc = launch_bp_tma(p, hv.data(), weighted != 0, st);
    if (rc != -1) return rc;
  }
  if (algo == BpAlgo::kTma) algo = BpAlgo::kQuad;
  if (algo == BpAlgo::kCoef || algo == BpAlgo::kQuad || algo == BpAlgo::kSmem)
    return launch_bp_quad(p, weighted != 0, zinv, algo == BpAlgo::kCoef, st);
  if (n_views > 2048) algo = BpAlgo::kLdg;  // layered arrays hold <= 2048 layers
  TexLease lease;
  if (algo != BpAlgo::kLdg) {
    TK_TRY_CUDA(tex_acquire(sino, cols, band_rows, n_views,
                            algo == BpAlgo::kHwTex ? TexKind::kLayeredLinear : TexKind::kLayeredPoint,
                            st, lease));
    p.tex = lease.tex;
  }
  if (zinv)
    launch_bp_t<ZB, true>(p, weighted != 0, algo, grid, block, st);
  else
    launch_bp_t<ZB, false>(p, weighted != 0, algo, grid, block, st);
  if (lease.slot) tex_release(lease, st);
  TK_LAUNCHED("cone_bp_kernel");
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
  if (n_views > 65535) return fail_arg("tk_back_cone_3d_adjoint: more than 65535 views per call");
  cudaStream_t st = as_stream(stream);
  const double cu = (cols - 1) / 2.0, cv = (rows - 1) / 2.0;
  std::vector<ConeVoxView> hv;
  bool zinv = true;
  pack_bp_views(mats, n_views, sx, sy, sz, cu, cv, hv, zinv);
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeVoxView) * n_views, st));
  const long long nvox = (long long)nx * ny * nz;
  dim3 grid(ceil_div(nvox, 256), n_views);
  const char *ta = getenv("TK_BPT_ALGO");  // red4 (default: detector quads) | scatter (scalar atomics)
  if (!(ta && !strcmp(ta, "scatter"))) {
    Scratch qs;
    const size_t nq = (size_t)n_views * (rows + 1) * (cols + 1);
    TK_TRY_CUDA(qs.alloc(sizeof(float4) * nq, st));
    TK_TRY_CUDA(cudaMemsetAsync(qs.ptr, 0, sizeof(float4) * nq, st));
    cone_bp_adjoint4_kernel<<<grid, 256, 0, st>>>(vol, nx, ny, nz, (float)((nx - 1) / 2.0), (float)((ny - 1) / 2.0),
                                                  (float)((nz - 1) / 2.0), dviews.as<ConeVoxView>(), rows, cols,
                                                  (float)cu, (float)cv, (float)sid, weighted, qs.as<float4>());
    TK_LAUNCHED("cone_bp_adjoint4_kernel");
    const long long npix = (long long)n_views * rows * cols;
    unquad_det_kernel<<<(unsigned)std::min<long long>(ceil_div(npix, 256), (long long)sm_count() * 16), 256, 0, st>>>(
        qs.as<float4>(), n_views, rows, cols, sino_out);
    TK_LAUNCHED("unquad_det_kernel");
    return TK_OK;
  }
  TK_TRY_CUDA(cudaMemsetAsync(sino_out, 0, sizeof(float) * (size_t)n_views * rows * cols, st));
  cone_bp_adjoint_kernel<<<grid, 256, 0, st>>>(vol, nx, ny, nz, (float)((nx - 1) / 2.0),
                                               (float)((ny - 1) / 2.0), (float)((nz - 1) / 2.0),
                                               dviews.as<ConeVoxView>(), n_views, rows, cols,
                                               (float)cu, (float)cv, (float)sid, weighted,
                                               sino_out);
  TK_LAUNCHED("cone_bp_adjoint_kernel");
  return TK_OK;
}

}  // extern "C"
