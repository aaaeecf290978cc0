// tk_fp.cu -- cone-beam forward projection A x (ray-driven), the default path.
//
// Reference semantics: /root/reference/pkg/src/tomokit/_kernels.py:254-278
// (forward_cone_3d: one ray per detector pixel (r, c), direction M^-1 (c, r, 1)
// normalised, _clip_ray_3d on the half-extents (n + 1) s / 2) and _march_3d,
// :117-157 (sample k at t0 + (k + 1/2) step, trilinear taps of the one-voxel
// zero-padded volume, exact last partial segment, sum * step).  Per-ray set-up
// in float64 (tk_cone_fp.cuh: cone_ray_setup), the march in float32 at
// e + (k + 1/2) g (no accumulated t).
//
// Thread = one ray (two for the mirror kernel).  Quarter-warp = 8 consecutive
// detector rows of ONE column: their rays lie in one vertical plane through the
// source and share the horizontal track, so x / y cell crossings coincide and
// only z crossings are per lane; the taps are stored z-fastest so a quarter's
// cells are contiguous.  CTA = an 8-column x 8-row detector tile
// (two warps of 4 columns x 8 rows) of each of VG = 8 consecutive views (rays of
// neighbouring views near the axis share L1 lines), 4 CTAs per SM; CTA order:
// column blocks, then view groups, then 8-row bands.
//
// Cells ("coefficient cells", 16 B): cell (z, y, x) of row y holds the bilinear
// (x, z) polynomial of its four taps, stored (A, C, B, D) for FFMA2 pairs,
// A = V00, B = V01 - V00, C = V10 - V00, D = (V11 - V10) - (V01 - V00) (V_zx);
// a sample is lerp(P(cell[y]), P(cell[y + 1]), wy) with P = A + wx B + wz (C + wx D).
// Pitches make the FADD.RM floor bias vanish modulo 2^32: the cell index formed
// from the float bits of the three floors IS the element index.
//
// cone_fp_mirror_kernel (circular orbits): the ray through pixel (R-1-r, c) is
// the z mirror image of the ray through (r, c) -- same x / y track, same clip
// interval and sample parameters.  A 32-byte pair cell holds the coefficient
// cell of V and of the reflected volume Vm[z] = V[K - z] at the SAME index, so
// one thread marches both rays with one position / floor / index computation
// and one pair of 32-byte loads per cell change; the arithmetic of the two rays
// runs as FFMA2 pairs.
//
// Measured and not kept: splitting every ray into 2-6
// segments, one launch per segment, to shrink the L2 working set of the
// resident CTAs (DRAM reads 187 -> 52 GB for the mirror kernel, but +3.5 % time
// per extra segment: the march is bound by L1 / L2 latency, not DRAM), and
// staging each CTA's results in shared memory for full-segment writes (+1.6 %);
// a slab-staged variant (the CTA's bundle of rays marched slab by slab along its
// major axis from shared-memory boxes filled by cp.async.bulk, bit-identical
// results): 726 ms at 8-cell slabs, 654 ms with the copies disabled, ~410 ms
// extrapolated to infinitely thick slabs -- the per-slab CTA-wide lockstep costs
// more than the L1 misses it removes (git history: tk_fp.cu before 2026-10-17 16:00).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tk_cone_fp.cuh"

namespace tk {

constexpr int kFpCols = 16, kFpRows = 8;  // detector tile of one view per 128-thread sub-block
constexpr int kFpColsDefault = 8;         // default launch: 8-column x 8-row view tiles (64 threads)
constexpr unsigned kFpFixS = 524032u;     // fixed y stride, 16-byte cells (2047 * 256): z pitch == 255 (mod 256)
constexpr unsigned kMirS = 262138u;       // fixed y stride, 32-byte pair cells (== 250 mod 256): z pitch == 5 (mod 256)

// ---------------------------------------------------------------------------
// layouts
// ---------------------------------------------------------------------------
// 32 (z) x 32 (x) tiles of one y row: reads along x, writes along z (coalesced).
__global__ void __launch_bounds__(256) fp_cells_kernel(const float *__restrict__ vol, int nz, int ny, int nx,
                                                       float4 *__restrict__ cq, unsigned zpitch,
                                                       unsigned long long ystride) {
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
    cq[(unsigned long long)(y + m) * ystride + (unsigned long long)(x + m) * zpitch + (z + m)] =
        make_float4(A, C, B, D);
  }
}

// Pair cells (V, Vm) of rows y for padded z in [0, zcells); K = nz - 1 + 2m.
__global__ void __launch_bounds__(256) fp_mirror_cells_kernel(const float *__restrict__ vol, int nz, int ny, int nx,
                                                              float4 *__restrict__ cq, unsigned zpitch,
                                                              unsigned long long ystride, int zcells) {
  __shared__ float tile[2][33][34];  // [V, Vm][x - x0][z - z0]
  constexpr int m = kFpMargin;
  const int px = nx + 2 * m, K = nz - 1 + 2 * m;
  const int z0 = blockIdx.x * 32, x0 = blockIdx.y * 32 - m, y = (int)blockIdx.z - m;
  const bool yin = (unsigned)y < (unsigned)ny;
  for (int e = threadIdx.x; e < 2 * 33 * 33; e += 256) {
    const int s = e / (33 * 33), r = e % (33 * 33);
    const int dx = r % 33, dz = r / 33;
    const int x = x0 + dx;
    const int zp = s ? K - (z0 + dz) : z0 + dz;  // padded z of V (s = 0) or of the reflection
    const int z = zp - m;
    float val = 0.f;
    if (yin && (unsigned)z < (unsigned)nz && (unsigned)x < (unsigned)nx)
      val = __ldg(vol + ((long long)z * ny + y) * nx + x);
    tile[s][dx][dz] = val;
  }
  __syncthreads();
  const int tz = threadIdx.x & 31;
  for (int tx = threadIdx.x >> 5; tx < 32; tx += 8) {
    const int z = z0 + tz, x = x0 + tx;  // padded z, padded x - m
    if (z >= zcells || x + m >= px) continue;
    float c[2][4];
    for (int s = 0; s < 2; ++s) {
      const float v00 = tile[s][tx][tz], v01 = tile[s][tx + 1][tz], v10 = tile[s][tx][tz + 1],
                  v11 = tile[s][tx + 1][tz + 1];
      c[s][0] = v00;                        // A
      c[s][1] = v10 - v00;                  // C
      c[s][2] = v01 - v00;                  // B
      c[s][3] = (v11 - v10) - (v01 - v00);  // D
    }
    float4 *dst = cq + 2 * ((unsigned long long)(y + m) * ystride + (unsigned long long)(x + m) * zpitch + z);
    dst[0] = make_float4(c[0][0], c[1][0], c[0][1], c[1][1]);  // (A, A'), (C, C')
    dst[1] = make_float4(c[0][2], c[1][2], c[0][3], c[1][3]);  // (B, B'), (D, D')
  }
}

// ---------------------------------------------------------------------------
// march helpers
// ---------------------------------------------------------------------------
struct __align__(32) Pair4 {
  unsigned long long a, c, b, d;  // (A, A'), (C, C'), (B, B'), (D, D')
};

template <bool FIXS>
__device__ __forceinline__ void ldg_pair4(const Pair4 *p, unsigned ys, Pair4 &lo, Pair4 &hi) {
  asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(lo.a), "=l"(lo.c), "=l"(lo.b), "=l"(lo.d)
               : "l"(p));
  if (FIXS) {  // far row (y + 1) at an immediate offset: kMirS * 32 B
    asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4+8388416];"
                 : "=l"(hi.a), "=l"(hi.c), "=l"(hi.b), "=l"(hi.d)
                 : "l"(p));
  } else {
    asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(hi.a), "=l"(hi.c), "=l"(hi.b), "=l"(hi.d)
                 : "l"(elem_ptr(p, ys)));
  }
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// Row-band destinations of the fused multi-GPU forward projection (BANDS = true):
// ray (v, r, c) is stored into every rank h whose band [r0[h], r1[h]) holds row r,
// at ptr[h][(view_offset + v) * view_stride + (r - r0[h]) * cols + c].  ptr[h] is a
// peer (NVLink P2P) or local address: the stores ARE the exchange, issued ray by ray
// as the projection proceeds.
constexpr int kFpMaxDest = 16;
struct FpDests {
  float *ptr[kFpMaxDest];
  int r0[kFpMaxDest], r1[kFpMaxDest];
  int n, view_offset;
  long long view_stride;
};

// PROBE (roofline decomposition, TK_FP_PROBE; not a projector): 1 = the march with its
// cell loads but a 1-FADD "interpolation" (the access stream alone), 2 = the full
// arithmetic on cell values synthesised from the cell index instead of loaded,
// 7 = the per-ray float64 set-up alone.
template <int VG, bool FIXS, bool BANDS, int COLS = kFpCols, int PROBE = 0, int ZP = 0, bool MOVE_FREE = true,
          int UNR = 2>
__device__ __forceinline__ void fp_rays(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy,
                                        double sz, const ConeRayView *__restrict__ views, int rows, int cols,
                                        int n_views, double step, float *__restrict__ out, unsigned zpitch,
                                        unsigned ystride, const FpDests *dests) {
  constexpr int SUB = COLS * kFpRows;  // threads per view: COLS columns x 8 rows (warps of 4 x 8)
  const int ncb = (cols + COLS - 1) / COLS;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int nvg = (n_views + VG - 1) / VG;
  const int v0 = (int)(bt % nvg) * VG, rb = (int)(bt / nvg);
  const int sub = threadIdx.x / SUB, t = threadIdx.x % SUB;
  const int v = v0 + sub, c = cb * COLS + (t >> 3), r = rb * kFpRows + (t & 7);
  if (c >= cols || r >= rows || v >= n_views) return;
  float *dst = BANDS ? nullptr : out + ((long long)v * rows + r) * cols + c;
  auto store = [&](float val) {
    if (BANDS) {
#pragma unroll 1
      for (int h = 0; h < dests->n; ++h)
        if (r >= dests->r0[h] && r < dests->r1[h])
          dests->ptr[h][(long long)(dests->view_offset + v) * dests->view_stride +
                        (long long)(r - dests->r0[h]) * cols + c] = val;
    } else {
      *dst = val;
    }
  };
  RaySetup rs;
  if (!cone_ray_setup(views[v], r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    store(0.f);
    return;
  }
  if (PROBE == 7) {  // per-ray set-up only (its share of the projector's time)
    store(rs.ex + rs.gz * (float)rs.n + rs.last);
    return;
  }
  const float ex = rs.ex + (kFpMargin - 1), ey = rs.ey + (kFpMargin - 1), ez = rs.ez + (kFpMargin - 1);
  const float magic = 8388608.f;  // coordinates >= 0: floor(f) = bits(f + 2^23) - 0x4B000000
  const unsigned sys = FIXS ? kFpFixS : ystride;
  const unsigned zp = ZP ? (unsigned)ZP : zpitch;  // compile-time z pitch (fixed stride, nz + 4 <= 1023)
  const unsigned long long e2 = pk2(ex, ey), g2 = pk2(rs.gx, rs.gy), m2 = pk2(magic, magic);
  const float gz = rs.gz;
  unsigned cell = 0xffffffffu;
  float4 lo4 = make_float4(0.f, 0.f, 0.f, 0.f), hi4 = lo4;
  auto sample = [&](float kk) -> float {
    const unsigned long long fxy = ffma2(pk2(kk, kk), g2, e2);
    const float fz = fmaf(kk, gz, ez);
    const unsigned long long xxy = fadd2_rm(fxy, m2);
    const float xz = __fadd_rd(fz, magic);
    const float2 xb = upk2(xxy);
    const unsigned id = __float_as_uint(xb.y) * sys + (__float_as_uint(xb.x) * zp + __float_as_uint(xz));
    const bool changed = id != cell;
    if (!MOVE_FREE) cell = changed ? id : cell;
    if (changed) {
      if (PROBE == 2) {
        lo4.x = __uint_as_float((id & 0x7fffu) | 0x3f800000u);
        lo4 = make_float4(lo4.x, lo4.x, lo4.x, lo4.x);
        hi4 = lo4;
      } else {
        const float4 *p = elem_ptr(q, id);
        lo4 = __ldg(p);
        hi4 = __ldg(p + sys);
      }
    }
    if (MOVE_FREE) cell = id;  // == the cell of the last load: no predicated move, renamed by the unroll
    if (PROBE == 1) return lo4.x + hi4.w;
    const float2 w = upk2(fsub2(fxy, fsub2(xxy, m2)));
    const float wz = fz - (xz - magic);
    const float2 tl = upk2(ffma2(pk2(lo4.z, lo4.w), pk2(w.x, w.x), pk2(lo4.x, lo4.y)));
    const float2 th = upk2(ffma2(pk2(hi4.z, hi4.w), pk2(w.x, w.x), pk2(hi4.x, hi4.y)));
    const float s0 = fmaf(wz, tl.y, tl.x), s1 = fmaf(wz, th.y, th.x);
    return lerpf(s0, s1, w.y);
  };
  float acc = 0.f;
  float kf = 0.5f;
  const int nfull = rs.n - 1;
  if (UNR == 3) {  // the default launch: 415.95 vs 417.31 ms at unroll 2 (1: 422.6, 4: 437.6, spills)
#pragma unroll 3
    for (int k = 0; k < nfull; ++k, kf += 1.f) acc += sample(kf);
  } else {
#pragma unroll 2
    for (int k = 0; k < nfull; ++k, kf += 1.f) acc += sample(kf);
  }
  acc = fmaf(rs.last, sample((float)nfull + 0.5f * rs.last), acc);  // exact last segment
  store(acc * (float)step);
}

template <int VG, int CPS, bool FIXS, int COLS = kFpCols, int PROBE = 0, int ZP = 0, int UNR = 2>
__global__ void __launch_bounds__(COLS * kFpRows * VG, CPS)
    cone_fp_kernel(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy, double sz,
                   const ConeRayView *__restrict__ views, int rows, int cols, int n_views, double step,
                   float *__restrict__ out, unsigned zpitch, unsigned ystride) {
  fp_rays<VG, FIXS, false, COLS, PROBE, ZP, true, UNR>(q, nx, ny, nz, sx, sy, sz, views, rows, cols, n_views, step, out, zpitch, ystride,
                                 nullptr);
}

// The same march storing into row-band destinations (tk_forward_cone_3d_bands).
template <bool FIXS>
__global__ void __launch_bounds__(kFpColsDefault * kFpRows * 8, 4)
    cone_fp_bands_kernel(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy, double sz,
                         const ConeRayView *__restrict__ views, int rows, int cols, int n_views, double step,
                         unsigned zpitch, unsigned ystride, const __grid_constant__ FpDests dests) {
  fp_rays<8, FIXS, true, kFpColsDefault, 0, 0, true, 3>(q, nx, ny, nz, sx, sy, sz, views, rows, cols, n_views, step,
                                                        nullptr, zpitch, ystride, &dests);
}

// Sub-block = 16 columns x 8 direct rows (lower detector half) plus their 8 mirror rows.
template <int VG, int CPS, bool FIXS, int COLS = kFpCols>
__global__ void __launch_bounds__(COLS * kFpRows * VG, CPS)
    cone_fp_mirror_kernel(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy, double sz,
                          const ConeRayView *__restrict__ views, int rows, int cols, int n_views, double step,
                          float *__restrict__ out, unsigned zpitch, unsigned ystride) {
  constexpr int SUB = COLS * kFpRows;
  const int half = (rows + 1) >> 1;  // direct rows [0, half); an odd detector's middle row is its own mirror
  const int ncb = (cols + COLS - 1) / COLS;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int nvg = (n_views + VG - 1) / VG;
  const int v0 = (int)(bt % nvg) * VG, rb = (int)(bt / nvg);
  const int sub = threadIdx.x / SUB, t = threadIdx.x % SUB;
  const int v = v0 + sub, c = cb * COLS + (t >> 3), r = rb * kFpRows + (t & 7);
  if (c >= cols || r >= half || v >= n_views) return;
  const int rm = rows - 1 - r;
  float *dst = out + ((long long)v * rows + r) * cols + c;
  float *dstm = out + ((long long)v * rows + rm) * cols + c;
  RaySetup rs;
  if (!cone_ray_setup(views[v], r, c, nx, ny, nz, sx, sy, sz, step, rs)) {
    *dst = 0.f;
    *dstm = 0.f;
    return;
  }
  const float ex = rs.ex + (kFpMargin - 1), ey = rs.ey + (kFpMargin - 1), ez = rs.ez + (kFpMargin - 1);
  const float magic = 8388608.f;
  const unsigned sys = FIXS ? kMirS : ystride;
  const unsigned long long e2 = pk2(ex, ey), g2 = pk2(rs.gx, rs.gy), m2 = pk2(magic, magic);
  const float gz = rs.gz;
  unsigned cell = 0xffffffffu;
  Pair4 lo{0ull, 0ull, 0ull, 0ull}, hi = lo;
  auto sample = [&](float kk) -> unsigned long long {
    const unsigned long long fxy = ffma2(pk2(kk, kk), g2, e2);
    const float fz = fmaf(kk, gz, ez);
    const unsigned long long xxy = fadd2_rm(fxy, m2);
    const float xz = __fadd_rd(fz, magic);
    const float2 xb = upk2(xxy);
    const unsigned id = __float_as_uint(xb.y) * sys + (__float_as_uint(xb.x) * zpitch + __float_as_uint(xz));
    if (id != cell) {
      cell = id;
      ldg_pair4<FIXS>(elem_ptr(reinterpret_cast<const Pair4 *>(q), id), sys, lo, hi);
    }
    const float2 w = upk2(fsub2(fxy, fsub2(xxy, m2)));
    const float wz = fz - (xz - magic);
    const unsigned long long wx2 = pk2(w.x, w.x), wz2 = pk2(wz, wz);
    // (x, z) bilinear polynomial of rows y and y + 1 for both rays: A + wx B + wz (C + wx D)
    const unsigned long long sl = ffma2(ffma2(lo.d, wx2, lo.c), wz2, ffma2(lo.b, wx2, lo.a));
    const unsigned long long sh = ffma2(ffma2(hi.d, wx2, hi.c), wz2, ffma2(hi.b, wx2, hi.a));
    return ffma2(fsub2(sh, sl), pk2(w.y, w.y), sl);  // lerp in y
  };
  unsigned long long acc = 0ull;  // (direct, mirror)
  float kf = 0.5f;
  const int nfull = rs.n - 1;
#pragma unroll 2
  for (int k = 0; k < nfull; ++k, kf += 1.f) acc = fadd2(acc, sample(kf));
  acc = ffma2(pk2(rs.last, rs.last), sample((float)nfull + 0.5f * rs.last), acc);  // exact last segment
  const float2 a = upk2(acc);
  const float fs = (float)step;
  *dst = a.x * fs;
  if (rm != r) *dstm = a.y * fs;
}


// ---------------------------------------------------------------------------
// Warp-cooperative march (TK_FP_ALGO=warp): the north star's formulation, kept
// as the measured comparison.  A warp walks ONE ray at a time: lane l takes the
// samples base + l of every 32-sample stride (same sample positions, cells and
// arithmetic as cone_fp_kernel) and the 32 partial sums are combined with a
// __shfl_xor_sync tree.  Each lane's consecutive samples are 32 apart, so no
// lane reuses a cell, and the 32 lanes' cells lie along the ray (a new line per
// x / y crossing) instead of across the quarter-warp's z-contiguous cells:
// every sample loads, ~16 lines per warp load.  CTA = the 16 x 8 detector tile
// of one view; lane i of warp w sets up ray i of the warp's 4-column x 8-row
// sub-tile (float64), then broadcasts it to the warp.
// ---------------------------------------------------------------------------
template <bool FIXS>
__global__ void __launch_bounds__(128)
    cone_fp_warp_kernel(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy, double sz,
                        const ConeRayView *__restrict__ views, int rows, int cols, int n_views, double step,
                        float *__restrict__ out, unsigned zpitch, unsigned ystride) {
  const int ncb = (cols + kFpCols - 1) / kFpCols;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int v = (int)(bt % n_views), rb = (int)(bt / n_views);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = cb * kFpCols + warp * 4 + (lane >> 3), r = rb * kFpRows + (lane & 7);
  const bool valid = c < cols && r < rows;
  RaySetup rs;
  const bool live = valid && cone_ray_setup(views[v], r, c, nx, ny, nz, sx, sy, sz, step, rs);
  const float magic = 8388608.f;
  const unsigned sys = FIXS ? kFpFixS : ystride;
  const unsigned long long m2 = pk2(magic, magic);
  float mine = 0.f;
  for (int i = 0; i < 32; ++i) {
    const int n = __shfl_sync(0xffffffffu, live ? rs.n : 0, i);
    if (n == 0) continue;  // warp-uniform
    const float ex = __shfl_sync(0xffffffffu, rs.ex, i) + (kFpMargin - 1);
    const float ey = __shfl_sync(0xffffffffu, rs.ey, i) + (kFpMargin - 1);
    const float ez = __shfl_sync(0xffffffffu, rs.ez, i) + (kFpMargin - 1);
    const float gx = __shfl_sync(0xffffffffu, rs.gx, i), gy = __shfl_sync(0xffffffffu, rs.gy, i);
    const float gz = __shfl_sync(0xffffffffu, rs.gz, i), last = __shfl_sync(0xffffffffu, rs.last, i);
    const unsigned long long e2 = pk2(ex, ey), g2 = pk2(gx, gy);
    float acc = 0.f;
    for (int k = lane; k < n; k += 32) {
      const float kk = k < n - 1 ? (float)k + 0.5f : (float)(n - 1) + 0.5f * last;
      const unsigned long long fxy = ffma2(pk2(kk, kk), g2, e2);
      const float fz = fmaf(kk, gz, ez);
      const unsigned long long xxy = fadd2_rm(fxy, m2);
      const float xz = __fadd_rd(fz, magic);
      const float2 xb = upk2(xxy);
      const unsigned id = __float_as_uint(xb.y) * sys + (__float_as_uint(xb.x) * zpitch + __float_as_uint(xz));
      const float4 *p = elem_ptr(q, id);
      const float4 lo4 = __ldg(p), hi4 = __ldg(p + sys);
      const float2 w = upk2(fsub2(fxy, fsub2(xxy, m2)));
      const float wz = fz - (xz - magic);
      const float2 tl = upk2(ffma2(pk2(lo4.z, lo4.w), pk2(w.x, w.x), pk2(lo4.x, lo4.y)));
      const float2 th = upk2(ffma2(pk2(hi4.z, hi4.w), pk2(w.x, w.x), pk2(hi4.x, hi4.y)));
      const float sv = lerpf(fmaf(wz, tl.y, tl.x), fmaf(wz, th.y, th.x), w.y);
      acc = k < n - 1 ? acc + sv : fmaf(last, sv, acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == i) mine = acc * (float)step;
  }
  if (valid) out[((long long)v * rows + r) * cols + c] = live ? mine : 0.f;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Every view z-mirror symmetric: source in z = 0 and M^-1 (c, R-1-r, 1) equal to
// the reflection of M^-1 (c, r, 1), i.e. with columns m0, m1, m2 of M^-1:
// m0_z = 0, m1_x = m1_y = 0, m2_z = -(R-1)/2 m1_z (relative tolerance 1e-9).
bool views_z_mirror(const double *sources, const double *minv, int n_views, int rows) {
  const double tol = 1e-9, h = (rows - 1) / 2.0;
  for (int i = 0; i < n_views; ++i) {
    const double *s = sources + 3 * i, *m = minv + 9 * i;
    const double sn = std::sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
    if (!(std::fabs(s[2]) <= tol * sn)) return false;
    const double n0 = std::sqrt(m[0] * m[0] + m[3] * m[3] + m[6] * m[6]);
    const double n1 = std::sqrt(m[1] * m[1] + m[4] * m[4] + m[7] * m[7]);
    const double n2 = std::sqrt(m[2] * m[2] + m[5] * m[5] + m[8] * m[8]);
    if (!(std::fabs(m[6]) <= tol * n0)) return false;
    if (!(std::fabs(m[1]) <= tol * n1 && std::fabs(m[4]) <= tol * n1)) return false;
    if (!(std::fabs(m[8] + h * m[7]) <= tol * (n2 + h * n1))) return false;
  }
  return true;
}


// Cell layout of one volume copy.  Fixed y stride (the far row at an immediate
// load offset) when it fits and its padding is affordable (make_layout);
// otherwise a runtime stride with bias-free pitches: zp (1 + xp) == -1 (mod 256).
struct FpLayout {
  bool mirror = false, fixs = false;
  unsigned zpitch = 0, xpitch = 0, ystride = 0;
  int zcells = 0;  // padded z cells stored per (y, x)
  size_t cell_bytes = 16;
};

static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

static bool make_layout(int nz, int ny, int nx, bool mirror, FpLayout &L, bool force_runtime_stride = false) {
  constexpr int m2 = 2 * kFpMargin;
  L = FpLayout();
  L.mirror = mirror;
  L.cell_bytes = mirror ? 32 : 16;
  // direct rays of the mirror kernel reach padded z <= K / 2 (+ rounding); taps floor, floor + 1
  L.zcells = mirror ? (nz - 1 + m2) / 2 + 2 : nz + m2;
  const unsigned zc = (unsigned)L.zcells, xc = (unsigned)(nx + m2);
  const unsigned long long rows = (unsigned long long)(ny + m2);
  const unsigned long long compact = rows * xc * zc;
  const unsigned fixs = mirror ? kMirS : kFpFixS, zres = mirror ? 5u : 255u;
  const unsigned zpf = zc + (zres + 256u - zc % 256u) % 256u;
  const bool nofix = force_runtime_stride || env_int("TK_FP_NOFIX", 0) != 0;  // 1: always the runtime stride (tests)
  // the fixed stride pads each row to kFpFixS cells: allowed while that costs at most 2x the
  // compact layout or at most 3 GB (cfg3 256^3: 2.2 GB, 9 % faster); an allocation failure
  // falls back to the compact layout (plan_cells)
  const unsigned long long fixed_bytes = rows * fixs * L.cell_bytes;
  const bool affordable = rows * fixs <= 2 * compact || fixed_bytes <= (3ull << 30);
  if (!nofix && (unsigned long long)xc * zpf <= fixs && affordable && rows * fixs < (1ull << 32)) {
    L.fixs = true;
    L.zpitch = zpf;
    L.xpitch = xc;
    L.ystride = fixs;
    return true;
  }
  long long best = -1;
  for (unsigned zp = zc | 1u; zp < zc + 128; zp += 2) {  // zp odd: 1 + xp solvable mod 256
    unsigned xp = xc;
    while ((zp * (1u + xp)) % 256u != 255u) ++xp;
    const long long cells = (long long)zp * xp;
    if (best < 0 || cells < best) {
      best = cells;
      L.zpitch = zp;
      L.xpitch = xp;
    }
  }
  L.ystride = L.xpitch * L.zpitch;
  return rows * L.ystride < (1ull << 32);
}

bool fp_mirror_fits(int nz, int ny, int nx) {
  FpLayout L;
  return make_layout(nz, ny, nx, true, L);
}

bool fp_use_mirror(const double *sources, const double *minv, int n_views, int rows, int nz, int ny, int nx) {
  if (!env_int("TK_FP_MIRROR", 0)) return false;  // 1: z-mirror-pair kernel for symmetric scans
  return fp_mirror_fits(nz, ny, nx) && views_z_mirror(sources, minv, n_views, rows);
}

// A forward-projection plan: the cell layout(s) of one volume, built on first
// use and reused by any number of view blocks (the e2e path projects view
// chunks so their D2H copies overlap the next chunk's kernel).
struct FpPlan {
  const float *vol = nullptr;
  int nz = 0, ny = 0, nx = 0;
  double sz = 0, sy = 0, sx = 0;
  FpLayout lay[2];             // [general, mirror]
  void *cells[2] = {nullptr, nullptr};
};

static int plan_cells(FpPlan &pl, bool mirror, cudaStream_t st) {
  const int k = mirror ? 1 : 0;
  if (pl.cells[k]) return TK_OK;
  FpLayout &L = pl.lay[k];
  if (!make_layout(pl.nz, pl.ny, pl.nx, mirror, L))
    return fail_arg("tk_forward_cone_3d: volume too large for 32-bit cell indices");
  size_t bytes = L.cell_bytes * (size_t)(pl.ny + 2 * kFpMargin) * L.ystride;
  cudaError_t e = cudaMallocAsync(&pl.cells[k], bytes, st);
  if (e == cudaErrorMemoryAllocation && L.fixs) {  // the fixed stride pads: retry with the compact layout
    (void)cudaGetLastError();
    make_layout(pl.nz, pl.ny, pl.nx, mirror, L, true);
    bytes = L.cell_bytes * (size_t)(pl.ny + 2 * kFpMargin) * L.ystride;
    e = cudaMallocAsync(&pl.cells[k], bytes, st);
  }
  if (e != cudaSuccess) {
    pl.cells[k] = nullptr;
    return check_cuda(e, "cudaMallocAsync (forward-projection cells)");
  }
  if (mirror) {
    dim3 g(ceil_div(L.zcells, 32), ceil_div(pl.nx + 2 * kFpMargin, 32), pl.ny + 2 * kFpMargin);
    fp_mirror_cells_kernel<<<g, 256, 0, st>>>(pl.vol, pl.nz, pl.ny, pl.nx, static_cast<float4 *>(pl.cells[k]),
                                              L.zpitch, L.ystride, L.zcells);
    TK_LAUNCHED("fp_mirror_cells_kernel");
  } else {
    dim3 g(ceil_div(pl.nz + 2 * kFpMargin, 32), ceil_div(pl.nx + 2 * kFpMargin, 32), pl.ny + 2 * kFpMargin);
    fp_cells_kernel<<<g, 256, 0, st>>>(pl.vol, pl.nz, pl.ny, pl.nx, static_cast<float4 *>(pl.cells[k]), L.zpitch,
                                       L.ystride);
    TK_LAUNCHED("fp_cells_kernel");
  }
  return TK_OK;
}

static void plan_free(FpPlan &pl, cudaStream_t st) {
  for (void *&p : pl.cells)
    if (p) {
      cudaFreeAsync(p, st);
      p = nullptr;
    }
}

using FpKern = void (*)(const float4 *, int, int, int, double, double, double, const ConeRayView *, int, int, int,
                        double, float *, unsigned, unsigned);

// Launch configurations (views per CTA x CTAs per SM): general 8x4 with 8-column view
// tiles (default: 32 registers, 64 warps/SM; 420.6 vs 423.7 ms for 16-column tiles at
// 8x2, profiles/r02/fp_ab_r02ap.log), 8x2 or 4x4 with 16-column tiles; mirror 4x3
// (default, 40 registers), 8x2, 8x1.
static FpKern pick_kernel(bool mirror, bool fixs, unsigned zpitch, int &vg, int &tcols) {
  tcols = kFpCols;
  const char *ce = getenv("TK_FP_CFG");
  const bool c8x1 = ce && !strcmp(ce, "8x1"), c8x2 = ce && !strcmp(ce, "8x2"), c4x4 = ce && !strcmp(ce, "4x4"),
             c4x3 = ce && !strcmp(ce, "4x3"), c6x2 = ce && !strcmp(ce, "6x2");
  if (mirror) {
    if (c6x2) return vg = 6, fixs ? cone_fp_mirror_kernel<6, 2, true> : cone_fp_mirror_kernel<6, 2, false>;
    if (c8x2) return vg = 8, fixs ? cone_fp_mirror_kernel<8, 2, true> : cone_fp_mirror_kernel<8, 2, false>;
    if (c8x1) return vg = 8, fixs ? cone_fp_mirror_kernel<8, 1, true> : cone_fp_mirror_kernel<8, 1, false>;
    return vg = 4, fixs ? cone_fp_mirror_kernel<4, 3, true> : cone_fp_mirror_kernel<4, 3, false>;
  }
  const int probe = env_int("TK_FP_PROBE", 0);  // roofline decomposition probes (not projectors)
  if (probe == 1)
    return vg = 8, tcols = kFpColsDefault,
           fixs ? cone_fp_kernel<8, 4, true, kFpColsDefault, 1> : cone_fp_kernel<8, 4, false, kFpColsDefault, 1>;
  if (probe == 2)
    return vg = 8, tcols = kFpColsDefault,
           fixs ? cone_fp_kernel<8, 4, true, kFpColsDefault, 2> : cone_fp_kernel<8, 4, false, kFpColsDefault, 2>;
  if (probe == 7 && fixs && zpitch == 767) {
    vg = 8, tcols = kFpColsDefault;
    return cone_fp_kernel<8, 4, true, kFpColsDefault, 7, 767, 3>;
  }
  if (c8x2) return vg = 8, fixs ? cone_fp_kernel<8, 2, true> : cone_fp_kernel<8, 2, false>;
  if (c4x4 || c4x3) return vg = 4, fixs ? cone_fp_kernel<4, 4, true> : cone_fp_kernel<4, 4, false>;
  if (fixs && env_int("TK_FP_ZP", 1)) {  // the fixed layout's z pitch as an immediate
    constexpr int C = kFpColsDefault;
    vg = 8, tcols = C;
    if (zpitch == 255) return cone_fp_kernel<8, 4, true, C, 0, 255, 3>;
    if (zpitch == 511) return cone_fp_kernel<8, 4, true, C, 0, 511, 3>;
    if (zpitch == 767 && env_int("TK_FP_UNR", 3) == 2) return cone_fp_kernel<8, 4, true, C, 0, 767, 2>;
    if (zpitch == 767) return cone_fp_kernel<8, 4, true, C, 0, 767, 3>;
    if (zpitch == 1023) return cone_fp_kernel<8, 4, true, C, 0, 1023, 3>;
  }
  return vg = 8, tcols = kFpColsDefault,
         fixs ? cone_fp_kernel<8, 4, true, kFpColsDefault, 0, 0, 3> : cone_fp_kernel<8, 4, false, kFpColsDefault, 0, 0, 3>;
}

static int plan_project(FpPlan &pl, const double *sources, const double *minv, int n_views, int rows, int cols,
                        double step, float *out, cudaStream_t st) {
  const bool mirror = fp_use_mirror(sources, minv, n_views, rows, pl.nz, pl.ny, pl.nx);
  int rc = plan_cells(pl, mirror, st);
  if (rc != TK_OK) return rc;
  const FpLayout &L = pl.lay[mirror ? 1 : 0];
  std::vector<ConeRayView> hv(n_views);
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].minv[j] = minv[9 * i + j];
  }
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeRayView) * n_views, st));
  const char *algo = getenv("TK_FP_ALGO");
  if (!mirror && algo && !strcmp(algo, "warp")) {  // warp-cooperative comparison kernel
    const long long nbw = (long long)ceil_div(cols, kFpCols) * ceil_div(rows, kFpRows) * n_views;
    if (nbw >= (1LL << 31)) return fail_arg("tk_forward_cone_3d: problem too large for one launch");
    auto kw = L.fixs ? cone_fp_warp_kernel<true> : cone_fp_warp_kernel<false>;
    kw<<<(unsigned)nbw, 128, 0, st>>>(static_cast<const float4 *>(pl.cells[0]), pl.nx, pl.ny, pl.nz, pl.sx, pl.sy,
                                      pl.sz, dviews.as<ConeRayView>(), rows, cols, n_views, step, out, L.zpitch,
                                      L.ystride);
    TK_LAUNCHED("cone_fp_warp_kernel");
    return TK_OK;
  }
  int vg = 1, tcols = kFpCols;
  FpKern kern = pick_kernel(mirror, L.fixs, L.zpitch, vg, tcols);
  const int brows = mirror ? (rows + 1) / 2 : rows;
  const long long nb = (long long)ceil_div(cols, tcols) * ceil_div(brows, kFpRows) * ceil_div(n_views, vg);
  if (nb >= (1LL << 31)) return fail_arg("tk_forward_cone_3d: problem too large for one launch");
  kern<<<(unsigned)nb, tcols * kFpRows * vg, 0, st>>>(static_cast<const float4 *>(pl.cells[mirror ? 1 : 0]), pl.nx, pl.ny, pl.nz,
                                          pl.sx, pl.sy, pl.sz, dviews.as<ConeRayView>(), rows, cols, n_views, step, out,
                                          L.zpitch, L.ystride);
  TK_LAUNCHED(mirror ? "cone_fp_mirror_kernel" : "cone_fp_kernel");
  return TK_OK;
}

// Fused view-sharded projection + row-band exchange: the general kernel with BANDS stores.
static int plan_project_bands(FpPlan &pl, const double *sources, const double *minv, int n_views, int rows, int cols,
                              double step, const FpDests &d, cudaStream_t st) {
  int rc = plan_cells(pl, false, st);
  if (rc != TK_OK) return rc;
  const FpLayout &L = pl.lay[0];
  std::vector<ConeRayView> hv(n_views);
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].minv[j] = minv[9 * i + j];
  }
  Scratch dviews;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeRayView) * n_views, st));
  const long long nb = (long long)ceil_div(cols, kFpColsDefault) * ceil_div(rows, kFpRows) * ceil_div(n_views, 8);
  if (nb >= (1LL << 31)) return fail_arg("tk_forward_cone_3d_bands: problem too large for one launch");
  auto kern = L.fixs ? cone_fp_bands_kernel<true> : cone_fp_bands_kernel<false>;
  kern<<<(unsigned)nb, kFpColsDefault * kFpRows * 8, 0, st>>>(static_cast<const float4 *>(pl.cells[0]), pl.nx, pl.ny, pl.nz, pl.sx, pl.sy, pl.sz,
                                      dviews.as<ConeRayView>(), rows, cols, n_views, step, L.zpitch, L.ystride, d);
  TK_LAUNCHED("cone_fp_bands_kernel");
  return TK_OK;
}

static int launch_fp_default(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                      const double *sources, const double *minv, int n_views, int rows, int cols, double step,
                      float *out, cudaStream_t st) {
  FpPlan pl;
  pl.vol = vol;
  pl.nz = nz, pl.ny = ny, pl.nx = nx;
  pl.sz = sz, pl.sy = sy, pl.sx = sx;
  const int rc = plan_project(pl, sources, minv, n_views, rows, cols, step, out, st);
  plan_free(pl, st);
  return rc;
}

}  // namespace tk

using namespace tk;

extern "C" {

// TK_FP_ALGO = default (tk_fp.cu) | warp (warp-cooperative comparison, tk_fp.cu) | tex | hwtex
// (texture-unit comparison, tk_fp_tex.cu)
int tk_forward_cone_3d(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                       const double *sources, const double *minv, int n_views, int rows, int cols, double step,
                       float *out, void *stream) {
  clear_error();
  if (!vol || !out || !sources || !minv) return fail_arg("tk_forward_cone_3d: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_forward_cone_3d: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0 && step > 0)) return fail_arg("tk_forward_cone_3d: spacing/step must be > 0");
  const char *algo = getenv("TK_FP_ALGO");
  if (algo && (!strcmp(algo, "tex") || !strcmp(algo, "hwtex")))
    return launch_fp_tex(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step,
                         !strcmp(algo, "hwtex"), out, as_stream(stream));
  return launch_fp_default(vol, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, out,
                           as_stream(stream));
}

int tk_fp_plan_create(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx, void **plan,
                      void *stream) {
  clear_error();
  (void)stream;
  if (!vol || !plan) return fail_arg("tk_fp_plan_create: null pointer");
  if (nz < 1 || ny < 1 || nx < 1) return fail_arg("tk_fp_plan_create: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0)) return fail_arg("tk_fp_plan_create: spacing must be > 0");
  FpLayout L;
  if (!make_layout(nz, ny, nx, false, L)) return fail_arg("tk_fp_plan_create: volume too large for 32-bit cell indices");
  FpPlan *pl = new FpPlan();
  pl->vol = vol;
  pl->nz = nz, pl->ny = ny, pl->nx = nx;
  pl->sz = sz, pl->sy = sy, pl->sx = sx;
  *plan = pl;
  return TK_OK;
}

int tk_fp_plan_project(void *plan, const double *sources, const double *minv, int n_views, int rows, int cols,
                       double step, float *out, void *stream) {
  clear_error();
  if (!plan || !sources || !minv || !out) return fail_arg("tk_fp_plan_project: null pointer");
  if (n_views < 1 || rows < 1 || cols < 1 || !(step > 0)) return fail_arg("tk_fp_plan_project: bad extent / step");
  return plan_project(*reinterpret_cast<FpPlan *>(plan), sources, minv, n_views, rows, cols, step, out,
                      as_stream(stream));
}

int tk_fp_plan_destroy(void *plan, void *stream) {
  clear_error();
  if (!plan) return TK_OK;
  FpPlan *pl = reinterpret_cast<FpPlan *>(plan);
  plan_free(*pl, as_stream(stream));
  delete pl;
  return TK_OK;
}

int tk_forward_cone_3d_bands(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                             const double *sources, const double *minv, int n_views, int rows, int cols, double step,
                             int view_offset, int n_dest, float *const *dest, const int *r0, const int *r1,
                             int band_pitch_rows, void *stream) {
  clear_error();
  if (!vol || !sources || !minv || !dest || !r0 || !r1) return fail_arg("tk_forward_cone_3d_bands: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1 || view_offset < 0)
    return fail_arg("tk_forward_cone_3d_bands: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0 && step > 0)) return fail_arg("tk_forward_cone_3d_bands: spacing/step must be > 0");
  if (n_dest < 1 || n_dest > kFpMaxDest) return fail_arg("tk_forward_cone_3d_bands: 1 to 16 destinations");
  FpDests d{};
  d.n = n_dest;
  d.view_offset = view_offset;
  d.view_stride = (long long)band_pitch_rows * cols;
  for (int h = 0; h < n_dest; ++h) {
    if (!dest[h]) return fail_arg("tk_forward_cone_3d_bands: null destination");
    if (r0[h] < 0 || r1[h] > rows || r1[h] - r0[h] > band_pitch_rows)
      return fail_arg("tk_forward_cone_3d_bands: band outside the detector or wider than the pitch");
    d.ptr[h] = dest[h];
    d.r0[h] = r0[h];
    d.r1[h] = r1[h];
  }
  FpPlan pl;
  pl.vol = vol;
  pl.nz = nz, pl.ny = ny, pl.nx = nx;
  pl.sz = sz, pl.sy = sy, pl.sx = sx;
  const int rc = plan_project_bands(pl, sources, minv, n_views, rows, cols, step, d, as_stream(stream));
  plan_free(pl, as_stream(stream));
  return rc;
}

int tk_forward_cone_3d_path(const double *sources, const double *minv, int n_views, int rows, int cols, int nz,
                            int ny, int nx) {
  (void)cols;
  if (!sources || !minv || n_views < 1 || rows < 1 || nz < 1 || ny < 1 || nx < 1) return 0;
  return fp_use_mirror(sources, minv, n_views, rows, nz, ny, nx) ? 1 : 0;
}

}  // extern "C"
