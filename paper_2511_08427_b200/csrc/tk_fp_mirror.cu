// tk_fp_mirror.cu -- cone-beam forward projector for z-mirror-symmetric scans
// (circular orbits: source in the z = 0 plane, detector v axis along z,
// principal row at (R-1)/2).  Reference semantics: _kernels.py:254-278
// (ray set-up) and _march_3d, _kernels.py:117-157 (midpoint rule, trilinear
// taps, exact last segment).
//
// For such a view the ray through detector pixel (R-1-r, c) is the mirror image
// z -> -z of the ray through (r, c): same source, same x/y track, same clip
// interval (the box is symmetric in z), hence the same sample count and the
// same sample parameters t_k.  In the kernel's padded index space z maps to
// K - z with K = nz - 1 + 2m, so the mirrored ray's sample k sits at
// (fx, fy, K - fz): its cell index along z is K - 1 - floor(fz) and its z
// weight 1 - wz.  Storing next to every cell of V the cell of the reflected
// volume Vm[z] = V[K - z] makes the mirrored sample an interpolation of Vm
// with EXACTLY the direct ray's cell index and weights.  One thread therefore
// marches both rays: one position / floor / index / weight computation and one
// pair of 32-byte loads per cell change serve two samples, and the bilinear
// (x, z) polynomials and the y lerp of the two rays run as FFMA2 / FADD2 pairs.
// The direct rays (rows r < R/2, v < 0) only reach z <= 0, so the cells cover
// half the z extent: the pair layout costs no more memory than one copy.
//
// Cell (y, x, z), 32 B: float pairs (A, A'), (C, C'), (B, B'), (D, D') with
// A = V00, B = V01 - V00, C = V10 - V00, D = (V11 - V10) - (V01 - V00)
// (V_zx of row y; primed: the same for Vm), the coefficient form of the
// z-fastest kernel (tk_cone.cu, coef_volume_z_kernel).  The y stride is the
// compile-time constant kMirS so the far row (y + 1) is an immediate offset
// of the near row's address, and the z pitch is == 5 (mod 256) so that
// 1 + zpitch + kMirS == 0 (mod 256): the cell index formed from the FADD.RM
// float bits (0x4B000000 + floor) carries no bias modulo 2^32.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tk_cone_fp.cuh"

namespace tk {

constexpr unsigned kMirS = 262138u;  // y stride in 32-byte cells: == 250 (mod 256), * 32 B < 2^23
constexpr unsigned kMirZP = 5u;      // z pitch residue (mod 256)
constexpr int kMirRB = 8;            // detector rows per quarter-warp (one column)

// Cells of rows y (padded) for z in [0, zcells) of the pair layout.
__global__ void __launch_bounds__(256) coef_volume_mirror_kernel(const float *__restrict__ vol, int nz, int ny,
                                                                 int nx, float4 *__restrict__ cq, int zpitch,
                                                                 int zcells) {
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
    const int z = z0 + tz, x = x0 + tx;  // cell (z, y, x) of the padded grid
    if (z >= zcells || x + m >= px) continue;
    float c[2][4];
    for (int s = 0; s < 2; ++s) {
      const float v00 = tile[s][tx][tz], v01 = tile[s][tx + 1][tz], v10 = tile[s][tx][tz + 1],
                  v11 = tile[s][tx + 1][tz + 1];
      c[s][0] = v00;                      // A
      c[s][1] = v10 - v00;                // C
      c[s][2] = v01 - v00;                // B
      c[s][3] = (v11 - v10) - (v01 - v00);  // D
    }
    float4 *dst = cq + 2 * ((long long)(y + m) * kMirS + (long long)(x + m) * zpitch + z);
    dst[0] = make_float4(c[0][0], c[1][0], c[0][1], c[1][1]);  // (A, A'), (C, C')
    dst[1] = make_float4(c[0][2], c[1][2], c[0][3], c[1][3]);  // (B, B'), (D, D')
  }
}

struct __align__(32) Pair4 {
  unsigned long long a, c, b, d;  // (A, A'), (C, C'), (B, B'), (D, D')
};

__device__ __forceinline__ void ldg_pair4(const Pair4 *p, Pair4 &lo, Pair4 &hi) {
  // near row (y) and far row (y + 1, an immediate offset of kMirS cells)
  asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(lo.a), "=l"(lo.c), "=l"(lo.b), "=l"(lo.d)
               : "l"(p));
  asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4+8388416];"
               : "=l"(hi.a), "=l"(hi.c), "=l"(hi.b), "=l"(hi.d)
               : "l"(p));
}

// CTA = VG sub-blocks of 128 threads on VG consecutive views; a sub-block =
// 16 columns x 8 direct rows (each quarter-warp 8 consecutive rows of one
// column) plus their 8 mirror rows.  Order: column blocks fastest, then view
// groups, then 8-row bands of the lower detector half.
template <int VG, int MINB>
__global__ void __launch_bounds__(128 * VG, MINB)
    cone_fp_mirror_kernel(const float4 *__restrict__ q, int nx, int ny, int nz, double sx, double sy, double sz,
                          const ConeRayView *__restrict__ views, int rows, int cols, int n_views, double step,
                          float *__restrict__ out, unsigned zpitch) {
  constexpr int kCols = 128 / kMirRB;
  const int half = (rows + 1) >> 1;  // direct rows [0, half); the middle row of an odd detector is its own mirror
  const int ncb = (cols + kCols - 1) / kCols;
  const unsigned b = blockIdx.x;
  const int cb = (int)(b % ncb);
  const unsigned bt = b / ncb;
  const int nvg = (n_views + VG - 1) / VG;
  const int v = (int)(bt % nvg) * VG + (int)(threadIdx.x >> 7);
  const int rb = (int)(bt / nvg);
  const int t = threadIdx.x & 127;
  const int c = cb * kCols + (t >> 3);
  const int r = rb * kMirRB + (t & 7);
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
  const float magic = 8388608.f;  // coordinates >= 0: floor(f) = bits(f + 2^23) - 0x4B000000
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
    const unsigned id = __float_as_uint(xb.y) * kMirS + (__float_as_uint(xb.x) * zpitch + __float_as_uint(xz));
    if (id != cell) {
      cell = id;
      ldg_pair4(elem_ptr(reinterpret_cast<const Pair4 *>(q), id), lo, hi);
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
  const float2 res = upk2(acc);
  const float fs = (float)step;
  *dst = res.x * fs;
  if (rm != r) *dstm = res.y * fs;
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

struct MirrorLayout {
  unsigned zpitch = 0;
  int zcells = 0;
  bool ok = false;
};

static MirrorLayout mirror_layout(int nz, int nx) {
  MirrorLayout L;
  const int K = nz - 1 + 2 * kFpMargin;
  L.zcells = K / 2 + 2;  // direct rays reach fz <= K/2 (+ rounding); taps floor(fz), floor(fz) + 1
  L.zpitch = (unsigned)L.zcells + (kMirZP + 256u - (unsigned)L.zcells % 256u) % 256u;
  L.ok = (unsigned long long)(nx + 2 * kFpMargin) * L.zpitch <= kMirS;
  return L;
}

bool fp_mirror_fits(int nz, int ny, int nx) {
  return mirror_layout(nz, nx).ok && (unsigned long long)(ny + 2 * kFpMargin) * kMirS < (1ull << 32);
}

bool fp_use_mirror(const double *sources, const double *minv, int n_views, int rows, int nz, int ny, int nx) {
  const char *me = getenv("TK_FP_MIRROR");  // 0: never use the z-mirror-pair kernel
  const char *algo = getenv("TK_FP_ALGO");  // only the default algorithm has a mirror form
  if ((me && !atoi(me)) || (algo && strcmp(algo, "ldg4z"))) return false;
  return fp_mirror_fits(nz, ny, nx) && views_z_mirror(sources, minv, n_views, rows);
}

int launch_fp_mirror(const float *vol, int nz, int ny, int nx, double sz, double sy, double sx,
                     const double *sources, const double *minv, int n_views, int rows, int cols, double step,
                     float *out, cudaStream_t st) {
  const MirrorLayout L = mirror_layout(nz, nx);
  if (!L.ok) return fail_arg("tk_forward_cone_3d: volume too wide for the mirror-pair layout");
  std::vector<ConeRayView> hv(n_views);
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].minv[j] = minv[9 * i + j];
  }
  Scratch dviews, cells;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeRayView) * n_views, st));
  const size_t bytes = (size_t)(ny + 2 * kFpMargin) * kMirS * 32u;
  TK_TRY_CUDA(cells.alloc(bytes, st));
  dim3 tg(ceil_div(L.zcells, 32), ceil_div(nx + 2 * kFpMargin, 32), ny + 2 * kFpMargin);
  coef_volume_mirror_kernel<<<tg, 256, 0, st>>>(vol, nz, ny, nx, cells.as<float4>(), (int)L.zpitch, L.zcells);
  TK_LAUNCHED("coef_volume_mirror_kernel");
  // TK_FPM_CFG = views per CTA x CTAs per SM: 4x3 (default, 40 registers, 48 warps/SM),
  // 8x1 (64 registers, 32 warps), 8x2 (32 registers, 64 warps)
  const char *ce = getenv("TK_FPM_CFG");
  int vg = 4;
  auto kern = cone_fp_mirror_kernel<4, 3>;
  if (ce && !strcmp(ce, "8x1")) vg = 8, kern = cone_fp_mirror_kernel<8, 1>;
  if (ce && !strcmp(ce, "8x2")) vg = 8, kern = cone_fp_mirror_kernel<8, 2>;
  const int half = (rows + 1) / 2;
  const long long nb = (long long)ceil_div(cols, 128 / kMirRB) * ceil_div(half, kMirRB) * ceil_div(n_views, vg);
  if (nb >= (1LL << 31)) return fail_arg("tk_forward_cone_3d: problem too large for one launch");
  kern<<<(unsigned)nb, 128 * vg, 0, st>>>(cells.as<float4>(), nx, ny, nz, sx, sy, sz, dviews.as<ConeRayView>(), rows,
                                         cols, n_views, step, out, L.zpitch);
  TK_LAUNCHED("cone_fp_mirror_kernel");
  return TK_OK;
}

}  // namespace tk

extern "C" int tk_forward_cone_3d_path(const double *sources, const double *minv, int n_views, int rows, int cols,
                                       int nz, int ny, int nx) {
  (void)cols;
  if (!sources || !minv || n_views < 1 || rows < 1 || nz < 1 || ny < 1 || nx < 1) return 0;
  return tk::fp_use_mirror(sources, minv, n_views, rows, nz, ny, nx) ? 1 : 0;
}
