// tk_fp_adjoint.cu -- the exact transpose A^T of the ray-driven cone forward
// projector (matched adjoint; reference autodiff.py:59-68 asks for the
// transposed operator, the reference itself pairs A with the voxel-driven B).
//
// The forward march transposed (same rays, set-up and sample positions as
// tk_fp.cu / _kernels.py:254-278, 117-157): each sample's 8 trilinear weights
// times y * seg are accumulated in registers while the ray stays in one cell
// and flushed as 16-byte vector reductions (REDG.E.ADD.F32x4, one per 4 taps)
// into z-fastest tap quads; tiled folds sum the 4 quads holding each voxel's
// tap back into the (z, y, x) volume.  fp32 atomics: summation order is not
// deterministic.  Deterministic mode: fixed-point quads with integer atomics
// (associative: bit-reproducible), the scale chosen from a magnitude pass (the
// same scatter of |y|) so no sum can overflow; two components per 64-bit word.
//
// Bound: the L2 vector-reduction pipeline (cfg5: 2.0e11 reduction sectors, atomic input
// 59 % busy, half the sectors miss L2).  Measured at cfg5 (profiles/r02): pair arithmetic
// (FFMA2 weights, 4 FFMA2 accumulations per sample) 1002 -> 984 ms; without the row
// carry-over 1300 ms; rays split into 2 / 3 / 4 / 6 launches by segment (smaller working set
// of the reduction targets) 1014 / 1036 / 1053 / 1082 ms -- not kept.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tk_cone_fp.cuh"

namespace tk {

constexpr int kFpzRows = 8;  // detector rows per quarter-warp (one column)


// z-fastest form of the quad scatter (the transpose of cone_fp_kernel, tk_fp.cu,
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
// 2^-e (scale = 2^e, exact) and added with 64-bit integer atomics.  Integer addition is
// associative, so the result does not depend on the order in which rays flush:
// bit-reproducible (torch.use_deterministic_algorithms).  Two components share one
// 64-bit word, a + 2^32 b: e is chosen so every component's total stays below 2^30 in
// magnitude, so the low 32 bits of the word, read as a signed int, are exactly sum(a)
// and (word - sum(a)) / 2^32 is exactly sum(b) -- two atomics per quad instead of four.
__device__ __forceinline__ unsigned long long fx_pack(float a, float b, float scale) {
  return (unsigned long long)((long long)__float2int_rn(a * scale) + ((long long)__float2int_rn(b * scale) << 32));
}
__device__ __forceinline__ void red_add_fx4(unsigned long long *p, const float4 &v, float scale) {
  atomicAdd(p, fx_pack(v.x, v.y, scale));
  atomicAdd(p + 1, fx_pack(v.z, v.w, scale));
}
__device__ __forceinline__ long long fx_unpack(unsigned long long w, int half) {
  const long long lo = (long long)(int)(unsigned)w;  // sign-extended low component
  return half ? ((long long)w - lo) >> 32 : lo;
}

// ABS: scatter |y| (fp32) -- the deterministic mode's magnitude pass (launch_fp_adjoint_det).
template <int MINB, bool DET = false, bool CARRY = true, bool ABS = false>
__global__ void __launch_bounds__(128, MINB)
    cone_fp_adjoint4z_kernel(const float *__restrict__ sino, void *__restrict__ qy_, void *__restrict__ qx_,
                             int nx, int ny, int nz, double sx, double sy, double sz,
                             const ConeRayView *__restrict__ views, int rows, int cols, int n_views, double step,
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
  const float y = ABS ? fabsf(__ldg(sino + ((long long)v * rows + r) * cols + c))
                      : __ldg(sino + ((long long)v * rows + r) * cols + c);
  if (y == 0.f) return;
  RaySetup rs;
  if (!cone_ray_setup(views[v], r, c, nx, ny, nz, sx, sy, sz, step, rs)) return;
  const bool xrow = fabsf(rs.gx) > fabsf(rs.gy);  // major horizontal axis (cells per step)
  void *qv = xrow ? qx_ : qy_;
  const float ea = (xrow ? rs.ey : rs.ex) + (kFpMargin - 1), eb = (xrow ? rs.ex : rs.ey) + (kFpMargin - 1);
  const float ez = rs.ez + (kFpMargin - 1);
  const float ga = xrow ? rs.gy : rs.gx, gb = xrow ? rs.gx : rs.gy, gz = rs.gz;
  const unsigned pz = (unsigned)(nz + 2 * kFpMargin);
  const unsigned sas = pz, sbs = (unsigned)((xrow ? ny : nx) + 2 * kFpMargin) * pz;  // a and b strides
  const unsigned bias = kFloorBits * (1u + sas + sbs);
  const float g = y * (float)step;
  // (a, b) position / floor / fraction as FFMA2 / FADD2 pairs; weights as pairs (1 - w, w);
  // the 8 accumulators as 4 pairs, each sample 4 FFMA2 (broadcast row-weight x (1 - wa, wa))
  const unsigned long long e2 = pk2(ea, eb), g2 = pk2(ga, gb), m2 = pk2(kFloorMagic, kFloorMagic);
  const unsigned long long one0 = pk2(1.f, 0.f), m1p1 = pk2(-1.f, 1.f);
  unsigned long long lo01 = 0ull, lo23 = 0ull, hi01 = 0ull, hi23 = 0ull;  // quads (row b, row b + 1)
  auto cell_of = [&](float kk) -> unsigned {
    const unsigned long long fab = ffma2(pk2(kk, kk), g2, e2);
    const float2 xab = upk2(fadd2_rm(fab, m2));
    const float xz = floor_magic(fmaf(kk, gz, ez));
    return __float_as_uint(xab.y) * sbs + (__float_as_uint(xab.x) * sas + __float_as_uint(xz));
  };
  auto flush = [&](unsigned cidx, unsigned long long q01, unsigned long long q23) {  // quad cidx += q
    const float2 a = upk2(q01), c = upk2(q23);
    const float4 v = make_float4(a.x, a.y, c.x, c.y);
    if (DET)
      red_add_fx4(static_cast<unsigned long long *>(qv) + 2ull * cidx, v, scale);
    else
      red_add_v4(static_cast<float4 *>(qv) + cidx, v);
  };
  unsigned cell = cell_of(0.5f);  // the first sample's cell: no flush before it
  auto sample = [&](float kk, float gs) {
    const unsigned long long fab = ffma2(pk2(kk, kk), g2, e2);
    const float fz = fmaf(kk, gz, ez);
    const unsigned long long xab = fadd2_rm(fab, m2);
    const float xz = floor_magic(fz);
    const float2 xb = upk2(xab);
    const unsigned id = __float_as_uint(xb.y) * sbs + (__float_as_uint(xb.x) * sas + __float_as_uint(xz));
    if (id != cell) {
      const unsigned c0 = cell - bias;
      if (CARRY && id == cell + sbs) {  // row b -> b + 1: the far row becomes the near row
        flush(c0, lo01, lo23);
        lo01 = hi01, lo23 = hi23, hi01 = 0ull, hi23 = 0ull;
      } else if (CARRY && id + sbs == cell) {  // row b -> b - 1: the near row becomes the far row
        flush(c0 + sbs, hi01, hi23);
        hi01 = lo01, hi23 = lo23, lo01 = 0ull, lo23 = 0ull;
      } else {
        flush(c0, lo01, lo23);
        flush(c0 + sbs, hi01, hi23);
        lo01 = lo23 = hi01 = hi23 = 0ull;
      }
      cell = id;
    }
    const float2 w = upk2(fsub2(fab, fsub2(xab, m2)));  // (wa, wb)
    const float wz = fz - (xz - kFloorMagic);
    const unsigned long long pa = ffma2(pk2(w.x, w.x), m1p1, one0);  // (1 - wa, wa)
    const unsigned long long pb = ffma2(pk2(w.y, w.y), m1p1, one0);  // (1 - wb, wb)
    const unsigned long long pzw = ffma2(pk2(wz, wz), m1p1, one0);   // (1 - wz, wz)
    const float2 gg = upk2(fmul2(pk2(gs, gs), pb));                 // (g0, g1): rows b, b + 1
    const float2 l = upk2(fmul2(pk2(gg.x, gg.x), pzw));             // (l0, l1): slices z, z + 1 of row b
    const float2 h = upk2(fmul2(pk2(gg.y, gg.y), pzw));             // (h0, h1): of row b + 1
    lo01 = ffma2(pk2(l.x, l.x), pa, lo01);
    lo23 = ffma2(pk2(l.y, l.y), pa, lo23);
    hi01 = ffma2(pk2(h.x, h.x), pa, hi01);
    hi23 = ffma2(pk2(h.y, h.y), pa, hi23);
  };
  const int nfull = rs.n - 1;
  float kf = 0.5f;
#pragma unroll 2
  for (int k = 0; k < nfull; ++k, kf += 1.f) sample(kf, g);
  sample((float)nfull + 0.5f * rs.last, g * rs.last);
  flush(cell - bias, lo01, lo23);
  flush(cell - bias + sbs, hi01, hi23);
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
    // (two packed components per 64-bit word: fx_unpack)
    auto Y = [&](long long yy, long long xx, long long zz, int c) {
      return fx_unpack(qy[2 * ((yy * px + xx) * pz + zz) + (c >> 1)], c & 1);
    };
    // qx: Qx[x][y][z] taps (z,y),(z,y+1),(z+1,y),(z+1,y+1) of row x
    auto X = [&](long long xx, long long yy, long long zz, int c) {
      return fx_unpack(qx[2 * ((xx * py + yy) * pz + zz) + (c >> 1)], c & 1);
    };
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


// Deterministic A^T.  Pass 1 scatters |y| in fp32 into the same quad cells: the largest
// component, doubled (fp32 rounding of a sum of non-negative terms is far below that), bounds
// every component total of the real scatter in magnitude.  The fixed-point scale 2^e keeps
// those totals below 2^30, so two components share each 64-bit atomic word (fx_pack): pass 2
// scatters y in fixed point with two integer atomics per quad, and the fold sums integers.
// The data-driven bound leaves ~30 bits for the largest tap (a geometric bound on the
// contributions per tap was ~1000x looser and cost the fixed point 5e-5 relative accuracy).
static int launch_fp_adjoint_det(const float *sino, int nz, int ny, int nx, double sz, double sy, double sx,
                                 Scratch &dviews, int n_views, int rows, int cols, double step, float *vol,
                                 cudaStream_t st) {
  constexpr int m2 = 2 * kFpMargin;
  const long long ncell = (long long)(nz + m2) * (ny + m2) * (nx + m2);
  Scratch dmax, qA, qB;
  TK_TRY_CUDA(qA.alloc(16 * ncell, st));
  TK_TRY_CUDA(qB.alloc(16 * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qA.ptr, 0, 16 * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qB.ptr, 0, 16 * ncell, st));
  const long long nbz = (long long)ceil_div(cols, 16) * ceil_div(rows, kFpzRows) * n_views;
  if (nbz >= (1LL << 31)) return fail_arg("tk_forward_cone_3d_adjoint: problem too large for one launch");
  cone_fp_adjoint4z_kernel<8, false, true, true><<<(unsigned)nbz, 128, 0, st>>>(
      sino, qA.ptr, qB.ptr, nx, ny, nz, sx, sy, sz, dviews.as<ConeRayView>(), rows, cols, n_views, step, 1.f);
  TK_LAUNCHED("cone_fp_adjoint4z_kernel");
  TK_TRY_CUDA(dmax.alloc(sizeof(unsigned), st));
  TK_TRY_CUDA(cudaMemsetAsync(dmax.ptr, 0, sizeof(unsigned), st));
  const unsigned mg = (unsigned)std::min<long long>(ceil_div(4 * ncell, 256), (long long)sm_count() * 8);
  absmax_kernel<<<mg, 256, 0, st>>>(qA.as<float>(), 4 * ncell, dmax.as<unsigned>());
  TK_LAUNCHED("absmax_kernel");
  absmax_kernel<<<mg, 256, 0, st>>>(qB.as<float>(), 4 * ncell, dmax.as<unsigned>());
  TK_LAUNCHED("absmax_kernel");
  unsigned bits = 0;
  TK_TRY_CUDA(cudaMemcpyAsync(&bits, dmax.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  TK_TRY_CUDA(cudaStreamSynchronize(st));
  float amax;
  std::memcpy(&amax, &bits, sizeof(float));
  if (!std::isfinite(amax)) return fail_arg("tk_forward_cone_3d_adjoint: non-finite sinogram");
  if (!(amax > 0.f)) {
    TK_TRY_CUDA(cudaMemsetAsync(vol, 0, sizeof(float) * (size_t)nz * ny * nx, st));
    return TK_OK;
  }
  const int e = std::min(100, (int)std::floor(30.0 - std::log2(2.0 * (double)amax)));
  const float scale = std::ldexp(1.0f, e);
  TK_TRY_CUDA(cudaMemsetAsync(qA.ptr, 0, 16 * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qB.ptr, 0, 16 * ncell, st));
  cone_fp_adjoint4z_kernel<8, true><<<(unsigned)nbz, 128, 0, st>>>(sino, qA.ptr, qB.ptr, nx, ny, nz, sx, sy, sz,
                                                                   dviews.as<ConeRayView>(), rows, cols, n_views, step,
                                                                   scale);
  TK_LAUNCHED("cone_fp_adjoint4z_kernel");
  const long long nv = (long long)nz * ny * nx;
  unquad_fx_kernel<<<(unsigned)std::min<long long>(ceil_div(nv, 256), (long long)sm_count() * 16), 256, 0, st>>>(
      qA.as<unsigned long long>(), qB.as<unsigned long long>(), nz, ny, nx, std::ldexp(1.0, -e), vol);
  TK_LAUNCHED("unquad_fx_kernel");
  return TK_OK;
}

static int launch_fp_adjoint(const float *sino, int nz, int ny, int nx, double sz, double sy, double sx,
                             const double *sources, const double *minv, int n_views, int rows, int cols, double step,
                             bool deterministic, float *vol, cudaStream_t st) {
  std::vector<ConeRayView> hv(n_views);
  for (int i = 0; i < n_views; ++i) {
    for (int j = 0; j < 3; ++j) hv[i].src[j] = sources[3 * i + j];
    for (int j = 0; j < 9; ++j) hv[i].minv[j] = minv[9 * i + j];
  }
  Scratch dviews, qA, qB;
  TK_TRY_CUDA(upload(dviews, hv.data(), sizeof(ConeRayView) * n_views, st));
  constexpr int m2 = 2 * kFpMargin;
  const long long ncell = (long long)(nz + m2) * (ny + m2) * (nx + m2);
  if (ncell >= (1LL << 32)) return fail_arg("tk_forward_cone_3d_adjoint: volume too large for 32-bit cell indices");
  if (deterministic)
    return launch_fp_adjoint_det(sino, nz, ny, nx, sz, sy, sx, dviews, n_views, rows, cols, step, vol, st);
  TK_TRY_CUDA(qA.alloc(sizeof(float4) * ncell, st));
  TK_TRY_CUDA(qB.alloc(sizeof(float4) * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qA.ptr, 0, sizeof(float4) * ncell, st));
  TK_TRY_CUDA(cudaMemsetAsync(qB.ptr, 0, sizeof(float4) * ncell, st));
  const long long nbz = (long long)ceil_div(cols, 16) * ceil_div(rows, kFpzRows) * n_views;
  if (nbz >= (1LL << 31)) return fail_arg("tk_forward_cone_3d_adjoint: problem too large for one launch");
  // TK_FPT_CARRY (default 1): carry the far-row quad over on row steps (one reduction instead of two)
  const char *ce = getenv("TK_FPT_CARRY");
  auto kern = (ce && !atoi(ce)) ? cone_fp_adjoint4z_kernel<8, false, false> : cone_fp_adjoint4z_kernel<8>;
  kern<<<(unsigned)nbz, 128, 0, st>>>(sino, qA.ptr, qB.ptr, nx, ny, nz, sx, sy, sz, dviews.as<ConeRayView>(), rows,
                                      cols, n_views, step, 1.f);
  TK_LAUNCHED("cone_fp_adjoint4z_kernel");
  unquad_z_kernel<<<dim3(ceil_div(nz, 32), ceil_div(nx, 32), ny), 256, 0, st>>>(qA.as<float4>(), nz, ny, nx, vol);
  TK_LAUNCHED("unquad_z_kernel");
  unquad_zx_kernel<<<dim3(ceil_div(nz, 32), ceil_div(nx, 32), ny), 256, 0, st>>>(qB.as<float4>(), nz, ny, nx, vol);
  TK_LAUNCHED("unquad_zx_kernel");
  return TK_OK;
}

}  // namespace tk

using namespace tk;

extern "C" {

static int fp_adjoint_args(const float *sino, const float *vol_out, const double *sources, const double *minv, int nz,
                           int ny, int nx, int n_views, int rows, int cols, double sx, double sy, double sz,
                           double step) {
  if (!sino || !vol_out || !sources || !minv) return fail_arg("tk_forward_cone_3d_adjoint: null pointer");
  if (nz < 1 || ny < 1 || nx < 1 || n_views < 1 || rows < 1 || cols < 1)
    return fail_arg("tk_forward_cone_3d_adjoint: non-positive extent");
  if (!(sx > 0 && sy > 0 && sz > 0 && step > 0))
    return fail_arg("tk_forward_cone_3d_adjoint: spacing/step must be > 0");
  return TK_OK;
}

int tk_forward_cone_3d_adjoint_ex(const float *sino, int n_views, int rows, int cols, const double *sources,
                                  const double *minv, int nz, int ny, int nx, double sz, double sy, double sx,
                                  double step, int deterministic, float *vol_out, void *stream) {
  clear_error();
  const int rc = fp_adjoint_args(sino, vol_out, sources, minv, nz, ny, nx, n_views, rows, cols, sx, sy, sz, step);
  if (rc != TK_OK) return rc;
  return launch_fp_adjoint(sino, nz, ny, nx, sz, sy, sx, sources, minv, n_views, rows, cols, step, deterministic != 0,
                           vol_out, as_stream(stream));
}

int tk_forward_cone_3d_adjoint(const float *sino, int n_views, int rows, int cols, const double *sources,
                               const double *minv, int nz, int ny, int nx, double sz, double sy, double sx, double step,
                               float *vol_out, void *stream) {
  return tk_forward_cone_3d_adjoint_ex(sino, n_views, rows, cols, sources, minv, nz, ny, nx, sz, sy, sx, step, 0,
                                       vol_out, stream);
}

}  // extern "C"
