// tk_bp_tma.cu -- TMA-staged voxel-driven cone back projector for sm_100a
// ("tma", default for z-invariant trajectories when the detector width is a
// multiple of 4).  Semantics: reference _kernels.py:281-322 (back_cone_3d).
//
// Why: the quad-gather back projector (tk_cone.cu) is bound by the L1 LSU
// data pipe -- every 16-byte quad load costs one wavefront per 128-byte line
// touched by each quarter-warp (~1.4 lines per quarter at cfg4, ncu), and the
// quad layout itself is a 12 GB expansion written every call.  Here
//   * a CTA owns a 16 x 16 x 32 voxel block; for every view a producer warp
//     projects the block's 8 corners (exact bound of a central projection of a
//     convex box), and one elected lane issues ONE 3D TMA copy of the covering
//     detector rectangle [r0, r0 + bh) x [c0, c0 + BW) of that view (c0 a
//     multiple of 4: TMA box starts must be 16-byte aligned) into a
//     shared-memory stage (out-of-detector texels are zero-filled by the TMA
//     unit: the reference's per-tap zero extension, _kernels.py:308-317);
//   * an mbarrier ring of up to 8 stages (as many as fit two CTAs per SM: 6 at
//     cfg4; full: TMA bytes landed, empty: all 256 consumer threads released)
//     keeps the next views in flight while the consumers (one (x, y) column and
//     32 z-voxels each) gather the 4 bilinear taps of every update with scalar
//     LDS at immediate offsets -- one data-pipe wavefront per warp and tap, the
//     tile pitch BW == 12 or 20 (mod 32) keeping a warp's rows in disjoint banks;
//   * column, depth and (sid/w)^2 are computed once per (column, view); only the
//     row advances along z; floors use floor_magic (no conversion-pipe ops).
// A (block, view) whose rectangle exceeds the TMA box (extreme magnification)
// or that reaches behind the source is gathered from global memory with the
// reference's per-tap bounds instead.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "tk_cone_bp.cuh"
#include "tk_tma.cuh"

namespace tk {

constexpr int kBtTX = 16, kBtTY = 16, kBtMaxStages = 8;
constexpr int kBtConsumers = kBtTX * kBtTY;       // 8 warps
constexpr int kBtThreads = kBtConsumers + 32;     // + 1 producer warp

struct BtMeta {
  int c0, r0, fits, pad;
};

// The views of one launch travel in the kernel's parameter block (constant bank):
// the per-view constants are then uniform constant loads, off the L1 data pipe the
// tile gathers saturate.  Longer scans are launched in blocks of views.
constexpr int kBtParamViews = 640;
struct BtViews {
  float4 q[3 * kBtParamViews];  // (a, b, w) of view v at q[3 v .. 3 v + 2]
};

// ZB = 32 z-voxels per thread (halves the per-view set-up per update against 16);
// BW = the tile row pitch (floats) = the TMA box width, a compile-time constant so a
// voxel's two tile rows are ONE IMAD (row bits x 4 BW + per-view base) and four LDS
// with immediate offsets (0, 4, 4 BW, 4 BW + 4); nst (<= kBtMaxStages) stages in the
// mbarrier ring.
__device__ __forceinline__ float lds_at(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
template <int OFF>
__device__ __forceinline__ float lds_off(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
  return v;
}

template <int BW>
__global__ void __launch_bounds__(kBtThreads, 2)
    cone_bp_tma_kernel(const __grid_constant__ CUtensorMap map, const BpParams p, int weighted, int bh,
                       int stage_floats, int nst, unsigned fbias, int v_base, const __grid_constant__ BtViews pv) {
  constexpr int kBtZB = 32, bw = BW;
  const int kBtStages = nst;
  extern __shared__ float bt_raw[];  // [kBtStages][stage_floats] at a 128-byte aligned base
  // align by an element offset (not through uintptr_t) so the compiler keeps
  // the pointer in the shared window: LDS with 32-bit addresses, not generic LD
  float *bt_tiles = bt_raw + (((128u - (smem_u32(bt_raw) & 127u)) & 127u) >> 2);
  const unsigned tiles_u32 = smem_u32(bt_tiles);
  __shared__ __align__(8) uint64_t full[kBtMaxStages], empty[kBtMaxStages];
  __shared__ BtMeta meta[kBtMaxStages];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kBtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBtConsumers);  // every consumer thread arrives after its last read of the stage
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int zl0 = blockIdx.z * kBtZB;

  if (warp == kBtConsumers / 32) {  // ---------------- producer warp ----------------
    // the block's voxel-centre box in centred index units (clipped to the volume)
    const float bx0 = (float)(blockIdx.x * kBtTX) - p.cx;
    const float bx1 = (float)(min((int)(blockIdx.x + 1) * kBtTX, p.nx) - 1) - p.cx;
    const float by0 = (float)(blockIdx.y * kBtTY) - p.cy;
    const float by1 = (float)(min((int)(blockIdx.y + 1) * kBtTY, p.ny) - 1) - p.cy;
    const float bz0 = (float)(p.z_begin + zl0) - p.cz;
    const float bz1 = bz0 + (float)(kBtZB - 1);  // consumers evaluate all kBtZB rows (stores are masked)
    const unsigned tx_bytes = (unsigned)(bw * bh * 4);
    int s = 0;
    unsigned eph = 1u;  // parity of the empty-barrier phase to wait for (the first lap does not wait)
    for (int v = 0; v < p.n_views; ++v, ++s) {
      if (s == kBtStages) s = 0, eph ^= 1u;
      if (v >= kBtStages) mbar_wait(&empty[s], eph);
      const float4 va = pv.q[3 * v], vb = pv.q[3 * v + 1], vw = pv.q[3 * v + 2];
      float cmin = 3e38f, cmax = -3e38f, rmin = 3e38f, rmax = -3e38f;
      bool behind = false;
      if (lane < 8) {
        const float x = (lane & 1) ? bx1 : bx0, y = (lane & 2) ? by1 : by0, z = (lane & 4) ? bz1 : bz0;
        const float w = fmaf(vw.x, x, fmaf(vw.y, y, fmaf(vw.z, z, vw.w)));
        behind = !(w > (float)kTiny);
        const float rw = 1.f / w;
        const float fc = fmaf(fmaf(va.x, x, fmaf(va.y, y, fmaf(va.z, z, va.w))), rw, p.cu);
        const float fr = fmaf(fmaf(vb.x, x, fmaf(vb.y, y, fmaf(vb.z, z, vb.w))), rw, p.cv);
        cmin = cmax = fc;
        rmin = rmax = fr;
      }
#pragma unroll
      for (int o = 4; o >= 1; o >>= 1) {
        cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
        cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
        rmin = fminf(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
        rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      }
      behind = __any_sync(0xffffffffu, behind);
      if (lane == 0) {
        BtMeta m;
        bool fits = !behind && cmax - cmin < 1e6f && rmax - rmin < 1e6f && cmin > -1e6f &&
                    cmax < 1e6f && rmin > -1e6f && rmax < 1e6f;
        // taps floor(f) and floor(f) + 1, one texel of rounding margin each side
        // the box's innermost start must be 16-byte aligned (TMA faults otherwise): c0 % 4 == 0
        m.c0 = fits ? (((int)floorf(cmin) - 1) & ~3) : 0;
        m.r0 = fits ? (int)floorf(rmin) - 1 : 0;
        fits = fits && (int)floorf(cmax) + 3 - m.c0 <= bw && (int)floorf(rmax) + 3 - m.r0 <= bh;
        m.fits = fits ? 1 : 0;
        m.pad = 0;
        meta[s] = m;
        if (fits) {
          mbar_arrive_tx(&full[s], tx_bytes);
          tma_load_3d(bt_tiles + (size_t)s * stage_floats, &map, m.c0, m.r0, v_base + v, &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- consumer warps: one (x, y) column x kBtZB z-voxels per thread ----------------
  // warp = 8 (x) x 4 (y) voxel columns: its taps cover a compact ~11 x 2-4 patch of
  // the tile, and with a row pitch bw == 12 or 20 (mod 32) the rows it touches fall
  // in disjoint banks -- 1.02 LDS wavefronts per warp instruction instead of 1.37
  // for 16 x 2 warps (scripts/bp_bank_model.py)
  const int ix = blockIdx.x * kBtTX + (warp & 1) * 8 + (lane & 7);
  const int iy = blockIdx.y * kBtTY + (warp >> 1) * 4 + (lane >> 3);
  const bool active = ix < p.nx && iy < p.ny;
  const float xc = (float)ix - p.cx, yc = (float)iy - p.cy;
  const float zc0 = (float)(p.z_begin + zl0) - p.cz;
  // accumulators as packed pairs (z-voxels 2j, 2j+1): the per-update arithmetic
  // runs as FFMA2 / FADD2 / FMUL2 on two voxels at once (same operations and
  // rounding as the scalar form, half the instructions)
  unsigned long long accp[kBtZB / 2];
#pragma unroll
  for (int j = 0; j < kBtZB / 2; ++j) accp[j] = 0ull;
  auto add_acc = [&](int k, float val) {
    float2 a = upk2(accp[k >> 1]);
    if (k & 1)
      a.y += val;
    else
      a.x += val;
    accp[k >> 1] = pk2(a.x, a.y);
  };

  int s = 0;
  unsigned fph = 0u;
  for (int v = 0; v < p.n_views; ++v, ++s) {
    if (s == kBtStages) s = 0, fph ^= 1u;
    mbar_wait(&full[s], fph);
    const BtMeta m = meta[s];
    // the view's constants: uniform constant-bank loads (as 12 scalar global loads they
    // were 8 % of the L1 data pipe's wavefronts, as three 16-byte broadcasts ~2 %)
    const float4 va = pv.q[3 * v], vb = pv.q[3 * v + 1], vw = pv.q[3 * v + 2];
    const float a0 = fmaf(va.x, xc, fmaf(va.y, yc, fmaf(va.z, zc0, va.w)));
    const float b0 = fmaf(vb.x, xc, fmaf(vb.y, yc, fmaf(vb.z, zc0, vb.w)));
    const float w0 = fmaf(vw.x, xc, fmaf(vw.y, yc, fmaf(vw.z, zc0, vw.w)));
    if (active && w0 > (float)kTiny) {  // _kernels.py:297-298
      float rw;  // MUFU.RCP (rel. error 2^-23), one instruction instead of the IEEE division sequence
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rw) : "f"(w0));
      const float fc = fmaf(a0, rw, p.cu);
      const float xcf = floor_magic(fc);
      const float wc = fc - (xcf - kFloorMagic);
      float q = 1.f;
      if (weighted) {  // (sid / w)^2, _kernels.py:318-320 (uniform branch)
        q = p.sid * rw;
        q *= q;
      }
      const float g0 = q * (1.f - wc), g1 = q * wc;
      const float fr0 = fmaf(b0, rw, p.cv);
      const float dr = vb.z * rw;
      if (m.fits) {
        // byte address of tap (row bits, c0) = row_bits * 4 BW + vbase (mod 2^32): the
        // FADD.RM floor's float bits ARE kFloorBits + row
        // fbias = 4 kFloorBits (BW + 1) (mod 2^32) arrives as a kernel argument: as a literal
        // the compiler splits it off the base and re-adds it before every LDS (4 IADD per voxel)
        const unsigned vbase = tiles_u32 + 4u * (unsigned)(s * stage_floats) +
                               4u * (__float_as_uint(xcf) - (unsigned)m.c0) - (unsigned)m.r0 * (4u * BW) - fbias;
        const unsigned long long drp = pk2(dr, dr), fr0p = pk2(fr0, fr0), g0p = pk2(g0, g0), g1p = pk2(g1, g1);
        const unsigned long long mg = pk2(kFloorMagic, kFloorMagic);
#pragma unroll
        for (int j = 0; j < kBtZB / 2; ++j) {
          const unsigned long long frp = ffma2(pk2((float)(2 * j), (float)(2 * j + 1)), drp, fr0p);
          const unsigned long long xrp = fadd2_rm(frp, mg);  // floor_magic of both rows
          const float2 xr = upk2(xrp);
          const unsigned ea = __float_as_uint(xr.x) * (4u * BW) + vbase;
          const unsigned eb = __float_as_uint(xr.y) * (4u * BW) + vbase;
          const unsigned long long e0 = pk2(lds_at(ea), lds_at(eb)), e1 = pk2(lds_off<4>(ea), lds_off<4>(eb));
          const unsigned long long e2 = pk2(lds_off<4 * BW>(ea), lds_off<4 * BW>(eb));
          const unsigned long long e3 = pk2(lds_off<4 * BW + 4>(ea), lds_off<4 * BW + 4>(eb));
          const unsigned long long top = ffma2(g1p, e1, fmul2(g0p, e0));
          const unsigned long long bot = ffma2(g1p, e3, fmul2(g0p, e2));
          const unsigned long long frac = fsub2(frp, fsub2(xrp, mg));
          accp[j] = fadd2(accp[j], ffma2(frac, fsub2(bot, top), top));
        }
      } else {  // rectangle exceeds the TMA box: bounded global gathers
        const float *sv = p.sino + (long long)v * p.view_stride;
        const int c0 = (int)(__float_as_uint(xcf) - kFloorBits);
        const bool ca = (unsigned)c0 < (unsigned)p.cols, cb = (unsigned)(c0 + 1) < (unsigned)p.cols;
#pragma unroll
        for (int k = 0; k < kBtZB; ++k) {
          const float fr = fmaf((float)k, dr, fr0);
          const float flr = floorf(fr);
          const int r0 = (int)flr;
          const bool ra = (unsigned)r0 < (unsigned)p.band_rows;
          const bool rb = (unsigned)(r0 + 1) < (unsigned)p.band_rows;
          const float *e = sv + (long long)r0 * p.cols + c0;
          const float t00 = (ra && ca) ? __ldg(e) : 0.f, t01 = (ra && cb) ? __ldg(e + 1) : 0.f;
          const float t10 = (rb && ca) ? __ldg(e + p.cols) : 0.f;
          const float t11 = (rb && cb) ? __ldg(e + p.cols + 1) : 0.f;
          const float top = fmaf(g1, t01, g0 * t00);
          const float bot = fmaf(g1, t11, g0 * t10);
          add_acc(k, fmaf(fr - flr, bot - top, top));
        }
      }
    }
    mbar_arrive(&empty[s]);  // release: this thread's reads of meta[s] and the tile happen before the refill
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < kBtZB; ++k) {
    const int zl = zl0 + k;
    if (zl < p.z_count) {
      const float2 a = upk2(accp[k >> 1]);
      const float ak = (k & 1) ? a.y : a.x;
      float *o = p.out + ((long long)zl * p.ny + iy) * p.nx + ix;
      *o = p.accumulate ? *o + ak : ak;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// Detector rectangle (columns, rows) a 16^3 block needs in the worst sampled
// (block, view): volume-shell and interior blocks x up to 24 views.  Blocks or
// views outside the sample that need more fall back to global gathers in-kernel.
static void footprint_box(const BpParams &p, const ConeVoxView *hv, int kBtZB, int &bw, int &bh) {
  const int nbx = (p.nx + kBtTX - 1) / kBtTX, nby = (p.ny + kBtTY - 1) / kBtTY;
  const int nbz = (p.z_count + kBtZB - 1) / kBtZB;
  auto picks = [](int n) {
    std::vector<int> v = {0, 1, n / 4, n / 2, (3 * n) / 4, n - 2, n - 1};
    std::vector<int> out;
    for (int x : v)
      if (x >= 0 && x < n && std::find(out.begin(), out.end(), x) == out.end()) out.push_back(x);
    return out;
  };
  const std::vector<int> px = picks(nbx), py = picks(nby), pz = picks(nbz);
  const int nv = std::min(p.n_views, 24);
  int wmax = 2, hmax = 2;
  for (int iv = 0; iv < nv; ++iv) {
    const ConeVoxView &V = hv[(long long)iv * p.n_views / nv];
    for (int bx : px)
      for (int by : py)
        for (int bz : pz) {
          const double x0 = bx * kBtTX - (double)p.cx, x1 = std::min((bx + 1) * kBtTX, p.nx) - 1 - (double)p.cx;
          const double y0 = by * kBtTY - (double)p.cy, y1 = std::min((by + 1) * kBtTY, p.ny) - 1 - (double)p.cy;
          const double z0 = p.z_begin + bz * kBtZB - (double)p.cz;
          const double z1 = z0 + (kBtZB - 1);
          double cmin = 1e300, cmax = -1e300, rmin = 1e300, rmax = -1e300;
          bool ok = true;
          for (int i = 0; i < 8; ++i) {
            const double x = (i & 1) ? x1 : x0, y = (i & 2) ? y1 : y0, z = (i & 4) ? z1 : z0;
            const double w = V.w[0] * x + V.w[1] * y + V.w[2] * z + V.w[3];
            if (!(w > 1e-12)) {
              ok = false;
              break;
            }
            const double fc = (V.a[0] * x + V.a[1] * y + V.a[2] * z + V.a[3]) / w + p.cu;
            const double fr = (V.b[0] * x + V.b[1] * y + V.b[2] * z + V.b[3]) / w + p.cv;
            cmin = std::min(cmin, fc), cmax = std::max(cmax, fc);
            rmin = std::min(rmin, fr), rmax = std::max(rmax, fr);
          }
          if (!ok || cmax - cmin > 4096 || rmax - rmin > 4096) continue;
          wmax = std::max(wmax, (int)std::floor(cmax) + 3 - ((int)std::floor(cmin) - 1));
          hmax = std::max(hmax, (int)std::floor(rmax) + 3 - ((int)std::floor(rmin) - 1));
        }
  }
  bw = ((wmax + 3 + 2 + 3) / 4) * 4;  // +3 for the 16-byte aligned start column, +2 slack
  bh = hmax + 2;
}

// Tile pitches: the TMA box width, == 12 or 20 (mod 32) so that an 8 x 4 warp's taps on
// neighbouring tile rows fall in disjoint banks (scripts/bp_bank_model.py).
template <int BW>
static int launch_bp_tma_t(const BpParams &p, const ConeVoxView *host_views, const CUtensorMap &map, bool weighted,
                           int bh, int stage_floats, int nst, cudaStream_t st) {
  const size_t smem = sizeof(float) * (size_t)stage_floats * nst + 128;
  auto kern = cone_bp_tma_kernel<BW>;
  TK_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((p.nx + kBtTX - 1) / kBtTX, (p.ny + kBtTY - 1) / kBtTY, (p.z_count + 31) / 32);
  static thread_local BtViews pv;
  const int nblk = (p.n_views + kBtParamViews - 1) / kBtParamViews;
  const int per = (p.n_views + nblk - 1) / nblk;  // equal blocks: each launch refills its ring once
  for (int v0 = 0; v0 < p.n_views; v0 += per) {
    const int cnt = std::min(per, p.n_views - v0);
    BpParams pb = p;
    pb.n_views = cnt;
    pb.sino = p.sino + (long long)v0 * p.view_stride;
    pb.views = p.views + v0;
    pb.accumulate = p.accumulate || v0 > 0;
    std::memcpy(pv.q, host_views + v0, sizeof(ConeVoxView) * cnt);
    kern<<<grid, kBtThreads, smem, st>>>(map, pb, weighted ? 1 : 0, bh, stage_floats, nst,
                                         kFloorBits * (4u * BW) + 4u * kFloorBits, v0, pv);
    TK_LAUNCHED("cone_bp_tma_kernel");
  }
  return TK_OK;
}

static const int kBtPitches[] = {44, 52, 76, 84, 108, 116, 140, 148, 172, 180, 204, 212, 236, 244};

int launch_bp_tma(const BpParams &p, const ConeVoxView *host_views, bool weighted, cudaStream_t st) {
  auto enc = encode_fn();
  if (!enc) return -1;
  if (p.cols % 4 != 0 || (reinterpret_cast<uintptr_t>(p.sino) & 15) != 0) return -1;
  if (p.view_stride != (long long)p.band_rows * p.cols) return -1;
  int need = 0, bh = 0;
  footprint_box(p, host_views, 32, need, bh);
  int bw = 0;
  for (int w : kBtPitches)
    if (w >= need) {
      bw = w;
      break;
    }
  if (bw == 0 || bh > 256) return -1;
  const int stage_floats = ((bw * bh + 31) / 32) * 32;  // 128-byte aligned stages
  // stages: as many as fit (<= 8) with two CTAs per SM
  int nst = kBtMaxStages;
  while (nst > 2 && sizeof(float) * (size_t)stage_floats * nst + 128 > 110 * 1024) --nst;
  if (sizeof(float) * (size_t)stage_floats * nst + 128 > 110 * 1024) return -1;

  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)p.cols, (cuuint64_t)p.band_rows, (cuuint64_t)p.n_views};
  const cuuint64_t strides[2] = {(cuuint64_t)p.cols * 4, (cuuint64_t)p.band_rows * p.cols * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(p.sino), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -1;
  switch (bw) {
    case 44: return launch_bp_tma_t<44>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 52: return launch_bp_tma_t<52>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 76: return launch_bp_tma_t<76>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 84: return launch_bp_tma_t<84>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 108: return launch_bp_tma_t<108>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 116: return launch_bp_tma_t<116>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 140: return launch_bp_tma_t<140>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 148: return launch_bp_tma_t<148>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 172: return launch_bp_tma_t<172>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 180: return launch_bp_tma_t<180>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 204: return launch_bp_tma_t<204>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 212: return launch_bp_tma_t<212>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    case 236: return launch_bp_tma_t<236>(p, host_views, map, weighted, bh, stage_floats, nst, st);
    default: return launch_bp_tma_t<244>(p, host_views, map, weighted, bh, stage_floats, nst, st);
  }
}

}  // namespace tk
