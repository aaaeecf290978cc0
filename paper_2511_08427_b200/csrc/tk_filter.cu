// tk_filter.cu -- FBP/FDK row filter on sm_100a: fused obliquity pre-weight,
// zero padding, FFT, real frequency weights, inverse FFT, crop and scale.
//
// Reference: /root/reference/pkg/src/tomokit/filters.py:136-171
// (fft_filter, cosine_preweight_cone, _preweight_fan).  Because the weights
// are real and even (weights[k] == weights[n_pad-k], filters.py:104-106), two
// real rows a, b are filtered with ONE complex transform of z = a + i b:
// IFFT(W * FFT(z)) = filt(a) + i filt(b).
//
// One CTA owns a row pair at a time (grid-stride).  The n_pad-point transform
// is a mixed-radix Stockham FFT (radix 8 stages, one radix 4/2 stage) with
// every butterfly in registers and shared memory only between stages, so a
// 2048-point transform is 4 stages instead of 11.  The first forward stage
// reads the (pre-weighted, zero-padded) rows straight from global memory and
// the last inverse stage writes the cropped result straight back; the weights
// and the 1/n_pad normalisation are applied while loading the first inverse
// stage.  The inverse uses IFFT(y) = conj(FFT(conj(y))) / n.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tk_common.cuh"

namespace tk {

constexpr int kMaxPad = 8192;

struct FilterParams {
  const float *in;
  float *out;
  long long n_rows;
  int width, band_rows, row_offset, det_rows, n_pad;
  const float2 *tw;  // exp(-2 pi i m / n_pad), m < n_pad
  const float *wgt;   // half weights * scale / n_pad, n_pad/2 + 1 entries
  float sdd, du, dv;  // obliquity pre-weight (disabled when sdd <= 0)
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // * (-i)

// forward DFTs in registers, natural order
__device__ __forceinline__ void dft2(float2 *v) {
  const float2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

__device__ __forceinline__ void dft4(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
  const float2 s02 = cadd(x0, x2), d02 = csub(x0, x2), s13 = cadd(x1, x3), d13 = csub(x1, x3);
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, mul_mi(d13));
  x3 = csub(d02, mul_mi(d13));
}

__device__ __forceinline__ void dft8(float2 *v) {
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4(e0, e1, e2, e3);
  dft4(o0, o1, o2, o3);
  const float r = 0.70710678118654752440f;
  o1 = make_float2(r * (o1.x + o1.y), r * (o1.y - o1.x));    // * W8^1 = (1 - i)/sqrt2
  o2 = mul_mi(o2);                                           // * W8^2 = -i
  o3 = make_float2(r * (o3.y - o3.x), -r * (o3.x + o3.y));   // * W8^3 = (-1 - i)/sqrt2
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1);
  v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2);
  v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3);
  v[7] = csub(e3, o3);
}

__device__ __forceinline__ float preweight(const FilterParams &p, long long row, int i) {
  if (!(p.sdd > 0.f)) return 1.f;
  const int r = (int)(row % p.band_rows) + p.row_offset;
  const float u = ((float)i - 0.5f * (float)(p.width - 1)) * p.du;
  const float v = ((float)r - 0.5f * (float)(p.det_rows - 1)) * p.dv;
  return p.sdd * rsqrtf(fmaf(p.sdd, p.sdd, fmaf(u, u, v * v)));  // ~2 ulp, well inside 1e-4
}

// Source of stage inputs: 0 = shared buffer, 1 = global rows (first forward
// stage), 2 = shared buffer x weights, conjugated (first inverse stage).
// Destination: 0 = shared buffer, 1 = global rows conjugated (last inverse stage).
//
// Every thread owns 8 complex values per stage: one radix-8 butterfly, two
// radix-4 or four radix-2 butterflies (blockDim = N/8), so the register
// footprint is the same 8 values in every stage.
template <int R>
__device__ __noinline__ void stockham_stage(float2 *x, const float2 *tw, int N, int Ns, int src,
                                               int dst, const FilterParams &p, const float *ia,
                                               const float *ib, long long ra, long long rb,
                                               bool has_b, float *oa, float *ob, const float *wgt) {
  constexpr int kB = 8 / R;  // butterflies per thread
  const int nb = N / R;
  const int tstride = N / (Ns * R);
  const bool active = (int)threadIdx.x * kB < nb;
  float2 v[8];
  if (active) {
#pragma unroll
    for (int c = 0; c < kB; ++c) {
      const int j = threadIdx.x * kB + c;
      const int k = j & (Ns - 1);  // Ns is a power of two
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int e = j + r * nb;
        float2 z;
        if (src == 1) {
          float a = 0.f, b = 0.f;
          if (e < p.width) {
            a = __ldg(ia + e) * preweight(p, ra, e);
            if (has_b) b = __ldg(ib + e) * preweight(p, rb, e);
          }
          z = make_float2(a, b);
        } else {
          z = x[e + (e >> 4)];  // one float2 of padding per 16: conflict-free strides
          if (src == 2) {
            const float w = wgt[e <= N / 2 ? e : N - e];
            z = make_float2(z.x * w, -z.y * w);
          }
        }
        v[c * R + r] = (r > 0 && Ns > 1) ? cmul(z, tw[r * k * tstride]) : z;
      }
      if (R == 8) dft8(v);
      if (R == 4) dft4(v[c * 4], v[c * 4 + 1], v[c * 4 + 2], v[c * 4 + 3]);
      if (R == 2) dft2(v + c * 2);
    }
  }
  __syncthreads();  // every thread has read its inputs (in-place buffer)
  if (active) {
#pragma unroll
    for (int c = 0; c < kB; ++c) {
      const int j = threadIdx.x * kB + c;
      const int k = j & (Ns - 1);  // Ns is a power of two
      const int base = (j - k) * R + k;  // (j / Ns) * Ns * R + k
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int o = base + r * Ns;
        if (dst == 1) {
          if (o < p.width) {
            oa[o] = v[c * R + r].x;
            if (has_b) ob[o] = -v[c * R + r].y;
          }
        } else {
          x[o + (o >> 4)] = v[c * R + r];
        }
      }
    }
  }
  __syncthreads();
}

// Compile-time stage plan for N = 2^LOGN: radix-8 stages first, then one
// radix-4 or radix-2 stage; stage S of the forward (INV = false) or inverse
// pass, recursing to the next stage.
template <int LOGN>
struct FftPlan {
  static constexpr int kN = 1 << LOGN;
  static constexpr int kStages8 = LOGN / 3;
  static constexpr int kRem = LOGN % 3;
  static constexpr int kStages = kStages8 + (kRem ? 1 : 0);
  static constexpr int radix(int s) { return s < kStages8 ? 8 : (kRem == 1 ? 2 : 4); }
  static constexpr int span(int s) { return s == 0 ? 1 : span(s - 1) * radix(s - 1); }
};

template <int LOGN, bool INV, int S>
__device__ __forceinline__ void fft_pass(float2 *x, const float2 *tw, const FilterParams &p,
                                         const float *ia, const float *ib, long long ra,
                                         long long rb, bool has_b, float *oa, float *ob,
                                         const float *wgt) {
  using P = FftPlan<LOGN>;
  if constexpr (S < P::kStages) {
    constexpr int src = S == 0 ? (INV ? 2 : 1) : 0;
    constexpr int dst = (INV && S == P::kStages - 1) ? 1 : 0;
    stockham_stage<P::radix(S)>(x, tw, P::kN, P::span(S), src, dst, p, ia, ib, ra, rb, has_b, oa,
                                ob, wgt);
    fft_pass<LOGN, INV, S + 1>(x, tw, p, ia, ib, ra, rb, has_b, oa, ob, wgt);
  }
}

template <int LOGN>
constexpr int filter_threads() {
  return (1 << LOGN) / 8 < 32 ? 32 : ((1 << LOGN) / 8 > 1024 ? 1024 : (1 << LOGN) / 8);
}

template <int LOGN>
__global__ void __launch_bounds__(filter_threads<LOGN>(), (filter_threads<LOGN>() <= 256 ? 3 : 1)) fft_filter_kernel(const FilterParams p) {
  extern __shared__ float smem[];
  constexpr int N = 1 << LOGN;
  float2 *x = reinterpret_cast<float2 *>(smem);
  float2 *tw = x + N + N / 16;
  float *wgt = reinterpret_cast<float *>(tw + N);
  for (int i = threadIdx.x; i < N; i += blockDim.x) tw[i] = p.tw[i];
  for (int i = threadIdx.x; i <= N / 2; i += blockDim.x) wgt[i] = p.wgt[i];
  __syncthreads();
  const long long n_pairs = (p.n_rows + 1) / 2;
  for (long long pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
    const long long ra = 2 * pair, rb = ra + 1;
    const bool has_b = rb < p.n_rows;
    const float *ia = p.in + ra * p.width;
    const float *ib = p.in + rb * p.width;
    float *oa = p.out + ra * p.width;
    float *ob = p.out + rb * p.width;
    fft_pass<LOGN, false, 0>(x, tw, p, ia, ib, ra, rb, has_b, oa, ob, wgt);  // forward
    fft_pass<LOGN, true, 0>(x, tw, p, ia, ib, ra, rb, has_b, oa, ob, wgt);   // x W, inverse
  }
}

// ---------------------------------------------------------------------------
// Warp-per-row-pair variant: each warp owns one row pair at a time and two
// private shared buffers (ping-pong), so a Stockham stage reads one buffer and
// writes the other with only __syncwarp between stages -- no CTA barriers, and
// every warp progresses independently (latency hidden across warps).
// Twiddles come from the global table through L1.
// ---------------------------------------------------------------------------
constexpr int kFwWarps = 4;

template <int R>
__device__ __forceinline__ void warp_stage(const float2 *__restrict__ xin, float2 *__restrict__ xout,
                                           const float2 *__restrict__ tw, int N, int Ns, int src,
                                           int dst, const FilterParams &p, const float *ia,
                                           const float *ib, long long ra, long long rb, bool has_b,
                                           float *oa, float *ob, const float *__restrict__ wgt) {
  const int lane = threadIdx.x & 31;
  const int nb = N / R;
  const int tstride = N / (Ns * R);
  for (int j = lane; j < nb; j += 32) {
    const int k = j & (Ns - 1);  // Ns is a power of two
    float2 v[8];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = j + r * nb;
      float2 z;
      if (src == 1) {
        float a = 0.f, b = 0.f;
        if (e < p.width) {
          a = __ldg(ia + e) * preweight(p, ra, e);
          if (has_b) b = __ldg(ib + e) * preweight(p, rb, e);
        }
        z = make_float2(a, b);
      } else {
        z = xin[e];
        if (src == 2) {
          const float w = __ldg(wgt + (e <= N / 2 ? e : N - e));
          z = make_float2(z.x * w, -z.y * w);
        }
      }
      v[r] = (r > 0 && Ns > 1) ? cmul(z, __ldg(tw + r * k * tstride)) : z;
    }
    if (R == 8) dft8(v);
    if (R == 4) dft4(v[0], v[1], v[2], v[3]);
    if (R == 2) dft2(v);
    const int base = (j - k) * R + k;  // (j / Ns) * Ns * R + k
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int o = base + r * Ns;
      if (dst == 1) {
        if (o < p.width) {
          oa[o] = v[r].x;
          if (has_b) ob[o] = -v[r].y;
        }
      } else {
        xout[o] = v[r];
      }
    }
  }
  __syncwarp();
}

template <int LOGN, bool INV, int S>
__device__ __forceinline__ void warp_pass(float2 *bufA, float2 *bufB, const float2 *tw,
                                          const FilterParams &p, const float *ia, const float *ib,
                                          long long ra, long long rb, bool has_b, float *oa,
                                          float *ob, const float *wgt) {
  using P = FftPlan<LOGN>;
  if constexpr (S < P::kStages) {
    constexpr int src = S == 0 ? (INV ? 2 : 1) : 0;
    constexpr int dst = (INV && S == P::kStages - 1) ? 1 : 0;
    // stage S reads buffer (S odd ? B : A) and writes the other; the forward
    // pass leaves its result in buffer (kStages odd ? B : A) = the inverse input
    constexpr bool flip = INV && (P::kStages % 2 == 1);
    constexpr bool read_b = ((S % 2) == 1) != flip;
    warp_stage<P::radix(S)>(read_b ? bufB : bufA, read_b ? bufA : bufB, tw, P::kN, P::span(S), src,
                            dst, p, ia, ib, ra, rb, has_b, oa, ob, wgt);
    warp_pass<LOGN, INV, S + 1>(bufA, bufB, tw, p, ia, ib, ra, rb, has_b, oa, ob, wgt);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(32 * kFwWarps) fft_filter_warp_kernel(const FilterParams p) {
  extern __shared__ float smem[];
  constexpr int N = 1 << LOGN;
  const int warp = threadIdx.x >> 5;
  float2 *bufA = reinterpret_cast<float2 *>(smem) + (size_t)warp * 2 * N;
  float2 *bufB = bufA + N;
  const long long n_pairs = (p.n_rows + 1) / 2;
  for (long long pair = (long long)blockIdx.x * kFwWarps + warp; pair < n_pairs;
       pair += (long long)gridDim.x * kFwWarps) {
    const long long ra = 2 * pair, rb = ra + 1;
    const bool has_b = rb < p.n_rows;
    const float *ia = p.in + ra * p.width;
    const float *ib = p.in + rb * p.width;
    float *oa = p.out + ra * p.width;
    float *ob = p.out + rb * p.width;
    // forward: stage 0 reads global and writes A (buffer names per warp_pass)
    warp_pass<LOGN, false, 0>(bufB, bufA, p.tw, p, ia, ib, ra, rb, has_b, oa, ob, p.wgt);
    warp_pass<LOGN, true, 0>(bufB, bufA, p.tw, p, ia, ib, ra, rb, has_b, oa, ob, p.wgt);
  }
}

// ---------------------------------------------------------------------------
// Register-resident radix-16 variant ("r16", default for 512 <= n_pad <= 4096).
//
// T = n_pad / 16 threads own one row pair; every thread holds 16 complex
// values.  Forward plan [16, 16, ..., r_last] (Stockham), inverse plan the
// mirror image [r_last, ..., 16]: the forward's last stage leaves thread t with
// the spectrum bins  j + (N / r_last) * r  of its butterflies j -- exactly the
// inputs of the inverse's first (Ns = 1) stage, so the frequency weights, the
// conjugation and that first inverse butterfly run on registers with no
// shared-memory round trip.  Shared memory (ping-pong, one barrier per
// exchange) only carries the data between the other stages.  The obliquity
// pre-weight's row term is computed once per row, not per sample.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dft16(float2 *v) {
  float2 e[8], o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  dft8(e);
  dft8(o);
  // o[k] *= W16^k = exp(-2 pi i k / 16)
  const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
  const float r2 = 0.70710678118654752440f;
  const float2 w[8] = {{1.f, 0.f}, {c1, -s1}, {r2, -r2}, {s1, -c1},
                       {0.f, -1.f}, {-s1, -c1}, {-r2, -r2}, {-c1, -s1}};
#pragma unroll
  for (int k = 1; k < 8; ++k) o[k] = cmul(o[k], w[k]);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = cadd(e[k], o[k]);
    v[k + 8] = csub(e[k], o[k]);
  }
}

template <int R>
__device__ __forceinline__ void dft_r(float2 *v) {
  if constexpr (R == 16) dft16(v);
  if constexpr (R == 8) dft8(v);
  if constexpr (R == 4) dft4(v[0], v[1], v[2], v[3]);
  if constexpr (R == 2) dft2(v);
}

template <int LOGN>
struct R16Plan {
  static constexpr int kN = 1 << LOGN;
  static constexpr int kT = kN / 16;                    // threads per row pair
  static constexpr int kFull = LOGN / 4;                // radix-16 stages
  static constexpr int kRem = LOGN % 4;                 // last radix 2^kRem (0: none)
  static constexpr int kStages = kFull + (kRem ? 1 : 0);
  static constexpr int radix(int s) { return s < kFull ? 16 : (1 << kRem); }     // forward
  static constexpr int iradix(int s) { return radix(kStages - 1 - s); }          // inverse
  static constexpr int span(int s) { return s == 0 ? 1 : span(s - 1) * radix(s - 1); }
  static constexpr int ispan(int s) { return s == 0 ? 1 : ispan(s - 1) * iradix(s - 1); }
  // per-stage twiddle tables (w1[NS], w4[NS]) for stages 1..kStages-1, forward then inverse
  static constexpr int fwd_off(int s) { return s <= 1 ? 0 : fwd_off(s - 1) + 2 * span(s - 1); }
  static constexpr int inv_off(int s) {
    return s <= 1 ? fwd_off(kStages) : inv_off(s - 1) + 2 * ispan(s - 1);
  }
  static constexpr int kTabs = inv_off(kStages);
};

__device__ __forceinline__ int r16_pad(int e) { return e + (e >> 4); }

// Twiddles W_{Ns R}^{r k}, r = 1..R-1, from two table entries w1 = W^k and
// w4 = W^{4k} (per-stage tables indexed by k: conflict-free shared loads; the
// full-circle table indexed by r k stride is 8- to 16-way bank conflicted).
// Products are at most four deep (a few ulp, far inside the 1e-4 budget).
template <int R>
__device__ __forceinline__ void apply_twiddles(float2 *v, float2 w1, float2 w4) {
  if constexpr (R == 2) {
    v[1] = cmul(v[1], w1);
  } else {
    const float2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    if constexpr (R >= 8) {
      v[4] = cmul(v[4], w4);
      v[5] = cmul(v[5], cmul(w4, w1));
      v[6] = cmul(v[6], cmul(w4, w2));
      v[7] = cmul(v[7], cmul(w4, w3));
    }
    if constexpr (R == 16) {
      const float2 w8 = cmul(w4, w4), w12 = cmul(w8, w4);
      v[8] = cmul(v[8], w8);
      v[9] = cmul(v[9], cmul(w8, w1));
      v[10] = cmul(v[10], cmul(w8, w2));
      v[11] = cmul(v[11], cmul(w8, w3));
      v[12] = cmul(v[12], w12);
      v[13] = cmul(v[13], cmul(w12, w1));
      v[14] = cmul(v[14], cmul(w12, w2));
      v[15] = cmul(v[15], cmul(w12, w3));
    }
  }
}

// One Stockham stage on registers v[16] (16/R butterflies per thread):
// twiddles (stage table `tab`: NS entries w1 then NS entries w4), then the DFT.
template <int R, int N, int NS>
__device__ __forceinline__ void r16_butterflies(float2 *v, const float2 *__restrict__ tab) {
  constexpr int kB = 16 / R;
#pragma unroll
  for (int c = 0; c < kB; ++c) {
    const int j = threadIdx.x * kB + c;
    const int k = j & (NS - 1);
    if constexpr (NS > 1) apply_twiddles<R>(v + c * R, tab[k], tab[NS + k]);
    dft_r<R>(v + c * R);
  }
}

template <int R, int N, int NS>
__device__ __forceinline__ void r16_gather(float2 *v, const float2 *__restrict__ buf) {
  constexpr int kB = 16 / R;
  constexpr int nb = N / R;
#pragma unroll
  for (int c = 0; c < kB; ++c) {
    const int j = threadIdx.x * kB + c;
#pragma unroll
    for (int r = 0; r < R; ++r) v[c * R + r] = buf[r16_pad(j + r * nb)];
  }
}

template <int R, int N, int NS>
__device__ __forceinline__ void r16_scatter(const float2 *v, float2 *__restrict__ buf) {
  constexpr int kB = 16 / R;
#pragma unroll
  for (int c = 0; c < kB; ++c) {
    const int j = threadIdx.x * kB + c;
    const int k = j & (NS - 1);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[r16_pad(base + r * NS)] = v[c * R + r];
  }
}

template <int LOGN, int S>
__device__ __forceinline__ void r16_forward(float2 *v, float2 *b0, float2 *b1, const float2 *tw) {
  using P = R16Plan<LOGN>;
  if constexpr (S < P::kStages) {
    constexpr int R = P::radix(S), NS = P::span(S);
    if constexpr (S > 0) {  // stage S reads buffer (S-1)&1
      r16_gather<R, P::kN, NS>(v, ((S - 1) & 1) ? b1 : b0);
    }
    r16_butterflies<R, P::kN, NS>(v, tw + P::fwd_off(S));
    if constexpr (S < P::kStages - 1) {
      r16_scatter<R, P::kN, NS>(v, (S & 1) ? b1 : b0);
      __syncthreads();
    }
    r16_forward<LOGN, S + 1>(v, b0, b1, tw);
  }
}

// inverse stages 1.. (stage 0 runs on registers in the kernel body and
// scatters to buffer X0); stage S reads buffer X0 ^ ((S-1)&1), writes X0 ^ (S&1)
template <int LOGN, int X0, int S>
__device__ __forceinline__ void r16_inverse(float2 *v, float2 *b0, float2 *b1, const float2 *tw) {
  using P = R16Plan<LOGN>;
  if constexpr (S < P::kStages) {
    constexpr int R = P::iradix(S), NS = P::ispan(S);
    r16_gather<R, P::kN, NS>(v, (X0 ^ ((S - 1) & 1)) ? b1 : b0);
    r16_butterflies<R, P::kN, NS>(v, tw + P::inv_off(S));
    if constexpr (S < P::kStages - 1) {
      r16_scatter<R, P::kN, NS>(v, (X0 ^ (S & 1)) ? b1 : b0);
      __syncthreads();
    }
    r16_inverse<LOGN, X0, S + 1>(v, b0, b1, tw);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(R16Plan<LOGN>::kT, 512 / R16Plan<LOGN>::kT) fft_filter_r16_kernel(const FilterParams p) {
  using P = R16Plan<LOGN>;
  constexpr int N = P::kN, T = P::kT;
  constexpr int padN = N + N / 16;
  constexpr int kX0 = 1 - ((P::kStages - 2) & 1);  // buffer not read by the last forward stage
  extern __shared__ float smem[];
  float2 *b0 = reinterpret_cast<float2 *>(smem);
  float2 *b1 = b0 + padN;
  float2 *tw = b1 + padN;  // per-stage twiddle tables (R16Plan::kTabs entries)
  float *wgt = reinterpret_cast<float *>(tw + P::kTabs);
  float *stage_in = wgt + (N / 2 + 1);  // next row pair (N/2 + N/2 floats), filled by cp.async
  for (int i = threadIdx.x; i < P::kTabs; i += T) {
    // locate stage (forward s or inverse s) and entry of table slot i
    int ns = 1, r = 1, base = 0;
    bool found = false;
#pragma unroll
    for (int st = 1; st < P::kStages; ++st) {
      if (!found && i >= P::fwd_off(st) && i < P::fwd_off(st) + 2 * P::span(st)) {
        ns = P::span(st), r = P::radix(st), base = P::fwd_off(st), found = true;
      }
      if (!found && i >= P::inv_off(st) && i < P::inv_off(st) + 2 * P::ispan(st)) {
        ns = P::ispan(st), r = P::iradix(st), base = P::inv_off(st), found = true;
      }
    }
    const int e = i - base, k = e % ns, mult = e < ns ? 1 : 4;
    const int tstride = N / (ns * r);  // W_{ns r}^{mult k} = W_N^{mult k tstride}
    tw[i] = p.tw[(mult * k * tstride) & (N - 1)];
  }
  for (int i = threadIdx.x; i <= N / 2; i += T) wgt[i] = p.wgt[i];
  __syncthreads();
  const bool pre = p.sdd > 0.f;
  const float ucen = 0.5f * (float)(p.width - 1), vcen = 0.5f * (float)(p.det_rows - 1);
  const float sdd2 = p.sdd * p.sdd;
  const long long n_pairs = (p.n_rows + 1) / 2;
  // Each thread stages exactly the input elements it consumes in forward stage
  // 0 (e = j + r N/16), so the prefetch of pair k+1 needs no barrier: it is
  // issued after this thread has read pair k's values into registers, and
  // lands while the rest of pair k's transforms run.
  constexpr int R0 = P::radix(0), kB0 = 16 / R0, nb0 = N / R0;
  auto prefetch = [&](long long pr) {
    if (pr >= n_pairs) return;
    const long long r0 = 2 * pr;
    const bool hb = r0 + 1 < p.n_rows;
    const float *ga = p.in + r0 * p.width, *gb = ga + p.width;
#pragma unroll
    for (int c = 0; c < kB0; ++c) {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int e = threadIdx.x * kB0 + c + r * nb0;
        if (e < p.width) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(stage_in + e);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(ga + e));
          if (hb) {
            const unsigned sb = (unsigned)__cvta_generic_to_shared(stage_in + N / 2 + e);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sb), "l"(gb + e));
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  prefetch(blockIdx.x);
  for (long long pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
    const long long ra = 2 * pair, rb = ra + 1;
    const bool has_b = rb < p.n_rows;
    asm volatile("cp.async.wait_all;" ::: "memory");
    // obliquity pre-weight: row term once per row (reference filters.py:154-171)
    float qa = 0.f, qb = 0.f;
    if (pre) {
      const float va = ((float)((int)(ra % p.band_rows) + p.row_offset) - vcen) * p.dv;
      const float vb = ((float)((int)(rb % p.band_rows) + p.row_offset) - vcen) * p.dv;
      qa = fmaf(va, va, sdd2);
      qb = fmaf(vb, vb, sdd2);
    }
    float2 v[16];
    {  // forward stage 0 (Ns = 1): the zero-padded rows from this thread's staged elements
#pragma unroll
      for (int c = 0; c < kB0; ++c) {
        const int j = threadIdx.x * kB0 + c;
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int e = j + r * nb0;
          float a = 0.f, b = 0.f;
          if (e < p.width) {
            a = stage_in[e];
            if (has_b) b = stage_in[N / 2 + e];
            if (pre) {
              const float u = ((float)e - ucen) * p.du;
              a *= p.sdd * rsqrtf(fmaf(u, u, qa));
              b *= p.sdd * rsqrtf(fmaf(u, u, qb));
            }
          }
          v[c * R0 + r] = make_float2(a, b);
        }
      }
    }
    prefetch(pair + gridDim.x);
    r16_forward<LOGN, 0>(v, b0, b1, tw);
    {  // weights (real, even, scale / N folded in), conjugate, inverse stage 0 -- on registers
      constexpr int RL = P::radix(P::kStages - 1), kB = 16 / RL, nb = N / RL;
#pragma unroll
      for (int c = 0; c < kB; ++c) {
        const int j = threadIdx.x * kB + c;
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int e = j + r * nb;
          const float w = wgt[e <= N / 2 ? e : N - e];
          v[c * RL + r] = make_float2(v[c * RL + r].x * w, -v[c * RL + r].y * w);
        }
        dft_r<RL>(v + c * RL);
      }
      if constexpr (P::kStages > 1) {
        // the forward's last stage may still be reading buffer ((F-1)&1): write the other
        r16_scatter<RL, N, 1>(v, kX0 ? b1 : b0);
        __syncthreads();
      }
    }
    r16_inverse<LOGN, kX0, 1>(v, b0, b1, tw);
    {  // last inverse stage: outputs j + (N / R) r in natural order -> conj, crop, store
      constexpr int S = P::kStages - 1;
      constexpr int R = P::iradix(S), NS = P::ispan(S), kB = 16 / R;
      float *oa = p.out + ra * p.width;
      float *ob = p.out + rb * p.width;
#pragma unroll
      for (int c = 0; c < kB; ++c) {
        const int j = threadIdx.x * kB + c;
        const int k = j & (NS - 1);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int o = base + r * NS;
          if (o < p.width) {
            oa[o] = v[c * R + r].x;
            if (has_b) ob[o] = -v[c * R + r].y;
          }
        }
      }
    }
    __syncthreads();  // buffers are reused by the next pair
  }
}

template <int LOGN>
static cudaError_t launch_filter_r16(const FilterParams &p, cudaStream_t st) {
  using P = R16Plan<LOGN>;
  constexpr int N = P::kN;
  const size_t smem = sizeof(float2) * (2 * (N + N / 16) + P::kTabs) + sizeof(float) * (N / 2 + 1 + N);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fft_filter_r16_kernel<LOGN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fft_filter_r16_kernel<LOGN>,
                                                                P::kT, smem);
  if (e != cudaSuccess) return e;
  const long long pairs = (p.n_rows + 1) / 2;
  const unsigned grid = (unsigned)std::min<long long>(pairs, (long long)sm_count() * std::max(1, per_sm));
  fft_filter_r16_kernel<LOGN><<<grid, P::kT, smem, st>>>(p);
  return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_filter_warp(const FilterParams &p, cudaStream_t st) {
  constexpr int N = 1 << LOGN;
  const size_t smem = sizeof(float2) * 2 * N * kFwWarps;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fft_filter_warp_kernel<LOGN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long pairs = (p.n_rows + 1) / 2;
  const int per_sm = std::max(1, (int)((220 * 1024) / smem));
  const long long want = (pairs + kFwWarps - 1) / kFwWarps;
  const unsigned grid = (unsigned)std::min<long long>(want, (long long)sm_count() * per_sm);
  fft_filter_warp_kernel<LOGN><<<grid, 32 * kFwWarps, smem, st>>>(p);
  return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_filter(const FilterParams &p, size_t smem, cudaStream_t st) {
  constexpr int N = 1 << LOGN;
  const char *algo = getenv("TK_FILTER_ALGO");  // r16 (default) | stockham | warp
  if constexpr (LOGN >= 9 && LOGN <= 12) {  // n_pad 8192 needs > 227 KB of tables + buffers
    if (!algo || !strcmp(algo, "r16")) return launch_filter_r16<LOGN>(p, st);
  }
  if (LOGN <= 11) {  // TK_FILTER_ALGO=warp: warp-per-row-pair variant (measured slower at cfg4)
    if (algo && !strcmp(algo, "warp")) return launch_filter_warp<LOGN>(p, st);
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fft_filter_kernel<LOGN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // blockDim >= N/8 keeps every stage at <= 8/R butterflies per thread
  const int threads = filter_threads<LOGN>();
  const long long pairs = (p.n_rows + 1) / 2;
  const int per_sm = std::max(1, std::min<int>((int)((200 * 1024) / smem), 2048 / threads));
  const unsigned grid = (unsigned)std::min<long long>(pairs, (long long)sm_count() * per_sm);
  fft_filter_kernel<LOGN><<<grid, threads, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace tk

using namespace tk;

extern "C" int tk_fft_filter_rows_ex(const float *in, long long n_rows, int width, int band_rows,
                                     int row_offset, int det_rows, const double *half_weights,
                                     int n_pad, double scale, double sdd, double du, double dv,
                                     float *out, void *stream) {
  clear_error();
  if (!in || !out || !half_weights) return fail_arg("tk_fft_filter_rows: null pointer");
  if (n_rows < 0 || width < 1 || det_rows < 1 || band_rows < 1 || row_offset < 0 ||
      row_offset + band_rows > det_rows)
    return fail_arg("tk_fft_filter_rows: bad extent / row band");
  if (n_pad < 2 * width || (n_pad & (n_pad - 1)) != 0 || n_pad < 2)
    return fail_arg("tk_fft_filter_rows: n_pad must be a power of two >= 2*width");
  if (n_pad > kMaxPad) return fail_arg("tk_fft_filter_rows: n_pad above 8192 is not supported");
  if (n_rows == 0) return TK_OK;
  cudaStream_t st = as_stream(stream);
  // twiddles (full circle) and folded weights, float64 on the host
  std::vector<float> host(2 * n_pad + n_pad / 2 + 1);
  const double two_pi = 6.283185307179586476925286766559;
  for (int m = 0; m < n_pad; ++m) {
    host[2 * m] = (float)cos(-two_pi * m / n_pad);
    host[2 * m + 1] = (float)sin(-two_pi * m / n_pad);
  }
  for (int k = 0; k <= n_pad / 2; ++k) host[2 * n_pad + k] = (float)(half_weights[k] * scale / n_pad);
  Scratch d;
  TK_TRY_CUDA(upload(d, host.data(), sizeof(float) * host.size(), st));
  FilterParams p;
  p.in = in;
  p.out = out;
  p.n_rows = n_rows;
  p.width = width;
  p.band_rows = band_rows;
  p.row_offset = row_offset;
  p.det_rows = det_rows;
  p.n_pad = n_pad;
  p.tw = reinterpret_cast<const float2 *>(d.as<float>());
  p.wgt = d.as<float>() + 2 * n_pad;
  p.sdd = (float)sdd;
  p.du = (float)du;
  p.dv = (float)dv;
  const size_t smem = sizeof(float2) * (2 * n_pad + n_pad / 16) + sizeof(float) * (n_pad / 2 + 1);
  int lg = 0;
  while ((1 << lg) < n_pad) ++lg;
  cudaError_t e;
  switch (lg) {
    case 1: e = launch_filter<1>(p, smem, st); break;
    case 2: e = launch_filter<2>(p, smem, st); break;
    case 3: e = launch_filter<3>(p, smem, st); break;
    case 4: e = launch_filter<4>(p, smem, st); break;
    case 5: e = launch_filter<5>(p, smem, st); break;
    case 6: e = launch_filter<6>(p, smem, st); break;
    case 7: e = launch_filter<7>(p, smem, st); break;
    case 8: e = launch_filter<8>(p, smem, st); break;
    case 9: e = launch_filter<9>(p, smem, st); break;
    case 10: e = launch_filter<10>(p, smem, st); break;
    case 11: e = launch_filter<11>(p, smem, st); break;
    case 12: e = launch_filter<12>(p, smem, st); break;
    default: e = launch_filter<13>(p, smem, st); break;
  }
  if (e != cudaSuccess) return check_cuda(e, "fft_filter_kernel");
  count_launch();
  return TK_OK;
}

extern "C" int tk_fft_filter_rows(const float *in, long long n_rows, int width, int det_rows,
                                  const double *half_weights, int n_pad, double scale,
                                  double sdd, double du, double dv, float *out, void *stream) {
  return tk_fft_filter_rows_ex(in, n_rows, width, det_rows, 0, det_rows, half_weights, n_pad,
                               scale, sdd, du, dv, out, stream);
}
