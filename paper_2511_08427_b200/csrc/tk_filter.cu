// tk_filter.cu -- FBP/FDK row filter on sm_100a: fused obliquity pre-weight,
// zero padding, FFT, real frequency weights, inverse FFT, crop and scale.
//
// Reference: /root/reference/pkg/src/tomokit/filters.py:136-171
// (fft_filter, cosine_preweight_cone, _preweight_fan).  Because the weights
// are real and even (weights[k] == weights[n_pad-k], filters.py:104-106), two
// real rows a, b are filtered with ONE complex transform of z = a + i b:
// IFFT(W * FFT(z)) = filt(a) + i filt(b).
//
// One CTA owns a row pair at a time (grid-stride); the n_pad-point transform
// runs in shared memory (radix-2, decimation in time forward on bit-reversed
// input, decimation in frequency inverse producing bit-reversed output, so no
// explicit permutation pass is needed).
#include <algorithm>
#include <cmath>
#include <vector>

#include "tk_common.cuh"

namespace tk {

constexpr int kMaxPad = 8192;

struct FilterParams {
  const float *in;
  float *out;
  long long n_rows;
  int width, band_rows, row_offset, det_rows, n_pad, log2n;
  const float2 *tw;    // exp(-2 pi i k / n_pad), k < n_pad/2
  const float *wgt;    // half weights * scale / n_pad, n_pad/2 + 1 entries
  float sdd, du, dv;   // obliquity pre-weight (disabled when sdd <= 0)
};

__device__ __forceinline__ unsigned bitrev(unsigned i, int bits) { return __brev(i) >> (32 - bits); }

__device__ __forceinline__ float preweight(const FilterParams &p, long long row, int i) {
  if (!(p.sdd > 0.f)) return 1.f;
  const int r = (int)(row % p.band_rows) + p.row_offset;
  const float u = ((float)i - 0.5f * (float)(p.width - 1)) * p.du;
  const float v = ((float)r - 0.5f * (float)(p.det_rows - 1)) * p.dv;
  return p.sdd / sqrtf(fmaf(p.sdd, p.sdd, fmaf(u, u, v * v)));
}

__global__ void __launch_bounds__(256) fft_filter_kernel(const FilterParams p) {
  extern __shared__ float smem[];
  const int N = p.n_pad;
  float2 *x = reinterpret_cast<float2 *>(smem);
  float2 *tw = x + N;
  float *wgt = reinterpret_cast<float *>(tw + N / 2);
  for (int i = threadIdx.x; i < N / 2; i += blockDim.x) tw[i] = p.tw[i];
  for (int i = threadIdx.x; i <= N / 2; i += blockDim.x) wgt[i] = p.wgt[i];
  const long long n_pairs = (p.n_rows + 1) / 2;
  for (long long pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
    const long long ra = 2 * pair, rb = ra + 1;
    const bool has_b = rb < p.n_rows;
    const float *ia = p.in + ra * p.width;
    const float *ib = p.in + rb * p.width;
    __syncthreads();  // previous pair's output reads complete before overwrite
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      float a = 0.f, b = 0.f;
      if (i < p.width) {
        a = __ldg(ia + i) * preweight(p, ra, i);
        if (has_b) b = __ldg(ib + i) * preweight(p, rb, i);
      }
      x[bitrev(i, p.log2n)] = make_float2(a, b);
    }
    // forward DIT
    for (int s = 1; s <= p.log2n; ++s) {
      __syncthreads();
      const int half = 1 << (s - 1);
      const int tstride = N >> s;
      for (int bI = threadIdx.x; bI < N / 2; bI += blockDim.x) {
        const int pos = bI & (half - 1);
        const int i0 = ((bI >> (s - 1)) << s) + pos;
        const int i1 = i0 + half;
        const float2 w = tw[pos * tstride];
        const float2 u = x[i0], v = x[i1];
        const float2 t = make_float2(w.x * v.x - w.y * v.y, w.x * v.y + w.y * v.x);
        x[i0] = make_float2(u.x + t.x, u.y + t.y);
        x[i1] = make_float2(u.x - t.x, u.y - t.y);
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const float w = wgt[k <= N / 2 ? k : N - k];
      const float2 v = x[k];
      x[k] = make_float2(v.x * w, v.y * w);
    }
    // inverse DIF with conjugate twiddles -> bit-reversed output
    for (int s = p.log2n; s >= 1; --s) {
      __syncthreads();
      const int half = 1 << (s - 1);
      const int tstride = N >> s;
      for (int bI = threadIdx.x; bI < N / 2; bI += blockDim.x) {
        const int pos = bI & (half - 1);
        const int i0 = ((bI >> (s - 1)) << s) + pos;
        const int i1 = i0 + half;
        const float2 w = tw[pos * tstride];
        const float2 u = x[i0], v = x[i1];
        const float2 d = make_float2(u.x - v.x, u.y - v.y);
        x[i0] = make_float2(u.x + v.x, u.y + v.y);
        x[i1] = make_float2(w.x * d.x + w.y * d.y, w.x * d.y - w.y * d.x);
      }
    }
    __syncthreads();
    float *oa = p.out + ra * p.width;
    float *ob = p.out + rb * p.width;
    for (int i = threadIdx.x; i < p.width; i += blockDim.x) {
      const float2 v = x[bitrev(i, p.log2n)];
      oa[i] = v.x;
      if (has_b) ob[i] = v.y;
    }
  }
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
  if (n_pad < 2 * width || (n_pad & (n_pad - 1)) != 0)
    return fail_arg("tk_fft_filter_rows: n_pad must be a power of two >= 2*width");
  if (n_pad > kMaxPad) return fail_arg("tk_fft_filter_rows: n_pad above 8192 is not supported");
  if (n_rows == 0) return TK_OK;
  cudaStream_t st = as_stream(stream);
  const int half = n_pad / 2;
  // twiddles and folded weights, float64 on the host
  std::vector<float> host(2 * half + half + 1);
  const double two_pi = 6.283185307179586476925286766559;
  for (int k = 0; k < half; ++k) {
    host[2 * k] = (float)cos(-two_pi * k / n_pad);
    host[2 * k + 1] = (float)sin(-two_pi * k / n_pad);
  }
  for (int k = 0; k <= half; ++k) host[2 * half + k] = (float)(half_weights[k] * scale / n_pad);
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
  int lg = 0;
  while ((1 << lg) < n_pad) ++lg;
  p.log2n = lg;
  p.tw = reinterpret_cast<const float2 *>(d.as<float>());
  p.wgt = d.as<float>() + 2 * half;
  p.sdd = (float)sdd;
  p.du = (float)du;
  p.dv = (float)dv;
  const size_t smem = sizeof(float2) * n_pad + sizeof(float2) * half + sizeof(float) * (half + 1);
  if (smem > 48 * 1024)
    TK_TRY_CUDA(cudaFuncSetAttribute(fft_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int threads = std::max(32, std::min(256, half));
  const long long pairs = (n_rows + 1) / 2;
  const int per_sm = std::max(1, (int)std::min<size_t>(8, (200 * 1024) / smem));
  const unsigned grid = (unsigned)std::min<long long>(pairs, (long long)sm_count() * per_sm);
  fft_filter_kernel<<<grid, threads, smem, st>>>(p);
  TK_LAUNCHED("fft_filter_kernel");
  return TK_OK;
}

extern "C" int tk_fft_filter_rows(const float *in, long long n_rows, int width, int det_rows,
                                  const double *half_weights, int n_pad, double scale,
                                  double sdd, double du, double dv, float *out, void *stream) {
  return tk_fft_filter_rows_ex(in, n_rows, width, det_rows, 0, det_rows, half_weights, n_pad,
                               scale, sdd, du, dv, out, stream);
}
