// tk_artifacts.cu -- sinogram degradation simulators on the GPU (SURVEY 8f,
// reference artifacts.py:50-211): detector jitter, Poisson and Gaussian noise,
// ring artifacts, gantry motion blur.  Elementwise / small-stencil HBM-bound
// work: one thread per output texel, grid-stride, coalesced along u.
//
// Randomness: a counter-based Philox4x32-10 stream keyed by (seed, view) and
// indexed by the texel, so every projection has its own stream and results do
// not depend on launch configuration or evaluation order -- the property the
// reference gets from SeedSequence(seed).spawn(n_views) (artifacts.py:28-31).
// As in the reference, cross-implementation bit-equality of the noise is not
// a goal; the distributions are the contract (artifacts.py:5-7).
#include <algorithm>
#include <cmath>
#include <vector>

#include "tk_common.cuh"

namespace tk {

// ---- Philox4x32-10 ------------------------------------------------------------
struct U4 {
  unsigned x, y, z, w;
};

__host__ __device__ inline void mulhilo(unsigned a, unsigned b, unsigned &hi, unsigned &lo) {
  const unsigned long long p = (unsigned long long)a * b;
  hi = (unsigned)(p >> 32);
  lo = (unsigned)p;
}

__host__ __device__ inline U4 philox(U4 c, unsigned k0, unsigned k1) {
  for (int r = 0; r < 10; ++r) {
    unsigned h0, l0, h1, l1;
    mulhilo(0xD2511F53u, c.x, h0, l0);
    mulhilo(0xCD9E8D57u, c.z, h1, l1);
    c = U4{h1 ^ c.y ^ k0, l1, h0 ^ c.w ^ k1, l0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// uniform in (0, 1) with 53 random bits from two 32-bit words
__host__ __device__ inline double u01(unsigned a, unsigned b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 0.5) * (1.0 / 9007199254740992.0);
}

// per-(seed, view) key; counter = (texel, draw index)
struct Stream {
  unsigned k0, k1;
  unsigned long long texel;
  unsigned draw = 0;
  U4 buf{};
  int left = 0;
  __host__ __device__ Stream(unsigned long long seed, unsigned view, unsigned long long t)
      : k0((unsigned)seed ^ (view * 0x85EBCA6Bu)), k1((unsigned)(seed >> 32) ^ 0xC2B2AE35u ^ view), texel(t) {}
  __host__ __device__ double uniform() {
    if (left == 0) {
      buf = philox(U4{(unsigned)texel, (unsigned)(texel >> 32), draw++, 0x5EEDu}, k0, k1);
      left = 2;
    }
    const double u = left == 2 ? u01(buf.x, buf.y) : u01(buf.z, buf.w);
    --left;
    return u;
  }
  __host__ __device__ double normal() {  // Box-Muller (one of the pair)
    const double a = uniform(), b = uniform();
    return sqrt(-2.0 * log(a)) * cos(6.283185307179586 * b);
  }
};

// Poisson(lam): multiplication method below 10, else PTRS (Hormann 1993, the
// transformed-rejection sampler numpy uses for lam >= 10).
__device__ double poisson(Stream &s, double lam) {
  if (!(lam > 0.0)) return 0.0;
  if (lam < 10.0) {
    const double enlam = exp(-lam);
    double prod = 1.0;
    long long x = 0;
    for (;;) {
      prod *= s.uniform();
      if (prod <= enlam) return (double)x;
      ++x;
    }
  }
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    const double U = s.uniform() - 0.5, V = s.uniform();
    const double us = 0.5 - fabs(U);
    const double k = floor((2.0 * a / us + b) * U + lam + 0.43);
    if (us >= 0.07 && V <= vr) return k;
    if (k < 0.0 || (us < 0.013 && V > us)) continue;
    if (log(V) + log(invalpha) - log(a / (us * us) + b) <= -lam + k * loglam - lgamma(k + 1.0)) return k;
  }
}

// one uniform integer in [-m, m] per (seed, view): the jitter offset
__host__ __device__ inline int jitter_shift(unsigned long long seed, unsigned view, int m) {
  Stream s(seed, view, 0xFFFFFFFFFFFFull);
  const int k = (int)floor(s.uniform() * (2 * m + 1));
  return (k > 2 * m ? 2 * m : k) - m;
}

// ---- kernels -------------------------------------------------------------------
__global__ void jitter_kernel(const float *__restrict__ in, float *__restrict__ out, int n_views, int rows, int cols,
                              int axis_v, int m, unsigned long long seed) {
  const long long per = (long long)rows * cols, n = per * n_views;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i / per);
    const int rem = (int)(i - (long long)v * per);
    const int r = rem / cols, c = rem - r * cols;
    const int sh = jitter_shift(seed, (unsigned)v, m);
    // out[r][c] = in[r][c - sh] along u (or in[r - sh][c] along v), zero where vacated
    const int sr = axis_v ? r - sh : r, sc = axis_v ? c : c - sh;
    out[i] = ((unsigned)sr < (unsigned)rows && (unsigned)sc < (unsigned)cols)
                 ? __ldg(in + (long long)v * per + (long long)sr * cols + sc)
                 : 0.f;
  }
}

__global__ void poisson_kernel(const float *__restrict__ in, float *__restrict__ out, int n_views, long long per,
                               double i0, int transmission, unsigned long long seed) {
  const long long n = per * n_views;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i / per);
    Stream s(seed, (unsigned)v, (unsigned long long)(i - (long long)v * per));
    const double p = (double)__ldg(in + i);
    if (transmission) {
      const double counts = fmax(poisson(s, i0 * exp(-p)), 1.0);  // artifacts.py:83-86
      out[i] = (float)(-log(counts / i0));
    } else {
      out[i] = (float)poisson(s, p);
    }
  }
}

__global__ void gaussian_kernel(const float *__restrict__ in, float *__restrict__ out, int n_views, long long per,
                                double mean, double std, unsigned long long seed) {
  const long long n = per * n_views;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i / per);
    Stream s(seed, (unsigned)v, (unsigned long long)(i - (long long)v * per));
    const double z = std > 0.0 ? std * s.normal() : 0.0;
    out[i] = (float)((double)__ldg(in + i) + mean + z);
  }
}

// colmask[c] = 1 for selected detector columns; views [start, end)
__global__ void ring_kernel(const float *__restrict__ in, float *__restrict__ out, int n_views, int rows, int cols,
                            const unsigned char *__restrict__ colmask, int start, int end, int zero, float factor) {
  const long long n = (long long)n_views * rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cols);
    const int v = (int)(i / ((long long)rows * cols));
    float x = __ldg(in + i);
    if (v >= start && v < end && colmask[c]) x = zero ? 0.f : x * factor;
    out[i] = x;
  }
}

// zero-padded 2D correlation with a per-view (2h+1)^2 kernel (ndimage.convolve
// with a kernel that is used flipped: out[r][c] = sum k[h+a][h+b] in[r-a][c-b])
__global__ void blur_kernel(const float *__restrict__ in, float *__restrict__ out, int n_views, int rows, int cols,
                            const float *__restrict__ kern, int h) {
  const int K = 2 * h + 1;
  const long long per = (long long)rows * cols, n = per * n_views;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i / per);
    const int rem = (int)(i - (long long)v * per);
    const int r = rem / cols, c = rem - r * cols;
    const float *kv = kern + (long long)v * K * K;
    const float *iv = in + (long long)v * per;
    double acc = 0.0;
    for (int a = -h; a <= h; ++a) {
      const int rr = r - a;
      if ((unsigned)rr >= (unsigned)rows) continue;
      for (int b = -h; b <= h; ++b) {
        const float w = __ldg(kv + (a + h) * K + (b + h));
        const int cc = c - b;
        if (w != 0.f && (unsigned)cc < (unsigned)cols) acc += (double)w * (double)__ldg(iv + (long long)rr * cols + cc);
      }
    }
    out[i] = (float)acc;
  }
}

static unsigned grid_for(long long n) { return (unsigned)std::min<long long>(ceil_div(n, 256), (long long)sm_count() * 32); }

}  // namespace tk

using namespace tk;

extern "C" {

int tk_jitter_shifts(unsigned long long seed, int n_views, int max_shift, int *shifts_out) {
  clear_error();
  if (!shifts_out || n_views < 0 || max_shift < 0) return fail_arg("tk_jitter_shifts: invalid argument");
  for (int v = 0; v < n_views; ++v) shifts_out[v] = jitter_shift(seed, (unsigned)v, max_shift);
  return TK_OK;
}

int tk_detector_jitter(const float *sino, int n_views, int rows, int cols, int axis_v, int max_shift,
                       unsigned long long seed, float *out, void *stream) {
  clear_error();
  if (!sino || !out) return fail_arg("tk_detector_jitter: null pointer");
  if (n_views < 0 || rows < 1 || cols < 1 || max_shift < 0) return fail_arg("tk_detector_jitter: invalid extent");
  const long long n = (long long)n_views * rows * cols;
  if (n == 0) return TK_OK;
  jitter_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(sino, out, n_views, rows, cols, axis_v, max_shift, seed);
  TK_LAUNCHED("jitter_kernel");
  return TK_OK;
}

int tk_poisson_noise(const float *sino, int n_views, long long view_size, double i0, int transmission,
                     unsigned long long seed, float *out, void *stream) {
  clear_error();
  if (!sino || !out) return fail_arg("tk_poisson_noise: null pointer");
  if (n_views < 0 || view_size < 1 || !(i0 > 0)) return fail_arg("tk_poisson_noise: invalid argument");
  const long long n = view_size * n_views;
  if (n == 0) return TK_OK;
  poisson_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(sino, out, n_views, view_size, i0, transmission, seed);
  TK_LAUNCHED("poisson_kernel");
  return TK_OK;
}

int tk_gaussian_noise(const float *sino, int n_views, long long view_size, double mean, double std,
                      unsigned long long seed, float *out, void *stream) {
  clear_error();
  if (!sino || !out) return fail_arg("tk_gaussian_noise: null pointer");
  if (n_views < 0 || view_size < 1 || !(std >= 0)) return fail_arg("tk_gaussian_noise: invalid argument");
  const long long n = view_size * n_views;
  if (n == 0) return TK_OK;
  gaussian_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(sino, out, n_views, view_size, mean, std, seed);
  TK_LAUNCHED("gaussian_kernel");
  return TK_OK;
}

int tk_ring_artifact(const float *sino, int n_views, int rows, int cols, const int *columns, int n_columns, int start,
                     int end, int zero, double factor, float *out, void *stream) {
  clear_error();
  if (!sino || !out || (n_columns > 0 && !columns)) return fail_arg("tk_ring_artifact: null pointer");
  if (n_views < 0 || rows < 1 || cols < 1 || start < 0 || end < start || end > n_views)
    return fail_arg("tk_ring_artifact: invalid extent");
  std::vector<unsigned char> mask(cols, 0);
  for (int i = 0; i < n_columns; ++i) {
    if (columns[i] < 0 || columns[i] >= cols) return fail_arg("tk_ring_artifact: column outside the detector");
    mask[columns[i]] = 1;
  }
  const long long n = (long long)n_views * rows * cols;
  if (n == 0) return TK_OK;
  cudaStream_t st = as_stream(stream);
  Scratch dmask;
  TK_TRY_CUDA(upload(dmask, mask.data(), mask.size(), st));
  ring_kernel<<<grid_for(n), 256, 0, st>>>(sino, out, n_views, rows, cols, dmask.as<unsigned char>(), start, end,
                                            zero, (float)factor);
  TK_LAUNCHED("ring_kernel");
  return TK_OK;
}

int tk_gantry_blur(const float *sino, int n_views, int rows, int cols, const double *kernels, int half,
                   float *out, void *stream) {
  clear_error();
  if (!sino || !out || !kernels) return fail_arg("tk_gantry_blur: null pointer");
  if (n_views < 0 || rows < 1 || cols < 1 || half < 0 || half > 64) return fail_arg("tk_gantry_blur: invalid extent");
  const long long n = (long long)n_views * rows * cols;
  if (n == 0) return TK_OK;
  const int K = 2 * half + 1;
  std::vector<float> k32((size_t)n_views * K * K);
  for (size_t i = 0; i < k32.size(); ++i) k32[i] = (float)kernels[i];
  cudaStream_t st = as_stream(stream);
  Scratch dk;
  TK_TRY_CUDA(upload(dk, k32.data(), sizeof(float) * k32.size(), st));
  blur_kernel<<<grid_for(n), 256, 0, st>>>(sino, out, n_views, rows, cols, dk.as<float>(), half);
  TK_LAUNCHED("blur_kernel");
  return TK_OK;
}

}  // extern "C"
