// tk_abi.cu -- error handling, scratch memory and small helpers behind the C ABI.
#include <cstdio>
#include <mutex>

#include "tk_common.cuh"

namespace tk {

static thread_local std::string g_error;
static std::atomic<unsigned long long> g_launches{0};

void set_error(const std::string &msg) { g_error = msg; }
void clear_error() { g_error.clear(); }
int fail_arg(const std::string &msg) {
  g_error = "invalid argument: " + msg;
  return TK_ERR_ARG;
}
int check_cuda(cudaError_t e, const char *what) {
  g_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorName(e) + " (" +
            cudaGetErrorString(e) + ")";
  return TK_ERR_CUDA;
}
void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::once_flag g_pool_once;

static void configure_pool() {
  // Keep freed stream-ordered scratch cached in the device pool instead of
  // returning it to the OS at every synchronisation point.
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t thresh = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
}

cudaError_t Scratch::alloc(size_t bytes, cudaStream_t s) {
  std::call_once(g_pool_once, configure_pool);
  stream = s;
  if (bytes == 0) bytes = 16;
  return cudaMallocAsync(&ptr, bytes, s);
}

Scratch::~Scratch() {
  if (ptr) cudaFreeAsync(ptr, stream);
}

cudaError_t upload(Scratch &dst, const void *host, size_t bytes, cudaStream_t s) {
  cudaError_t e = dst.alloc(bytes, s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(dst.ptr, host, bytes, cudaMemcpyHostToDevice, s);
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}

__global__ void scale_kernel(const float *__restrict__ in, long long n, float s,
                             float *__restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i] * s;
}

}  // namespace tk

extern "C" {

int tk_version(void) { return 1 * 10000 + 1 * 100 + 0; }

const char *tk_last_error(void) { return tk::g_error.c_str(); }

unsigned long long tk_launch_count(void) {
  return tk::g_launches.load(std::memory_order_relaxed);
}

int tk_device_info(int *sm_major, int *sm_minor, int *sm_count) {
  tk::clear_error();
  int dev = 0;
  TK_TRY_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  TK_TRY_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (sm_major) *sm_major = prop.major;
  if (sm_minor) *sm_minor = prop.minor;
  if (sm_count) *sm_count = prop.multiProcessorCount;
  return TK_OK;
}

int tk_scale(const float *in, long long n, double scale, float *out, void *stream) {
  tk::clear_error();
  if (n < 0 || (n > 0 && (!in || !out))) return tk::fail_arg("tk_scale: bad buffer");
  if (n == 0) return TK_OK;
  unsigned grid = (unsigned)std::min<long long>(tk::ceil_div(n, 256), 148LL * 16);
  tk::scale_kernel<<<grid, 256, 0, tk::as_stream(stream)>>>(in, n, (float)scale, out);
  TK_LAUNCHED("scale_kernel");
  return TK_OK;
}

}  // extern "C"
