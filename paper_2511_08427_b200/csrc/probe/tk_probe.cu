// tk_probe.cu -- measured L1 load-path ceilings of the GPU the bench runs on
// (the roofline the gather kernels are reported against).  Built
// as its own library (libtkprobe.so), not part of the operator library:
//   ldg128: every quarter-warp reads one full 128-byte line per LDG.128 from an
//           L1-resident 32 KB buffer (best case for a vector gather);
//   lds32:  conflict-free LDS.32, one 128-byte wavefront per warp instruction.
// bench.py calls tkp_l1_peak() on the same lease right before its timed
// region; `python -m paper_2511_08427_b200.build` builds it next to libtkb200.so.
#include <cuda_runtime.h>

namespace {

constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) ldg128_kernel(const float4 *__restrict__ buf, float *out, unsigned mask) {
  // 2048 float4 = 32 KB per SM-resident working set; lane l of the warp reads
  // element (base + l): each quarter-warp covers one 128-byte line
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  unsigned idx = (threadIdx.x & ~31u) + (threadIdx.x & 31u);
#pragma unroll 8
  for (int i = 0; i < kIters; ++i) {
    const float4 v = __ldg(buf + (idx & mask));
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
    idx += 256;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[threadIdx.x] = acc.x;
}

__global__ void __launch_bounds__(256) lds32_kernel(float *out) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += 256) sm[i] = (float)i;
  __syncthreads();
  float acc = 0.f;
  unsigned idx = threadIdx.x;
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) {
    acc += sm[idx & 8191u];
    idx += 32 * 9;  // stays conflict-free: lanes hit 32 consecutive words
  }
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

}  // namespace

extern "C" {

// out[0] = LDG.128 GB/s, out[1] = LDS.32 GB/s, out[2] = SM count,
// out[3] = max SM clock (MHz, device attribute).  Returns a cudaError_t.
int tkp_l1_peak(double *out) {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max boost)
  float4 *buf = nullptr;
  float *o = nullptr;
  if (cudaMalloc(&buf, 2048 * sizeof(float4)) != cudaSuccess) return (int)cudaGetLastError();
  cudaMemset(buf, 0, 2048 * sizeof(float4));
  cudaMalloc(&o, 1024 * sizeof(float));
  const int blocks = sms * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best_ldg = 1e30f, best_lds = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    float ms;
    cudaEventRecord(a);
    ldg128_kernel<<<blocks, 256>>>(buf, o, 2047u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best_ldg = ms < best_ldg ? ms : best_ldg;
    cudaEventRecord(a);
    lds32_kernel<<<blocks, 256>>>(o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best_lds = ms < best_lds ? ms : best_lds;
  }
  const double ldg_bytes = (double)blocks * 256 * kIters * 16, lds_bytes = (double)blocks * 256 * kIters * 4;
  out[0] = ldg_bytes / (best_ldg * 1e-3) / 1e9;
  out[1] = lds_bytes / (best_lds * 1e-3) / 1e9;
  out[2] = sms;
  out[3] = clk / 1e3;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(o);
  return (int)cudaGetLastError();
}

}  // extern "C"
