// Canonical CCCL TMA example (CUDA programming guide) + a plain bulk copy, to
// check that TMA works at all on the box.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda/barrier>
#include <cstdio>
#include <vector>
using barrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;

constexpr int H = 8, W = 32;

__global__ void ktensor(const __grid_constant__ CUtensorMap tensor_map, int x, int y, float *out) {
  __shared__ alignas(128) float smem_buffer[H][W];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  barrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_tensor_2d_global_to_shared(&smem_buffer, &tensor_map, x, y, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, sizeof(smem_buffer));
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < H * W; i += blockDim.x) out[i] = (&smem_buffer[0][0])[i];
}

__global__ void kbulk(const float *src, float *out) {
  __shared__ alignas(128) float buf[H * W];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  barrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_global_to_shared(buf, src, sizeof(buf), bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, sizeof(buf));
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < H * W; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int C = 64, R = 32;
  std::vector<float> h(C * R);
  for (int i = 0; i < C * R; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, H * W * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  kbulk<<<1, 128>>>(d, o);
  printf("bulk: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  void *f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  CUtensorMap map;
  cuuint64_t dims[2] = {C, R};
  cuuint64_t str[1] = {C * 4};
  cuuint32_t box[2] = {W, H}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  ktensor<<<1, 128>>>(map, -3, -2, o);
  printf("tensor negative coords: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  ktensor<<<1, 128>>>(map, 8, 4, o);
  printf("tensor: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> g(H * W);
  cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
  printf("g[0]=%g (want %g) g[last]=%g (want %g)\n", g[0], h[4 * C + 8], g[H * W - 1], h[(4 + H - 1) * C + 8 + W - 1]);
  return 0;
}
