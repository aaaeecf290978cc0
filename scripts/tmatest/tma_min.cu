// Minimal TMA load test: copies a (bw x bh) box at (c0, r0, v) into smem and back.
// argv[1] bit mask: 1 = descriptor in global memory (pointer param), 2 = L2 promotion none,
// 4 = 2D map over a single view, 8 = no fence.mbarrier_init, 16 = box inner 32 floats, 32 = in-bounds box
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap *gmap, int bw, int bh, int c0, int r0,
                  int v, float *out, int mode) {
  extern __shared__ float raw[];
  float *tile = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    if (!(mode & 8)) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t desc = (mode & 1) ? reinterpret_cast<uint64_t>(gmap) : reinterpret_cast<uint64_t>(&map);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bw * bh * 4) : "memory");
    if (mode & 4)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(tile)), "l"(desc), "r"(c0), "r"(r0), "r"(su32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(su32(tile)), "l"(desc), "r"(c0), "r"(r0), "r"(v), "r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = tile[i];
}

int main(int argc, char **argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int C = 48, R = 40, V = 5, bh = 12;
  const int c0 = (mode & 32) ? 3 : -3, r0 = (mode & 32) ? 3 : 30;
  const int bw = (mode & 16) ? 32 : 20;
  const int v = (mode & 4) ? 0 : 2;
  std::vector<float> h(C * R * V);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  CUtensorMap *gm;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, bw * bh * 4);
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void *f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  printf("entry point %d q %d f %p\n", (int)ge, (int)q, f);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  alignas(64) CUtensorMap map;
  cuuint64_t dims[3] = {C, R, V};
  cuuint64_t str[2] = {C * 4, (cuuint64_t)C * R * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, bh, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (mode & 4) ? 2 : 3, d, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   (mode & 2) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
  printf("mode %d encode %d\n", mode, (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(map, gm, bw, bh, c0, r0, v, o, mode);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> g(bw * bh);
  cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < bh; ++y)
    for (int x = 0; x < bw; ++x) {
      int c = c0 + x, rr = r0 + y;
      float want = (c >= 0 && c < C && rr >= 0 && rr < R) ? h[((size_t)v * R + rr) * C + c] : 0.f;
      if (g[y * bw + x] != want) ++bad;
    }
  printf("mismatches %d\n", bad);
  return 0;
}
