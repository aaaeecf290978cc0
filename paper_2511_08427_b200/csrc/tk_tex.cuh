// tk_tex.cuh -- pooled CUDA arrays + texture objects for the gather kernels.
//
// Volumes / sinograms are copied (stream-ordered, device to device) into
// block-linear layered CUDA arrays so the texture path can fetch 2x2 tap
// quads with one TLD4 (tld4.a2d) and zero-border addressing.  Arrays are
// large and slow to allocate, so they are pooled per (device, extent, mode):
// a slot is handed to one caller at a time, and a CUDA event recorded after
// the consuming kernel orders the next user's copy behind it, whichever stream
// that user runs on.  tk_release_cached_memory() frees every idle slot.
#pragma once

#include <cuda_runtime.h>

namespace tk {

enum class TexKind { kLayeredPoint = 0, kLayeredLinear = 1, kVolumeLinear = 2 };

struct TexLease {
  cudaTextureObject_t tex = 0;
  void *slot = nullptr;
};

// Copy `src` (device, C-order [layers][h][w] fp32) into a pooled array and
// return its texture object.  Returns a cudaError_t.
cudaError_t tex_acquire(const float *src, int w, int h, int layers, TexKind kind,
                        cudaStream_t st, TexLease &out);
// Hand the slot back; work already enqueued on `st` keeps using it safely.
void tex_release(TexLease &lease, cudaStream_t st);

// tld4.a2d gather of the 2x2 quad whose lower-left texel is (x0, y0) of layer
// `layer`: returns (T[y0+1][x0], T[y0+1][x0+1], T[y0][x0+1], T[y0][x0]) --
// the D3D/CUDA gather order -- with zero outside the layer (border mode).
__device__ __forceinline__ float4 gather_a2d(cudaTextureObject_t t, int layer, float x_center,
                                             float y_center) {
  float4 r;
  asm("tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %7}];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(t), "r"(layer), "f"(x_center), "f"(y_center));
  return r;
}

}  // namespace tk
