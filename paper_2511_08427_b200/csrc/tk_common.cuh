// tk_common.cuh -- shared helpers for the sm_100a CT-operator kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/tk_b200.h"

namespace tk {

// Reference constant _TINY (_kernels.py:24).
constexpr double kTiny = 1e-12;

// ---- error plumbing (thread-local message, int status) ----------------------
void set_error(const std::string &msg);
void clear_error();
int fail_arg(const std::string &msg);
int check_cuda(cudaError_t e, const char *what);
void count_launch(unsigned n = 1);

#define TK_TRY_CUDA(expr)                                  \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return ::tk::check_cuda(_e, #expr); \
  } while (0)

// Check the last launch and count it.
#define TK_LAUNCHED(name)                                         \
  do {                                                            \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return ::tk::check_cuda(_e, name);     \
    ::tk::count_launch();                                         \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync).
struct Scratch {
  void *ptr = nullptr;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(const Scratch &) = delete;
  Scratch &operator=(const Scratch &) = delete;
  cudaError_t alloc(size_t bytes, cudaStream_t s);
  ~Scratch();
  template <class T> T *as() const { return reinterpret_cast<T *>(ptr); }
};

// Upload a host array to fresh stream-ordered scratch.
cudaError_t upload(Scratch &dst, const void *host, size_t bytes, cudaStream_t s);

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

int sm_count();

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ float lerpf(float a, float b, float w) { return fmaf(w, b - a, a); }

// floor() without the conversion pipe (FRND / F2I are quarter rate): for
// |x| < 2^22, x + 1.5 * 2^23 rounded toward -inf is exactly 1.5 * 2^23 + floor(x),
// so the sum's bit pattern is kFloorBits + floor(x) (an integer, usable in
// index arithmetic modulo 2^32) and sum - kFloorMagic is floor(x) as a float.
constexpr float kFloorMagic = 12582912.f;
constexpr unsigned kFloorBits = 0x4B400000u;
__device__ __forceinline__ float floor_magic(float x) { return __fadd_rd(x, kFloorMagic); }

// base + idx elements as ONE IMAD.WIDE.U32 (keeps the compiler from re-forming
// 64-bit (outer * stride + idx) << log2(size) chains per gather).
template <class T>
__device__ __forceinline__ const T *elem_ptr(const T *base, unsigned idx) {
  const T *r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "n"((int)sizeof(T)), "l"(base));
  return r;
}

// Packed fp32 pairs (sm_100a FFMA2 / FADD2: two fp32 FMAs / adds per
// instruction, operand-selectable halves and broadcast scalars).
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2_rm(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 16-byte vector reduction into global memory (REDG.E.ADD.F32x4): one L2 atomic
// operation for four fp32 adds.
__device__ __forceinline__ void red_add_v4(float4 *p, const float4 &v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

}  // namespace tk
