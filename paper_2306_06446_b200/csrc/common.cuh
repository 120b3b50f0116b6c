// Shared helpers for the ShiftAddViT sm_100a kernels (C-ABI status handling,
// launch checks, small device utilities).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/shiftadd_b200.h"

namespace sa {

void set_error(const char* fmt, ...);
void count_launch(int n = 1);
// glue.cu: y[b*rows_per_img] = cls (+ pos[0]) for every image b
int write_cls_rows(const float* cls, const float* pos, float* y, int64_t B, int64_t rows_per_img,
                   int64_t d, cudaStream_t s);

#define SA_REQUIRE(cond, code, ...)        \
  do {                                     \
    if (!(cond)) {                         \
      ::sa::set_error(__VA_ARGS__);        \
      return (code);                       \
    }                                      \
  } while (0)

#define SA_LAUNCH_CHECK(what)                                                      \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      ::sa::set_error("%s: launch failed: %s", (what), cudaGetErrorString(_e));   \
      return SA_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

// Kernel-variant switches for A/B experiments. Only the debug library
// (libshiftadd_b200_debug.so, built with -DSA_DEBUG) has them as mutable state
// with an sa_debug_* setter; in the product library they are compile-time
// constants, so kernel selection depends on the call arguments alone.
#ifdef SA_DEBUG
#define SA_DEBUG_SWITCH(type, name, init, setter) \
  static type name = init;                        \
  extern "C" void setter(type v) { name = v; }
#else
#define SA_DEBUG_SWITCH(type, name, init, setter) static constexpr type name = init;
#endif

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Shift code byte (see include/shiftadd_b200.h): bit7 = sign, bits0-4 = P - p_min.
__device__ __forceinline__ float decode_shift(uint32_t byte, int p_min) {
  uint32_t sign = (byte >> 7) & 1u;
  int p = int(byte & 31u) + p_min;
  return __uint_as_float((sign << 31) | (uint32_t(p + 127) << 23));
}

// tanh-form GELU (ref tensor.py:149-152); plain float ops, no fast-math.
__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  float inner = c * (x + a * (x * x * x));
  return 0.5f * x * (1.0f + tanhf(inner));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace sa
