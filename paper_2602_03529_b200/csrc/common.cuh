// Shared device helpers for the semstream B200 codec path.
//
// Everything here reproduces numpy float64 semantics exactly: the library is
// compiled with -fmad=false so every a*b+c below is two separately rounded
// IEEE-754 operations, like numpy's ufunc loops in the reference.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/semstream_b200.h"

namespace sst {

constexpr int kGop = 9;        // video.py:12 GOP_SIZE
constexpr int kBlock = 8;      // codec.py:20 BLOCK
constexpr int kChannels = 12;  // codec.py:32 (3 colours x 4 zigzag coefficients)
constexpr int kHdr = 22;       // transport.py:44 ">HBBIHHBBff"

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// np.clip(x, 0.0, 1.0): comparisons only, so -0.0 passes through unchanged.
__device__ __forceinline__ double clip01(double x) {
  return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
}

__device__ __forceinline__ double clip_pm1(double x) {
  return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
}

// Total order used for row min/max: -0.0 sorts below +0.0.
__device__ __forceinline__ bool lt_total(double a, double b) {
  if (a == b) return __double_as_longlong(a) < 0 && __double_as_longlong(b) >= 0;
  return a < b;
}
__device__ __forceinline__ double min_total(double a, double b) { return lt_total(b, a) ? b : a; }
__device__ __forceinline__ double max_total(double a, double b) { return lt_total(a, b) ? b : a; }

__device__ __forceinline__ double warp_min_total(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min_total(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_total(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max_total(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// float64 -> float32 -> float64 (np.float32(x) then float()), round-to-nearest.
__device__ __forceinline__ double round_f32(double x) { return (double)__double2float_rn(x); }

// Big-endian stores into a byte buffer.
__device__ __forceinline__ void put_be16(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v >> 8); p[1] = (uint8_t)v;
}
__device__ __forceinline__ void put_be32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v >> 24); p[1] = (uint8_t)(v >> 16); p[2] = (uint8_t)(v >> 8); p[3] = (uint8_t)v;
}
__device__ __forceinline__ uint32_t get_be16(const uint8_t* p) {
  return ((uint32_t)p[0] << 8) | p[1];
}
__device__ __forceinline__ uint32_t get_be32(const uint8_t* p) {
  return ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
}

}  // namespace sst

#define SST_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return SST_ERR_CUDA;              \
  } while (0)

#define SST_LAUNCH_CHECK() SST_CUDA_TRY(cudaGetLastError())
