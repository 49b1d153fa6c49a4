// ckv_common.cuh — shared device helpers for the sm_100a ClusterKV kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include <cuda_fp16.h>

#include "ckv_cuda.h"

namespace ckvb {

constexpr int D = CKV_HEAD_DIM;  // 128, the only head dim the kernels specialise

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, status codes of ckv_cuda.h)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* where);

#define CKV_CUDA_TRY(expr)                                         \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return ::ckvb::cuda_status(_e, #expr);  \
  } while (0)

#define CKV_LAUNCH_CHECK(name)                                       \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::ckvb::cuda_status(_e, name);     \
  } while (0)

#define CKV_TRY(expr)          \
  do {                         \
    int _rc = (expr);          \
    if (_rc != CKV_OK) return _rc; \
  } while (0)

// ---------------------------------------------------------------------------
// numerics shared with the reference contract:
// float x float is exact in double, so a sequential FMA chain in index order
// reproduces dot_f64 (common.hpp:86-90) bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
  return __uint_as_float(uint32_t(b) << 16);
}

// f32 -> the fp16 tensor-core operand (ckv_assign_tc.cu): round to nearest
// even, saturated to +-65504, results below the normal range (|h| < 2^-14)
// flushed to signed zero so no subnormal reaches the tensor cores.  Callers
// measure |x - f16_to_f32(h)| themselves: that is the error the band carries.
__device__ __forceinline__ uint16_t f32_to_f16_tc(float f) {
  f = fminf(fmaxf(f, -65504.f), 65504.f);
  uint16_t b = __half_as_ushort(__float2half_rn(f));
  if ((b & 0x7c00u) == 0u) b &= 0x8000u;
  return b;
}
__device__ __forceinline__ float f16_to_f32(uint16_t b) {
  return __half2float(__ushort_as_half(b));
}

__device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7f800000u) == 0x7f800000u) return uint16_t((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  uint32_t r = ((u >> 16) & 1u) + 0x7fffu;
  return uint16_t((u + r) >> 16);
}

// sequential f64 dot of two f32 vectors of length D (strides in elements)
__device__ __forceinline__ double dot_seq_ff(const float* __restrict__ a,
                                             const float* __restrict__ b) {
  double s = 0.0;
#pragma unroll 16
  for (int j = 0; j < D; ++j) s = __fma_rn(double(a[j]), double(b[j]), s);
  return s;
}

// sequential f64 dot: bf16 row (as uint16 bits) with f32 vector
__device__ __forceinline__ double dot_seq_bf(const uint16_t* __restrict__ a,
                                             const float* __restrict__ b) {
  double s = 0.0;
#pragma unroll 16
  for (int j = 0; j < D; ++j) s = __fma_rn(double(bf16_to_f32(a[j])), double(b[j]), s);
  return s;
}

__device__ __forceinline__ double dot_seq_bb(const uint16_t* __restrict__ a,
                                             const uint16_t* __restrict__ b) {
  double s = 0.0;
#pragma unroll 16
  for (int j = 0; j < D; ++j)
    s = __fma_rn(double(bf16_to_f32(a[j])), double(bf16_to_f32(b[j])), s);
  return s;
}

// order-preserving map of a double to u64 (larger double -> larger key)
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long u = __double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// argmax over (score desc, id asc) across a warp; returns winner in all lanes
__device__ __forceinline__ void warp_argmax_d(double& s, uint32_t& id) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double os = __shfl_xor_sync(0xffffffffu, s, o);
    uint32_t oi = __shfl_xor_sync(0xffffffffu, id, o);
    if (os > s || (os == s && oi < id)) { s = os; id = oi; }
  }
}

// host helpers
int num_sms();

}  // namespace ckvb
