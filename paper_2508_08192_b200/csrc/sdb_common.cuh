// Shared device helpers for the specdec_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/specdec_b200.h"

#define SDB_FULL_MASK 0xffffffffu

namespace sdb {

// Records the last launch error for sdb_last_cuda_error(); returns SDB_E_CUDA.
int record_cuda_error(cudaError_t e);

#define SDB_CHECK_LAUNCH()                                  \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return ::sdb::record_cuda_error(_e); \
  } while (0)

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(SDB_FULL_MASK, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(SDB_FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(SDB_FULL_MASK, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(SDB_FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ long long warp_max_i64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long w = __shfl_xor_sync(SDB_FULL_MASK, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Monotone map float -> uint32 (larger float -> larger key; -0 < +0 is fine:
// the reference argmax treats -0 == +0 but ties break on the lowest index and
// a -0/+0 pair is a tie there; we order -0 below +0, see argmax_key note).
__device__ __forceinline__ uint32_t orderable_u32(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Packed argmax key, signed-int64 comparable: high word = orderable value
// shifted into signed range, low word = 0xFFFFFFFF - index (lowest index wins
// ties under MAX).
__device__ __forceinline__ long long argmax_key(float v, uint32_t idx) {
  // canonicalise -0.0 to +0.0 so that numpy's argmax tie semantics hold
  if (v == 0.0f) v = 0.0f;
  int32_t hi = (int32_t)(orderable_u32(v) ^ 0x80000000u);
  return (long long)(((unsigned long long)(uint32_t)hi << 32) | (unsigned long long)(0xFFFFFFFFu - idx));
}
__device__ __forceinline__ uint32_t key_index(long long key) {
  return 0xFFFFFFFFu - (uint32_t)((unsigned long long)key & 0xFFFFFFFFull);
}

template <typename T> __device__ __forceinline__ float to_f32(T x);
template <> __device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__host__ __device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

}  // namespace sdb
