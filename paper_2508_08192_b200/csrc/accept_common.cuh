// Shared pieces of the acceptance kernels (accept.cu, accept_sharded.cu):
// block reductions and the per-row softmax / nucleus statistics.
#pragma once

#include <limits.h>
#include <math.h>

#include "sdb_common.cuh"

namespace sdb {

// ---------------------------------------------------------------------------
// block reductions
// ---------------------------------------------------------------------------
template <int kThreads>
__device__ __forceinline__ float block_max(float v, float *red) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kThreads / 32 ? red[lane] : -INFINITY;
    v = warp_max(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double *red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kThreads / 32 ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

template <int kThreads>
__device__ __forceinline__ long long block_max_i64(long long v, long long *red) {
  v = warp_max_i64(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kThreads / 32 ? red[lane] : LLONG_MIN;
    v = warp_max_i64(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// ---------------------------------------------------------------------------
// per-row statistics of target_dist (sampling.py:87-102): softmax of
// logit * a (a = log2(e) / T) with the top-p nucleus as a (key, index) cut
// ---------------------------------------------------------------------------
struct RowStats {
  float m2;        // max of logit * a (a = log2(e) / T)
  float log2_z;    // log2 of the normaliser of kept mass (S, or Z for nucleus rows)
  double s;        // sum of exp2(x2 - m2) over the row
  double z;        // kept mass (== s when the whole row is kept)
  uint32_t cut_key;
  int32_t cut_idx;
  int32_t keep_all;
  int32_t valid;
};

// Probability order key: the fp32 logit order with -0 == +0 (equal
// probabilities tie on the index in the reference's lexsort, sampling.py:57-72).
__device__ __forceinline__ uint32_t prob_key(float l) { return orderable_u32(l == 0.0f ? 0.0f : l); }

__device__ __forceinline__ bool kept(const RowStats &st, float l, int idx) {
  if (st.keep_all) return true;
  uint32_t k = prob_key(l);
  return k > st.cut_key || (k == st.cut_key && idx <= st.cut_idx);
}

// Bulk prefetch of [p, p + bytes) into L2 (TMA engine; one thread issues it).
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- packed fp32x2 math (FFMA2 / FADD2 / FMUL2) and MUFU ex2 ----------------
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2splat(float a) { return f2pack(a, a); }
// 2^x on the MUFU (flush-to-zero below 2^-126: those weights are 0 for
// every decision here)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// max over three values propagating NaN (sm_100 3-input FMNMX)
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

}  // namespace sdb
