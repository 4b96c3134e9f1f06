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

__device__ __forceinline__ bool kept(const RowStats &st, float l, int idx) {
  if (st.keep_all) return true;
  uint32_t k = orderable_u32(l);
  return k > st.cut_key || (k == st.cut_key && idx <= st.cut_idx);
}

// Bulk prefetch of [p, p + bytes) into L2 (TMA engine; one thread issues it).
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace sdb
