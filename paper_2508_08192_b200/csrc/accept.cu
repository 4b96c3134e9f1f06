// K4/K5: acceptance of the drafted tree against the target logits.
//
// Greedy (temperature 0).  target_dist(row, 0, .) is a one-hot at the row
// argmax (numcore.py:51-55) and mss_verify then reduces exactly to the
// argmax walk (pinned by tests/golden/accept_greedy):
// accept the first child (priority = index order) whose token equals the
// argmax of its parent's row, bonus = argmax of the stop row.  Split into a
// vocab-shardable packed-key argmax (one int64 MAX all-reduce combines
// shards) and the walk.
//
// Stochastic (temperature > 0).  Phase A computes, for every target row, the
// softmax normaliser and the exact top-p nucleus cut (sampling.py:52-72) as a
// (key, index) threshold -- a value histogram locates the cut, the few
// elements around it are sorted exactly -- and for every draft parent row
// the softmax normaliser.  Phase B walks the tree (sampling.py:173-202); a
// rejection's residual norm(max(p - q, 0)) is kept in closed form
// p_k = max(P - c_k Q, 0) / M_k (siblings share their parent's q,
// engine.py:405-407), so each rejection costs one block-wide pass over the
// vocab and the bonus draw one inverse-CDF pass.
#include <float.h>

#include <algorithm>
#include <math.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include "accept_common.cuh"

namespace cg = cooperative_groups;

namespace sdb {


// ---------------------------------------------------------------------------
// greedy: packed argmax keys
// ---------------------------------------------------------------------------
constexpr int kArgmaxThreads = 1024;  // one row per CTA: 2048 rows at C3 = 6.9 waves of 296 CTAs (small tail)

__device__ __forceinline__ float max_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ float max_nan3(float a, float b, float c) {
  return max_nan(max_nan(a, b), c);
}

// Row argmax.  The streaming loop tracks, per thread, the maximum of each
// 16-byte chunk and the first chunk where the thread's running maximum was
// reached (strict >, so the earliest chunk wins ties); NaN propagates into a
// separate max.NaN accumulator.  ~1.5 instructions per fp32 element instead
// of a packed 64-bit key per element.  The winning chunk is re-read once to
// pick the first element equal to the maximum, and only then packed into the
// (value, lowest index) key of the cross-thread reduction.
// streaming load of the greedy scan (SDB_ARGMAX_LD: 0 ld.global.cs, 1 ld.global.nc, 2 ld.global.cg).
// ncu at C3 (1.05 GB of logits): DRAM read 1.23 GB with .cs (evict-first),
// 1.16 GB with .nc, 1.15 GB with .cg at the same kernel time; step 630 ->
// 609 us on one box
#ifndef SDB_ARGMAX_LD
#define SDB_ARGMAX_LD 2
#endif
template <typename V>
__device__ __forceinline__ V scan_ld(const V *p) {
#if SDB_ARGMAX_LD == 1
  return __ldg(p);
#elif SDB_ARGMAX_LD == 2
  return __ldcg(p);
#else
  return __ldcs(p);
#endif
}

// fp32 rows, SDB_ARGMAX_STAGES > 0: each thread streams its 16-byte elements
// through a private ring of shared-memory slots filled by cp.async (no
// register destination: 2 CTAs x 1024 threads keep STAGES x 32 KB in flight
// per SM).  Measured at C3 (tools/cycles/r2_argmax_cpasync.sh): the scan
// alone 164 us with 6 stages vs 185 with plain loads, but the bench step --
// the scan on the 20 SMs beside the attention -- 626 vs 607-617 us at every
// reserve (14-20 SMs): the deeper stream slows the attention more than it
// gains.  Default 0: plain loads (4 in flight per thread).
#ifndef SDB_ARGMAX_STAGES
#define SDB_ARGMAX_STAGES 0
#endif
constexpr int kArgmaxStages = SDB_ARGMAX_STAGES;
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename T>
__device__ __forceinline__ void argmax_row(const T *__restrict__ row, int vocab, int64_t vocab_offset,
                                           bool vec_ok, long long &best, bool &nan) {
  float nacc = 0.f;
  if (sizeof(T) == 4 && vec_ok) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    const int n4 = vocab >> 2;
    float bv = -INFINITY;
    int bi = threadIdx.x < n4 ? (int)threadIdx.x : -1;
    int i = threadIdx.x;
    if (kArgmaxStages > 0) {
      extern __shared__ float4 am_ring[];  // [kArgmaxStages][kArgmaxThreads], slot = this thread's
      const int nk = (int)threadIdx.x < n4 ? (n4 - (int)threadIdx.x + kArgmaxThreads - 1) / kArgmaxThreads : 0;
#pragma unroll
      for (int k = 0; k < kArgmaxStages - 1; ++k) {
        if (k < nk) cp_async16(&am_ring[k * kArgmaxThreads + threadIdx.x], r4 + threadIdx.x + k * kArgmaxThreads);
        cp_async_commit();
      }
      for (int k = 0; k < nk; ++k) {
        const int kk = k + kArgmaxStages - 1;
        if (kk < nk)
          cp_async16(&am_ring[(kk % kArgmaxStages) * kArgmaxThreads + threadIdx.x],
                     r4 + threadIdx.x + kk * kArgmaxThreads);
        cp_async_commit();
        cp_async_wait<kArgmaxStages - 1>();  // element k has landed (this thread's own copies)
        const float4 v = am_ring[(k % kArgmaxStages) * kArgmaxThreads + threadIdx.x];
        const float m = max_nan(max_nan3(v.x, v.y, v.z), v.w);
        nacc = max_nan(nacc, m);
        if (m > bv) {
          bv = m;
          bi = (int)threadIdx.x + k * kArgmaxThreads;
        }
      }
      cp_async_wait<0>();
      i = n4;  // the loops below have nothing left
    }
    // 4 independent 16-byte loads in flight per thread
    for (; i + 3 * kArgmaxThreads < n4; i += 4 * kArgmaxThreads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = scan_ld(r4 + i + u * kArgmaxThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float m = max_nan(max_nan3(v[u].x, v[u].y, v[u].z), v[u].w);
        nacc = max_nan(nacc, m);
        if (m > bv) {
          bv = m;
          bi = i + u * kArgmaxThreads;
        }
      }
    }
    for (; i < n4; i += kArgmaxThreads) {
      const float4 v = scan_ld(r4 + i);
      const float m = max_nan(max_nan3(v.x, v.y, v.z), v.w);
      nacc = max_nan(nacc, m);
      if (m > bv) {
        bv = m;
        bi = i;
      }
    }
    if (bi >= 0) {
      const float4 v = r4[bi];
      const float e[4] = {v.x, v.y, v.z, v.w};
      int c = 3;
#pragma unroll
      for (int q = 2; q >= 0; --q)
        if (e[q] == bv) c = q;
      best = argmax_key(bv, (uint32_t)(vocab_offset + 4 * bi + c));
    }
    for (int j = 4 * n4 + threadIdx.x; j < vocab; j += kArgmaxThreads) {
      float e = to_f32<T>(row[j]);
      nan |= e != e;
      long long k = argmax_key(e, (uint32_t)(vocab_offset + j));
      best = k > best ? k : best;
    }
  } else if (sizeof(T) == 2 && vec_ok) {
    const uint4 *r8 = reinterpret_cast<const uint4 *>(row);
    const int n8 = vocab >> 3;
    float bv = -INFINITY;
    int bi = threadIdx.x < n8 ? (int)threadIdx.x : -1;
    for (int i = threadIdx.x; i < n8; i += kArgmaxThreads) {
      const uint4 v = scan_ld(r8 + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      float m = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        m = max_nan3(m, __uint_as_float(w[c] << 16), __uint_as_float(w[c] & 0xffff0000u));
      nacc = max_nan(nacc, m);
      if (m > bv) {
        bv = m;
        bi = i;
      }
    }
    if (bi >= 0) {
      const uint4 v = r8[bi];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      int c = 7;
#pragma unroll
      for (int q = 7; q >= 0; --q) {
        const float e = __uint_as_float((q & 1) ? (w[q >> 1] & 0xffff0000u) : (w[q >> 1] << 16));
        if (e == bv) c = q;
      }
      best = argmax_key(bv, (uint32_t)(vocab_offset + 8 * bi + c));
    }
    for (int j = 8 * n8 + threadIdx.x; j < vocab; j += kArgmaxThreads) {
      float e = to_f32<T>(row[j]);
      nan |= e != e;
      long long k = argmax_key(e, (uint32_t)(vocab_offset + j));
      best = k > best ? k : best;
    }
  } else {
    for (int j = threadIdx.x; j < vocab; j += kArgmaxThreads) {
      float e = to_f32<T>(row[j]);
      nan |= e != e;
      long long k = argmax_key(e, (uint32_t)(vocab_offset + j));
      best = k > best ? k : best;
    }
  }
  nan |= nacc != nacc;
}

// grid.x = rows (flat) or (r_max * split, batch) with n_rows gating; with
// split > 1 each row's vocabulary is cut into `split` segments (multiples of
// 8 elements) scanned by separate CTAs, keys[row * split + s] (small batches:
// enough CTAs to stream at HBM speed); the walk takes the max over segments.
template <typename T>
__global__ void __launch_bounds__(kArgmaxThreads, 2) argmax_keys_kernel(const T *__restrict__ logits, int vocab,
                                                                     int64_t row_stride, int64_t vocab_offset,
                                                                     const int32_t *__restrict__ n_rows,
                                                                     int r_max, long long *__restrict__ keys,
                                                                     int32_t *__restrict__ err, bool vec_ok,
                                                                     int split) {
  __shared__ long long red[kArgmaxThreads / 32];
  int64_t row;
  int seg = 0;
  if (n_rows) {
    const int r = blockIdx.x / split, b = blockIdx.y;
    seg = blockIdx.x % split;
    if (r >= n_rows[b]) return;
    row = (int64_t)b * r_max + r;
  } else {
    row = blockIdx.x + (int64_t)blockIdx.y * gridDim.x;
  }
  const int seg_len = split > 1 ? ((vocab + split - 1) / split + 7) & ~7 : vocab;
  const int v0 = min(vocab, seg * seg_len), v1 = min(vocab, v0 + seg_len);
  long long best = LLONG_MIN;
  bool nan = false;
  argmax_row<T>(logits + row * row_stride + v0, v1 - v0, vocab_offset + v0, vec_ok, best, nan);
  best = block_max_i64<kArgmaxThreads>(best, red);
  if (__syncthreads_or(nan) && threadIdx.x == 0 && err) atomicOr(err, SDB_ERR_NAN);
  if (threadIdx.x == 0) keys[row * split + seg] = best;
}

// dynamic shared memory of argmax_keys_kernel<float> (the cp.async ring),
// attribute set once
static size_t argmax_smem() {
  const size_t bytes = (size_t)kArgmaxStages * kArgmaxThreads * sizeof(float4);
  static bool set = false;
  if (!set && bytes > 0) {
    cudaFuncSetAttribute(argmax_keys_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    set = true;
  }
  return bytes;
}

// Greedy acceptance over FSM-masked rows (target_dist(row, 0, ., allowed),
// sampling.py:94-99: the argmax of the ALLOWED logits, lowest index on ties;
// a row with no allowed token is SamplingError).  Simple per-element keys:
// the unmasked rows keep the chunk-max fast path above.
__global__ void __launch_bounds__(kArgmaxThreads) argmax_keys_masked_kernel(
    const float *__restrict__ logits, int vocab, int64_t row_stride, const int32_t *__restrict__ n_rows, int r_max,
    const uint32_t *__restrict__ allowed, int n_mw, long long *__restrict__ keys, int32_t *__restrict__ err) {
  __shared__ long long red[kArgmaxThreads / 32];
  const int r = blockIdx.x, b = blockIdx.y;
  if (r >= n_rows[b]) return;
  const int64_t row = (int64_t)b * r_max + r;
  const float *lr = logits + row * row_stride;
  const uint32_t *mw = allowed + row * n_mw;
  long long best = LLONG_MIN;
  bool nan = false, any = false;
  for (int j = threadIdx.x; j < vocab; j += kArgmaxThreads) {
    if (!((__ldg(mw + (j >> 5)) >> (j & 31)) & 1u)) continue;
    any = true;
    const float e = lr[j];
    nan |= e != e;
    const long long k = argmax_key(e, (uint32_t)j);
    best = k > best ? k : best;
  }
  best = block_max_i64<kArgmaxThreads>(best, red);
  const bool any_b = __syncthreads_or(any);
  if (__syncthreads_or(nan) && threadIdx.x == 0) atomicOr(err, SDB_ERR_NAN);
  if (threadIdx.x == 0) {
    if (!any_b) atomicOr(err, SDB_ERR_NO_ALLOWED);
    keys[row * 1] = best;
  }
}

// One warp per sequence: the argmax walk in the augmented frame (row 0 =
// root; children of row r = rows j > r with parent[j] == r, index order).
constexpr int kWalkStage = 256;  // tree rows staged in shared memory per sequence (12 KB per 4 warps)

__global__ void greedy_walk_kernel(const long long *__restrict__ keys, const int32_t *__restrict__ parent,
                                   const int32_t *__restrict__ n_rows, const int32_t *__restrict__ tokens,
                                   int batch, int r_max, int32_t *__restrict__ path, int32_t *__restrict__ path_len,
                                   int64_t *__restrict__ next_token, int32_t *__restrict__ uniforms_used,
                                   int split) {
  // small trees: the sequence's parents, tokens and per-row argmax are
  // staged into shared memory with coalesced loads first, so the walk's
  // level-by-level decisions cost no dependent global round trips
  __shared__ int32_t s_par[4][kWalkStage], s_tok[4][kWalkStage], s_amax[4][kWalkStage];
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = (threadIdx.x >> 5) & 3;
  if (b >= batch) return;
  const int n = min(n_rows[b], r_max);
  const int32_t *par = parent + (int64_t)b * r_max;
  const int32_t *tok = tokens + (int64_t)b * r_max;
  const long long *key = keys + (int64_t)b * r_max * split;
  auto row_key = [&](int r) {  // max over the row's vocabulary segments
    long long k = key[(int64_t)r * split];
    for (int s = 1; s < split; ++s) k = max(k, key[(int64_t)r * split + s]);
    return k;
  };
  const bool staged = n <= kWalkStage;
  if (staged) {
    for (int r = lane; r < n; r += 32) {
      s_par[wib][r] = par[r];
      s_tok[wib][r] = tok[r];
      s_amax[wib][r] = (int)key_index(row_key(r));
    }
    __syncwarp();
  }
  auto P = [&](int j) { return staged ? s_par[wib][j] : par[j]; };
  auto T = [&](int j) { return staged ? s_tok[wib][j] : tok[j]; };
  auto A = [&](int r) { return staged ? s_amax[wib][r] : (int)key_index(row_key(r)); };
  int cur = 0, used = 0, len = 0;
  while (true) {
    const int want = A(cur);
    int accepted = -1, examined = 0;
    for (int j0 = cur + 1; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool child = j < n && P(j) == cur;
      const bool hit = child && T(j) == want;
      const unsigned cm = __ballot_sync(SDB_FULL_MASK, child);
      const unsigned hm = __ballot_sync(SDB_FULL_MASK, hit);
      if (hm) {
        const int first = __ffs(hm) - 1;
        examined += __popc(cm & ((2u << first) - 1u));
        accepted = j0 + first;
        break;
      }
      examined += __popc(cm);
    }
    used += examined;
    if (accepted < 0) break;
    if (lane == 0) path[(int64_t)b * r_max + len] = accepted - 1;
    ++len;
    cur = accepted;
  }
  if (lane == 0) {
    path_len[b] = len;
    next_token[b] = (int64_t)A(cur);
    uniforms_used[b] = used + 1;
  }
}

// ---------------------------------------------------------------------------
// stochastic
// ---------------------------------------------------------------------------
constexpr int kValSmsPer148 = 52;      // SMs of 148 the persistent validation scan takes beside the lazy chain
constexpr int kStThreads = 1024;       // one row per SM: its L2-resident working set (148 x 0.5 MB) fits the 126 MB L2
constexpr int kHistBins = 4096;        // width 1/64 log2 unit below the row max (64 log2 units)
constexpr float kHistScale = 64.0f;
constexpr int kHistCopies = 2;         // fixed-point histograms (warp-parity private copies)
constexpr int kBinsPerThread = kHistBins / kStThreads;
constexpr int kRefBins = kStThreads;   // key-space refinement bins (fallback)
constexpr int kCandCap = 4 * kStThreads;  // exact-sort capacity around the cut
// Bin b holds weights w in (2^-(b+1)/64, 2^-b/64]; it accumulates r = w *
// 2^(b/64) in (0.989, 1] as round(r * 2^14) in a native 32-bit shared atomic
// (float / 64-bit shared atomics are CAS loops).  |rounding| <= 2^-15 per
// element, i.e. a bin mass is exact to 3.1e-5 relative -- only used to pick
// the window; the mass above it is summed exactly in f64 afterwards.
constexpr float kFixScale = 16384.0f;
constexpr double kBinTol = 1e-4;

__device__ __forceinline__ int hist_bin(float x2, float m2) {
  float d = (m2 - x2) * kHistScale;
  return d >= (float)(kHistBins - 1) ? kHistBins - 1 : (int)d;
}

__device__ __forceinline__ float key_weight(uint32_t k, float a, float m2) {
  const uint32_t bits = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return exp2f(__uint_as_float(bits) * a - m2);
}

// Inclusive block scan of one double per thread (kStThreads threads).
__device__ double block_inclusive_scan(double v, double *red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(SDB_FULL_MASK, v, o);
    if (lane >= o) v += t;
  }
  __syncthreads();
  if (lane == 31) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < kStThreads / 32 ? red[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t = __shfl_up_sync(SDB_FULL_MASK, w, o);
      if (lane >= o) w += t;
    }
    red[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += red[warp - 1];
  __syncthreads();
  return v;
}

struct StSmem {
  uint32_t hist[kHistCopies][kHistBins];  // pass-2 masses (fixed point, window selection only)
  unsigned long long cand[kCandCap];   // (key << 32) | ~index
  double rh[kRefBins];                 // fallback key-space refinement (f64)
  double red[32];
  float redf[32];
  int count;
  int lo, hi, cut;
  unsigned klo, khi;
  int idx;
  double tot;
  // cluster exchange slots (lazy chain: a row split over kCS CTAs)
  float xf;
  double xd;
  int xi;
  uint32_t xlo, xhi;
};

// Guided-decoding masks (target_dist(allowed=...), sampling.py:94-97): one
// bit per token, word j of a row covers tokens [32 j, 32 j + 32); a cleared
// bit turns the logit into -inf before anything else (nullptr = all allowed).
__device__ __forceinline__ float4 mask4(float4 v, const uint32_t *mw, int i4) {
  if (mw) {
    const uint32_t bits = (__ldg(mw + (i4 >> 3)) >> ((i4 & 7) * 4)) & 0xFu;
    if (!(bits & 1u)) v.x = -INFINITY;
    if (!(bits & 2u)) v.y = -INFINITY;
    if (!(bits & 4u)) v.z = -INFINITY;
    if (!(bits & 8u)) v.w = -INFINITY;
  }
  return v;
}
__device__ __forceinline__ float mask1(float v, const uint32_t *mw, int j) {
  return (mw && !((__ldg(mw + (j >> 5)) >> (j & 31)) & 1u)) ? -INFINITY : v;
}

// Streaming max (+ NaN flag) of a row: 4 independent 16-byte loads in flight
// per thread.
__device__ __forceinline__ void row_max_nan(const float *row, int vocab, bool vec, float &mx, bool &nan,
                                            const uint32_t *mw) {
  mx = -INFINITY;
  nan = false;
  if (vec) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    const int n4 = vocab >> 2;
    int i = threadIdx.x;
    for (; i + 3 * kStThreads < n4; i += 4 * kStThreads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = mask4(__ldg(r4 + i + u * kStThreads), mw, i + u * kStThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        nan |= (v[u].x != v[u].x) | (v[u].y != v[u].y) | (v[u].z != v[u].z) | (v[u].w != v[u].w);
        mx = fmaxf(mx, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
      }
    }
    for (; i < n4; i += kStThreads) {
      const float4 v = mask4(__ldg(r4 + i), mw, i);
      nan |= (v.x != v.x) | (v.y != v.y) | (v.z != v.z) | (v.w != v.w);
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (int j = (n4 << 2) + threadIdx.x; j < vocab; j += kStThreads) {
      const float v = mask1(row[j], mw, j);
      nan |= v != v;
      mx = fmaxf(mx, v);
    }
  } else {
    for (int j = threadIdx.x; j < vocab; j += kStThreads) {
      const float v = mask1(row[j], mw, j);
      nan |= v != v;
      mx = fmaxf(mx, v);
    }
  }
}

// Exact cut among `count` (<= kCandCap) candidates in sm.cand whose mass
// above is mass_above: sort by (key desc, index asc), first position whose
// cumulative mass reaches tau.  Returns the kept mass; sets cut key / index.
__device__ double exact_cut(StSmem &sm, int count, double mass_above, double tau, float a, float m2,
                            uint32_t &cut_key, int &cut_idx) {
  const unsigned long long *buf = sm.cand;
  if (count <= kStThreads) {
    // rank sort (keys are unique: the low word is ~index): one pass over the
    // candidates per thread and a scatter, instead of log^2 barrier stages
    unsigned long long *sorted = reinterpret_cast<unsigned long long *>(&sm.hist[0][0]);  // histogram is done
    if ((int)threadIdx.x < count) {
      const unsigned long long me = sm.cand[threadIdx.x];
      int rank = 0;
      for (int j = 0; j < count; ++j) rank += sm.cand[j] > me;
      sorted[rank] = me;
    }
    __syncthreads();
    buf = sorted;
  } else {
    int np2 = 1;
    while (np2 < count) np2 <<= 1;
    for (int i = count + threadIdx.x; i < np2; i += kStThreads) sm.cand[i] = 0ull;
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < np2; i += kStThreads) {
          const int j = i ^ stride;
          if (j > i) {
            const bool desc = (i & size) == 0;
            const unsigned long long x = sm.cand[i], y = sm.cand[j];
            if (desc ? (x < y) : (x > y)) {
              sm.cand[i] = y;
              sm.cand[j] = x;
            }
          }
        }
        __syncthreads();
      }
    }
  }
  // per-thread chunk of 4 consecutive sorted candidates
  constexpr int kPer = kCandCap / kStThreads;
  double loc[kPer], wv[kPer];
  double tot = 0.0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = threadIdx.x * kPer + u;
    wv[u] = i < count ? (double)key_weight((uint32_t)(buf[i] >> 32), a, m2) : 0.0;
    tot += wv[u];
    loc[u] = tot;
  }
  const double incl = block_inclusive_scan(tot, sm.red);
  const double base = mass_above + incl - tot;
  if (threadIdx.x == 0) sm.cut = count - 1;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = threadIdx.x * kPer + u;
    if (i < count && base + loc[u] >= tau) atomicMin(&sm.cut, i);
  }
  __syncthreads();
  const int cpos = sm.cut;
  double zz = 0.0;
#pragma unroll
  for (int u = 0; u < kPer; ++u)
    if (threadIdx.x * kPer + u <= cpos) zz += wv[u];
  const double z = mass_above + block_sum<kStThreads>(zz, sm.red);
  cut_key = (uint32_t)(buf[cpos] >> 32);
  cut_idx = (int)(0xffffffffu - (uint32_t)(buf[cpos] & 0xffffffffu));
  return z;
}

// Phase A.  grid (r_max, batch, 2): z = 0 target rows (nucleus), z = 1 draft
// rows that have children (full softmax).  One HBM pass (max); then, from
// L2, the normaliser with a 1/64-log2-unit mass histogram (nucleus rows) and
// one pass that sums the exact (f64) mass above the bins straddling the cut
// and collects their few elements, which are sorted exactly by (key desc,
// index asc) -- the reference's top_p_mask order (sampling.py:57-72).
#ifdef SDB_TRACE
// [launch][phase] clock64 stamps of the target row of sequence 0 (trace builds)
__device__ unsigned long long g_st_trace[16][8];
__device__ unsigned int g_st_launch;
#define ST_TRACE(ph)                                                                          \
  do {                                                                                        \
    if (st_tr && threadIdx.x == 0) g_st_trace[st_launch & 15][ph] = clock64();                \
  } while (0)
#else
#define ST_TRACE(ph) \
  do {               \
  } while (0)
#endif
// kCS > 1 (lazy chain, launched as clusters of kCS CTAs per row): every CTA of
// the cluster streams a contiguous 1/kCS of the row through the three passes;
// the max, the normaliser, the mass histogram, the mass above the window and
// the window's candidates are combined through distributed shared memory, and
// CTA 0 finishes the cut (and, in the rare refinement cases, re-reads the
// whole row alone).  At the chain's later levels, with few rows left, a row's
// passes then run on kCS SMs instead of one.
template <bool kMasked, int kCS>
__global__ void __launch_bounds__(kStThreads, 1) row_stats_kernel(
    const float *__restrict__ target, const float *__restrict__ draft, int r_max, int vocab, float a,
    float top_p, const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows,
    RowStats *__restrict__ stats, int32_t *__restrict__ err, const uint32_t *__restrict__ allowed, int n_mw,
    const int32_t *__restrict__ cur_rows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StSmem &sm = *reinterpret_cast<StSmem *>(smem_raw);
  const int crank = kCS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  // lazy mode (cur_rows): the one row per sequence the walk is at (-1: done)
  const int r = cur_rows ? cur_rows[blockIdx.y] : (int)(blockIdx.x / kCS), b = blockIdx.y, is_draft = blockIdx.z;
#ifdef SDB_TRACE
  const bool st_tr = b == 0 && is_draft == 0 && (cur_rows || blockIdx.x == 0);
  unsigned int st_launch = 0;
  if (st_tr && threadIdx.x == 0) st_launch = atomicAdd(&g_st_launch, 1u);
#endif
  ST_TRACE(0);
  if (r < 0) return;
  const int n = min(n_rows[b], r_max);
  RowStats *out = stats + ((int64_t)b * r_max + r) * 2 + is_draft;
  if (r >= n) {
    if (threadIdx.x == 0 && crank == 0) out->valid = 0;
    return;
  }
  if (is_draft) {
    // only parent rows carry a q (their children's proposal distribution)
    const int32_t *par = parent + (int64_t)b * r_max;
    int has = 0;
    for (int j = r + 1 + threadIdx.x; j < n; j += kStThreads) has |= par[j] == r;
    if (!__syncthreads_or(has)) {
      if (threadIdx.x == 0 && crank == 0) out->valid = 0;
      return;
    }
  }
  const float *row = (is_draft ? draft : target) + ((int64_t)b * r_max + r) * vocab;
  // the row's FSM mask masks its target dist and the q its children were
  // drafted from alike (engine.py:465-475, 266-269: same FSM state)
  const uint32_t *mw = kMasked ? allowed + ((int64_t)b * r_max + r) * n_mw : nullptr;
  const bool vec = (vocab & 3) == 0 && ((uintptr_t)row & 15) == 0;
  const bool nucleus = !is_draft && top_p < 1.0f;
  // row split: CTA crank streams [v0, v1); unaligned rows stay on CTA 0
  const bool solo = kCS == 1 || !vec;
  if (solo && crank != 0) return;  // (uniform over the other CTAs: no exchange follows)
  int v0 = 0, v1 = vocab;
  if (!solo) {
    const int per = ((vocab + kCS - 1) / kCS + 3) & ~3;
    v0 = min(vocab, crank * per);
    v1 = min(vocab, v0 + per);
  }
  // [write own slot; cluster barrier; read every CTA's; cluster barrier]:
  // the second barrier keeps a CTA's slots alive until every peer read them
  auto cl_sync = [&]() {
    if (!solo) cg::this_cluster().sync();
  };
  auto peer = [&](auto *p_, int q) { return cg::this_cluster().map_shared_rank(p_, q); };
  // the whole row streams into L2 through the TMA engine (deep memory-level
  // parallelism); the passes below then hit L2
// whole-row L2 bulk prefetch before pass 1: off by default (C5 eager 1316 vs
// 1350 us with it; lazy unchanged at 941-946: the chain's row stats are bound
// by the histogram / window passes -- clock64 trace, tools/trace_rowstats.py:
// max pass 12-18 k cycles, normaliser + histogram 27 k, mass above + window
// collection 23-41 k, exact cut 7-14 k)
#ifndef SDB_ST_PREFETCH
#define SDB_ST_PREFETCH 0
#endif
  if (SDB_ST_PREFETCH && vec && threadIdx.x == 0) {
    constexpr uint32_t kChunk = 64u << 10;
    const uint32_t bytes = (uint32_t)vocab * 4u;
    for (uint32_t o = 0; o < bytes; o += kChunk) prefetch_l2((const char *)row + o, min(kChunk, bytes - o));
  }
  const int n4 = vec ? (v1 - v0) >> 2 : 0;  // this CTA's slice (the whole row when solo)
  const int i4_0 = v0 >> 2;                 // its first float4 index in the row
  const float4 *r4 = reinterpret_cast<const float4 *>(row + v0);
  constexpr int kU = 4;  // 16-byte loads in flight per thread
  if (nucleus)
    for (int i = threadIdx.x; i < kHistCopies * kHistBins; i += kStThreads) (&sm.hist[0][0])[i] = 0u;
  // pass 1: max + NaN (3-input max.NaN: NaN propagates into the maximum)
#ifndef SDB_ST_KU1
#define SDB_ST_KU1 4
#endif
  constexpr int kU1 = SDB_ST_KU1;  // loads in flight per thread in the HBM pass
  float mx = -INFINITY;
  for (int i0 = 0; i0 < n4; i0 += kU1 * kStThreads) {
    float4 v[kU1];
#pragma unroll
    for (int u = 0; u < kU1; ++u) {
      const int i = i0 + u * kStThreads + threadIdx.x;
      v[u] = i < n4 ? mask4(__ldg(r4 + i), mw, i4_0 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < kU1; ++u) mx = max3_nan(mx, max3_nan(v[u].x, v[u].y, v[u].z), v[u].w);
  }
  for (int j = v0 + (n4 << 2) + threadIdx.x; j < v1; j += kStThreads) mx = max3_nan(mx, mask1(row[j], mw, j), mask1(row[j], mw, j));
  bool has_nan = __syncthreads_or(mx != mx);
  if (!has_nan) mx = block_max<kStThreads>(mx, sm.redf);
  if (!solo) {
    if (threadIdx.x == 0) sm.xf = has_nan ? NAN : mx;
    cl_sync();
    float m_all = -INFINITY;
    bool nan_all = false;
#pragma unroll
    for (int q = 0; q < kCS; ++q) {
      const float x = *peer(&sm.xf, q);
      nan_all |= x != x;
      m_all = fmaxf(m_all, x);
    }
    cl_sync();
    has_nan = nan_all;
    mx = m_all;
  }
  if (has_nan) {
    if (threadIdx.x == 0 && crank == 0) {
      atomicOr(err, SDB_ERR_NAN);
      out->valid = 0;
    }
    return;
  }
  ST_TRACE(1);
  if (mx == -INFINITY) {  // no allowed token (dead FSM state, sampling.py:96-97) / no finite logit
    if (threadIdx.x == 0 && crank == 0) {
      atomicOr(err, mw ? SDB_ERR_NO_ALLOWED : SDB_ERR_BAD_DIST);
      out->valid = 0;
    }
    return;
  }
  const float m2 = mx * a;
  if (!nucleus) {
    // draft rows (and top_p = 1): the normaliser, two elements per packed op
    const uint64_t A2 = f2splat(a), NM2 = f2splat(-m2);
    uint64_t s2 = 0;
    for (int i0 = 0; i0 < n4; i0 += kU * kStThreads) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kStThreads + threadIdx.x;
        v[u] = i < n4 ? mask4(__ldg(r4 + i), mw, i4_0 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float e0, e1, e2, e3;
        f2unpack(ffma2(f2pack(v[u].x, v[u].y), A2, NM2), e0, e1);
        f2unpack(ffma2(f2pack(v[u].z, v[u].w), A2, NM2), e2, e3);
        s2 = fadd2(s2, fadd2(f2pack(ex2(e0), ex2(e1)), f2pack(ex2(e2), ex2(e3))));
      }
    }
    float s_lo, s_hi;
    f2unpack(s2, s_lo, s_hi);
    float s_loc = s_lo + s_hi;
    for (int j = v0 + (n4 << 2) + threadIdx.x; j < v1; j += kStThreads) s_loc += ex2(fmaf(mask1(row[j], mw, j), a, -m2));
    double s = block_sum<kStThreads>((double)s_loc, sm.red);
    if (!solo) {
      if (threadIdx.x == 0) sm.xd = s;
      cl_sync();
      s = 0.0;
#pragma unroll
      for (int q = 0; q < kCS; ++q) s += *peer(&sm.xd, q);
      cl_sync();
    }
    if (threadIdx.x == 0 && crank == 0) {
      RowStats st;
      st.m2 = m2;
      st.s = s;
      st.z = s;
      st.log2_z = (float)log2(s);
      st.cut_key = 0;
      st.cut_idx = 0;
      st.keep_all = 1;
      st.valid = 1;
      *out = st;
    }
    return;
  }
  // pass 2 (L2): normaliser + mass histogram, two elements per packed op.
  // d = (m2 - x a) * 64 >= 0; bin = round(d) by the 1.5 * 2^23 magic add;
  // r = 2^-(d - bin)/64 = e^-t by a quadratic (|error| < 3e-8); the bin
  // accumulates round(r * 2^14) in a native 32-bit shared atomic.
  constexpr float kMagic = 12582912.0f;
  const uint32_t kMagicBits = __float_as_uint(kMagic);
  uint32_t *hist = sm.hist[(threadIdx.x >> 5) & (kHistCopies - 1)];
  const uint64_t A2 = f2splat(a), NM2 = f2splat(-m2), DA2 = f2splat(-kHistScale * a),
                 DM2 = f2splat(kHistScale * m2), MAG2 = f2splat(kMagic), NMAG2 = f2splat(-kMagic),
                 TC2 = f2splat(0.6931471805599453f / kHistScale), HALF2 = f2splat(0.5f), NEG1 = f2splat(-1.0f),
                 ONE2 = f2splat(1.0f), FIX2 = f2splat(kFixScale);
  uint64_t s2 = 0;  // packed (0.f, 0.f)
  auto acc2 = [&](uint64_t l2) {
    float e0, e1;
    f2unpack(ffma2(l2, A2, NM2), e0, e1);
    s2 = fadd2(s2, f2pack(ex2(e0), ex2(e1)));
    const uint64_t d = ffma2(l2, DA2, DM2);
    const uint64_t g = fadd2(d, MAG2);
    const uint64_t t = fmul2(fsub2(d, fadd2(g, NMAG2)), TC2);
    const uint64_t rr = ffma2(t, ffma2(t, HALF2, NEG1), ONE2);
    const uint64_t fx = ffma2(rr, FIX2, MAG2);
    // branch-free: out-of-range bins (d >= 4095, or -inf padding) add 0 to
    // some bin (spread, so masked/-inf rows do not serialise on one address)
    const uint32_t b0 = (uint32_t)g - kMagicBits, b1 = (uint32_t)(g >> 32) - kMagicBits;
    const uint32_t f0 = b0 < (uint32_t)(kHistBins - 1) ? (uint32_t)fx - kMagicBits : 0u;
    const uint32_t f1 = b1 < (uint32_t)(kHistBins - 1) ? (uint32_t)(fx >> 32) - kMagicBits : 0u;
    atomicAdd(&hist[b0 & (kHistBins - 1)], f0);
    atomicAdd(&hist[b1 & (kHistBins - 1)], f1);
  };
  for (int i0 = 0; i0 < n4; i0 += kU * kStThreads) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kStThreads + threadIdx.x;
      v[u] = i < n4 ? mask4(__ldg(r4 + i), mw, i4_0 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      acc2(f2pack(v[u].x, v[u].y));
      acc2(f2pack(v[u].z, v[u].w));
    }
  }
  float s_lo, s_hi;
  f2unpack(s2, s_lo, s_hi);
  float s_loc = s_lo + s_hi;
  for (int j = v0 + (n4 << 2) + threadIdx.x; j < v1; j += kStThreads) {
    const float x = mask1(row[j], mw, j);
    const uint64_t l2 = f2pack(x, -INFINITY);
    s2 = 0;
    acc2(l2);
    f2unpack(s2, s_lo, s_hi);
    s_loc += s_lo;
  }
  double s = block_sum<kStThreads>((double)s_loc, sm.red);  // (also orders the histogram atomics)
  if (!solo) {
    if (threadIdx.x == 0) sm.xd = s;
    cl_sync();  // every CTA's normaliser and histogram are complete
    s = 0.0;
#pragma unroll
    for (int q = 0; q < kCS; ++q) s += *peer(&sm.xd, q);
  }
  ST_TRACE(2);
  const double tau = ((double)top_p - 1e-12) * s;
  // window [lo, hi] of bins whose cumulative (bin 0 = largest values) may
  // straddle tau given the fixed-point bin sums
  {
    double loc[kBinsPerThread];
    double tsum = 0.0;
#pragma unroll
    for (int u = 0; u < kBinsPerThread; ++u) {
      const int bb = threadIdx.x * kBinsPerThread + u;
      unsigned long long q = 0;
#pragma unroll
      for (int c = 0; c < kHistCopies; ++c) {
        if (solo) {
          q += sm.hist[c][bb];
        } else {
#pragma unroll
          for (int w = 0; w < kCS; ++w) q += *peer(&sm.hist[c][bb], w);
        }
      }
      // mass = 2^(-bb/64) * q / 2^14
      tsum += (double)q * (double)exp2f(-(float)bb * (1.0f / kHistScale)) * (1.0 / kFixScale);
      loc[u] = tsum;
    }
    if (threadIdx.x == 0) {
      sm.lo = kHistBins - 1;
      sm.hi = kHistBins - 1;
      sm.count = 0;
      sm.klo = 0xffffffffu;
      sm.khi = 0u;
    }
    const double excl = block_inclusive_scan(tsum, sm.red) - tsum;
    int mlo = kHistBins - 1, mhi = kHistBins - 1;
#pragma unroll
    for (int u = kBinsPerThread - 1; u >= 0; --u) {
      const double cv = excl + loc[u];
      if (cv >= tau * (1.0 - kBinTol)) mlo = threadIdx.x * kBinsPerThread + u;
      if (cv >= tau * (1.0 + kBinTol)) mhi = threadIdx.x * kBinsPerThread + u;
    }
    atomicMin(&sm.lo, mlo);
    atomicMin(&sm.hi, mhi);
    __syncthreads();
  }
  const int lo = sm.lo, hi = max(sm.hi, sm.lo);
  cl_sync();  // every CTA read the peers' histograms (exact_cut reuses them as scratch)
  ST_TRACE(3);
  // pass 3 (L2): the same d splits the keys monotonically into above (d <
  // lo - 1/2), the window and below; exact mass above, window elements
  // collected with warp-aggregated slots.  Keys with equal logits share d,
  // so ties are never split.
  const float dlo = (float)lo - 0.5f, dhi = (float)hi + 0.5f;
  float above = 0.f;
  {
    unsigned kl = 0xffffffffu, kh = 0u;
    const int lane = threadIdx.x & 31;
    // append this thread's `cnt` window elements (warp prefix -> slots)
    auto append_slots = [&](int cnt) {
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(SDB_FULL_MASK, incl, o);
        if (lane >= o) incl += t;
      }
      int base = 0;
      if (lane == 31) base = atomicAdd(&sm.count, incl);
      return __shfl_sync(SDB_FULL_MASK, base, 31) + incl - cnt;
    };
    auto put = [&](int slot, float x, int idx) {
      const uint32_t k = prob_key(x);
      if (slot < kCandCap) sm.cand[slot] = ((unsigned long long)k << 32) | (0xffffffffu - (uint32_t)idx);
      kl = min(kl, k);
      kh = max(kh, k);
    };
    uint64_t ab2 = 0;
    for (int i0 = 0; i0 < n4; i0 += kU * kStThreads) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kStThreads + threadIdx.x;
        v[u] = i < n4 ? mask4(__ldg(r4 + i), mw, i4_0 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
      uint32_t mask = 0;  // bit 4u+e: element e of v[u] lies in the window
#pragma unroll
      for (int u = 0; u < kU; ++u) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint64_t l2 = h ? f2pack(v[u].z, v[u].w) : f2pack(v[u].x, v[u].y);
          float d0, d1, e0, e1;
          f2unpack(ffma2(l2, DA2, DM2), d0, d1);
          f2unpack(ffma2(l2, A2, NM2), e0, e1);
          ab2 = fadd2(ab2, f2pack(d0 < dlo ? ex2(e0) : 0.f, d1 < dlo ? ex2(e1) : 0.f));
          mask |= (uint32_t)(d0 >= dlo && d0 < dhi) << (4 * u + 2 * h);
          mask |= (uint32_t)(d1 >= dlo && d1 < dhi) << (4 * u + 2 * h + 1);
        }
      }
      if (__any_sync(SDB_FULL_MASK, mask != 0)) {
        int slot = append_slots(__popc(mask));
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int bi = v0 + 4 * (i0 + u * kStThreads + threadIdx.x);
          if (mask & (1u << (4 * u))) put(slot++, v[u].x, bi);
          if (mask & (2u << (4 * u))) put(slot++, v[u].y, bi + 1);
          if (mask & (4u << (4 * u))) put(slot++, v[u].z, bi + 2);
          if (mask & (8u << (4 * u))) put(slot++, v[u].w, bi + 3);
        }
      }
    }
    float a_lo, a_hi;
    f2unpack(ab2, a_lo, a_hi);
    above = a_lo + a_hi;
    // scalar tail (and the non-vector path): one element per thread per step
    const int t0 = v0 + (n4 << 2);
    for (int j0 = t0; j0 < v1; j0 += kStThreads) {
      const int j = j0 + threadIdx.x;
      float x = 0.f;
      int cnt = 0;
      if (j < v1) {
        x = mask1(row[j], mw, j);
        float d0, d1, e0, e1;
        const uint64_t l2 = f2pack(x, x);
        f2unpack(ffma2(l2, DA2, DM2), d0, d1);
        f2unpack(ffma2(l2, A2, NM2), e0, e1);
        if (d0 < dlo) above += ex2(e0);
        cnt = d0 >= dlo && d0 < dhi;
      }
      if (__any_sync(SDB_FULL_MASK, cnt != 0)) {
        const int slot = append_slots(cnt);
        if (cnt) put(slot, x, j);
      }
    }
    atomicMin(&sm.klo, kl);
    atomicMax(&sm.khi, kh);
  }
  double mass_above = block_sum<kStThreads>((double)above, sm.red);  // (syncs sm.count / klo / khi too)
  if (!solo) {
    // combine: mass above, key range, candidates (gathered into CTA 0's list)
    if (threadIdx.x == 0) {
      sm.xd = mass_above;
      sm.xi = sm.count;
      sm.xlo = sm.klo;
      sm.xhi = sm.khi;
    }
    cl_sync();
    double ma = 0.0;
    int total = 0, base = 0;
    uint32_t kl = 0xffffffffu, kh = 0u;
#pragma unroll
    for (int q = 0; q < kCS; ++q) {
      const int cq = *peer(&sm.xi, q);
      if (q < crank) base += cq;
      total += cq;
      ma += *peer(&sm.xd, q);
      kl = min(kl, *peer(&sm.xlo, q));
      kh = max(kh, *peer(&sm.xhi, q));
    }
    if (crank == 0 && total <= kCandCap) {
      int off = sm.count;  // CTA 0's own candidates stay at [0, count)
#pragma unroll
      for (int q = 1; q < kCS; ++q) {
        const int cq = *peer(&sm.xi, q);
        const unsigned long long *pc = peer(&sm.cand[0], q);
        for (int k = threadIdx.x; k < cq; k += kStThreads) sm.cand[off + k] = pc[k];
        off += cq;
      }
    }
    (void)base;
    cl_sync();  // the peers' candidates are read: they may leave
    if (crank != 0) return;
    mass_above = ma;
    if (threadIdx.x == 0) {
      sm.count = total;
      sm.klo = kl;
      sm.khi = kh;
    }
    __syncthreads();
  }
  ST_TRACE(4);
  uint32_t klo = sm.klo, khi = sm.khi;
  uint32_t cut_key = 0;
  int cut_idx = -1;
  double z = 0.0;
  bool collected = true;
  if (mass_above >= tau || sm.count == 0) {
    // the f32 histogram misplaced the window (never expected): refine over
    // every key from scratch
    klo = 0u;
    khi = 0xffffffffu;
    mass_above = 0.0;
    collected = false;
  }
  for (int level = 0; level < 8; ++level) {
    if (!collected) {
      if (threadIdx.x == 0) sm.count = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < vocab; i += kStThreads) {
        const uint32_t k = prob_key(mask1(row[i], mw, i));
        if (k >= klo && k <= khi) {
          const int slot = atomicAdd(&sm.count, 1);
          if (slot < kCandCap) sm.cand[slot] = ((unsigned long long)k << 32) | (0xffffffffu - (uint32_t)i);
        }
      }
      __syncthreads();
    }
    collected = false;
    const int count = sm.count;
    if (count == 0) {  // empty range (defensive): everything above is kept
      cut_key = khi;
      cut_idx = INT_MAX;
      z = mass_above;
      break;
    }
    if (count <= kCandCap) {
      z = exact_cut(sm, count, mass_above, tau, a, m2, cut_key, cut_idx);
      ST_TRACE(5);
      break;
    }
    if (klo == khi) {
      // only ties remain: all candidates share the weight w*; the first j by
      // index are kept, j = ceil((tau - mass_above) / w*)
      const double w = (double)key_weight(klo, a, m2);
      long long need = (long long)ceil((tau - mass_above) / w);
      need = need < 1 ? 1 : (need > count ? count : need);
      // index of the need-th tied element in index order: chunked prefix count
      if (threadIdx.x == 0) sm.idx = vocab - 1;
      __syncthreads();
      long long seen = 0;
      for (int c0 = 0; c0 < vocab; c0 += kStThreads) {
        const int i = c0 + threadIdx.x;
        const bool t = i < vocab && prob_key(mask1(row[i], mw, i)) == klo;
        const double pre = block_inclusive_scan(t ? 1.0 : 0.0, sm.red);
        if (t && seen + (long long)pre == need) sm.idx = i;
        if (threadIdx.x == kStThreads - 1) sm.tot = pre;
        __syncthreads();
        seen += (long long)sm.tot;
        __syncthreads();
        if (seen >= need) break;
      }
      __syncthreads();
      cut_key = klo;
      cut_idx = sm.idx;
      z = mass_above + w * (double)need;
      break;
    }
    // refine: kRefBins sub-ranges of [klo, khi] by key (bin 0 = highest keys)
    sm.rh[threadIdx.x] = 0.0;
    __syncthreads();
    const unsigned long long span = (unsigned long long)(khi - klo) + 1ull;
    for (int i = threadIdx.x; i < vocab; i += kStThreads) {
      const float l = mask1(row[i], mw, i);
      const uint32_t k = prob_key(l);
      if (k >= klo && k <= khi) {
        const int bin = (int)(((unsigned long long)(khi - k) * kRefBins) / span);
        atomicAdd(&sm.rh[bin], (double)exp2f(l * a - m2));
      }
    }
    __syncthreads();
    const double rc = mass_above + block_inclusive_scan(sm.rh[threadIdx.x], sm.red);
    if (threadIdx.x == 0) {
      sm.lo = kRefBins - 1;
      sm.hi = kRefBins - 1;
    }
    __syncthreads();
    if (rc >= tau * (1.0 - 1e-9)) atomicMin(&sm.lo, (int)threadIdx.x);
    if (rc >= tau * (1.0 + 1e-9)) atomicMin(&sm.hi, (int)threadIdx.x);
    __syncthreads();
    const int blo = sm.lo, bhi = max(sm.hi, sm.lo);
    if (threadIdx.x == blo - 1) sm.tot = rc;
    __syncthreads();
    if (blo > 0) mass_above = sm.tot;
    // key range of bins [blo, bhi]: bin(k) = floor((khi - k) * B / span)
    const uint32_t nkhi = khi - (uint32_t)(((unsigned long long)blo * span + kRefBins - 1) / kRefBins);
    const uint32_t nklo_off = (uint32_t)((((unsigned long long)(bhi + 1)) * span + kRefBins - 1) / kRefBins) - 1u;
    const uint32_t nklo = khi - min((unsigned long long)nklo_off, (unsigned long long)(khi - klo));
    klo = nklo;
    khi = nkhi;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    RowStats st;
    st.m2 = m2;
    st.s = s;
    st.z = z;
    st.log2_z = (float)log2(z);
    st.cut_key = cut_key;
    st.cut_idx = cut_idx;
    st.keep_all = 0;
    st.valid = 1;
    *out = st;
  }
}

// Phase B: one thread-block cluster of kCl CTAs per sequence.  Every CTA
// makes the same walk decisions (sampling.py:173-202) from the same inputs;
// each owns a contiguous 1/kCl of the vocabulary for the full-row passes (a
// rejection's residual mass, the bonus inverse CDF), whose block sums are
// exchanged through distributed shared memory.  A rejection's residual
// norm(max(p - q, 0)) is kept in closed form max(P - c Q, 0) / M (siblings
// share the parent's q, engine.py:405-407).
constexpr int kWThreads = 512;

struct WalkRow {
  const float *tl;  // target logits row
  const float *dl;  // draft logits row (nullptr when the row has no children)
  float p_off, q_off;  // -(m2 + log2 Z) of the target / draft softmax
  float cut_l;         // nucleus cut logit (keys above are kept; ties by index)
  int cut_idx, keep_all;
  const uint32_t *mw;  // FSM allowed-token bits of the row (nullptr = all)
};

__device__ __forceinline__ float key_to_logit(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// target p of logit l at vocab index i (target_dist, sampling.py:87-102)
__device__ __forceinline__ float p_val(const WalkRow &w, float a, float l, int i) {
  const bool keep = w.keep_all || l > w.cut_l || (l == w.cut_l && i <= w.cut_idx);
  return keep ? ex2(fmaf(l, a, w.p_off)) : 0.f;
}
__device__ __forceinline__ float q_val(const WalkRow &w, float a, float d) { return ex2(fmaf(d, a, w.q_off)); }
__device__ __forceinline__ float p_of(const WalkRow &w, float a, int t) {
  return p_val(w, a, mask1(w.tl[t], w.mw, t), t);
}
__device__ __forceinline__ float q_of(const WalkRow &w, float a, int t) {
  return w.dl ? q_val(w, a, mask1(w.dl[t], w.mw, t)) : 0.f;
}

// sum over [v0, v1) of max(P - c Q, 0) / M (per-element fp32, f64
// accumulation), with the values optionally stored (residual); 16-byte
// loads, 4 iterations in flight.
// `store` (global, vocab-indexed) and `sst` (shared, slice-indexed) are optional.
__device__ __forceinline__ double residual_part(const WalkRow &w, float a, double c, double M, int v0, int v1,
                                                bool vec, float *__restrict__ store, float *__restrict__ sst) {
  double part = 0.0;
  const float *__restrict__ tl = w.tl;
  const float *__restrict__ dl = w.dl;
  const float cf = (float)c, inv_m = (float)(1.0 / M);
  auto one = [&](float l, float d, int i) {
    const float p = p_val(w, a, l, i);
    const float q = dl ? q_val(w, a, d) : 0.f;
    const float v = fmaxf(fmaf(-cf, q, p), 0.f) * inv_m;
    if (store) store[i] = v;
    if (sst) sst[i - v0] = v;
    part += (double)v;
  };
  if (vec) {
    const float4 *__restrict__ t4 = reinterpret_cast<const float4 *>(tl + v0);
    const float4 *__restrict__ d4 = dl ? reinterpret_cast<const float4 *>(dl + v0) : nullptr;
    const int n4 = (v1 - v0) >> 2;
#pragma unroll 4
    for (int i = threadIdx.x; i < n4; i += kWThreads) {
      const float4 t = mask4(__ldg(t4 + i), w.mw, (v0 >> 2) + i);
      const float4 d = d4 ? mask4(__ldg(d4 + i), w.mw, (v0 >> 2) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      const int base = v0 + 4 * i;
      one(t.x, d.x, base);
      one(t.y, d.y, base + 1);
      one(t.z, d.z, base + 2);
      one(t.w, d.w, base + 3);
    }
    for (int i = v0 + (n4 << 2) + threadIdx.x; i < v1; i += kWThreads)
      one(mask1(tl[i], w.mw, i), dl ? mask1(dl[i], w.mw, i) : 0.f, i);
  } else {
    for (int i = v0 + threadIdx.x; i < v1; i += kWThreads) one(mask1(tl[i], w.mw, i), dl ? mask1(dl[i], w.mw, i) : 0.f, i);
  }
  return part;
}

// A node's first rejection pass also compacts the (P, Q) pairs with P > 0
// into shared memory (kWCap pairs per CTA): every later sibling's residual
// sum then reads only the nucleus -- elements with P == 0 add exactly 0 to
// sum max(P - c Q, 0).  Overflow (a nucleus wider than kWCap per slice, e.g.
// top_p = 1) falls back to full-row passes.
constexpr int kWCap = 12288;  // 96 KB of float2 per CTA (two CTAs per SM)

__device__ __forceinline__ double residual_compact(const WalkRow &w, float a, float cf, int v0, int v1, bool vec,
                                                   float2 *__restrict__ list, int *s_cnt) {
  double part = 0.0;
  const float *__restrict__ tl = w.tl;
  const float *__restrict__ dl = w.dl;
  const int lane = threadIdx.x & 31;
  // warp-aggregated, order-free append of this thread's kept pairs
  auto append = [&](int n, const float *pp, const float *qq) {
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(SDB_FULL_MASK, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(SDB_FULL_MASK, incl, 31);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(s_cnt, total);
    base = __shfl_sync(SDB_FULL_MASK, base, 31) + incl - n;
    for (int k = 0; k < n; ++k)
      if (base + k < kWCap) list[base + k] = make_float2(pp[k], qq[k]);
  };
  auto one = [&](float l, float d, int i, float *pp, float *qq, int &n) {
    const float p = p_val(w, a, l, i);
    const float q = dl ? q_val(w, a, d) : 0.f;
    part += (double)fmaxf(fmaf(-cf, q, p), 0.f);
    if (p > 0.f) {
      pp[n] = p;
      qq[n] = q;
      ++n;
    }
  };
  const int start = vec ? v0 + (((v1 - v0) >> 2) << 2) : v0;
  if (vec) {
    const float4 *__restrict__ t4 = reinterpret_cast<const float4 *>(tl + v0);
    const float4 *__restrict__ d4 = dl ? reinterpret_cast<const float4 *>(dl + v0) : nullptr;
    const int n4 = (v1 - v0) >> 2;
    // warp-uniform trip count (every lane takes part in the append)
    for (int i = threadIdx.x; i - lane < n4; i += kWThreads) {
      float pp[4], qq[4];
      int n = 0;
      if (i < n4) {
        const float4 t = mask4(__ldg(t4 + i), w.mw, (v0 >> 2) + i);
        const float4 d = d4 ? mask4(__ldg(d4 + i), w.mw, (v0 >> 2) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        const int base = v0 + 4 * i;
        one(t.x, d.x, base, pp, qq, n);
        one(t.y, d.y, base + 1, pp, qq, n);
        one(t.z, d.z, base + 2, pp, qq, n);
        one(t.w, d.w, base + 3, pp, qq, n);
      }
      append(n, pp, qq);
    }
  }
  for (int i = start + threadIdx.x; i - lane < v1; i += kWThreads) {
    float pp[1], qq[1];
    int n = 0;
    if (i < v1) one(mask1(tl[i], w.mw, i), dl ? mask1(dl[i], w.mw, i) : 0.f, i, pp, qq, n);
    append(n, pp, qq);
  }
  return part;
}

__device__ __forceinline__ double residual_list(const float2 *__restrict__ list, int cnt, float cf) {
  double part = 0.0;
#pragma unroll 4
  for (int i = threadIdx.x; i < cnt; i += kWThreads) {
    const float2 pq = list[i];
    part += (double)fmaxf(fmaf(-cf, pq.y, pq.x), 0.f);
  }
  return part;
}

// Cluster-wide exchange of one double per CTA: returns all kCl values in
// CTA-rank order (identical on every CTA).  Two alternating slots make one
// cluster barrier per exchange sufficient.
template <int kCl>
__device__ __forceinline__ void cluster_exchange(double v, double *slots, int &phase, double *out) {
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) slots[phase & 1] = v;
  cl.sync();
#pragma unroll
  for (int q = 0; q < kCl; ++q) out[q] = *cl.map_shared_rank(&slots[phase & 1], q);
  ++phase;
}

// Lazy mode (kLazy): one tree level per launch.  The walk state lives in
// `lw` and the current node in `cur_rows`; row_stats ran for exactly those
// rows beforehand.  Only the rows the walk visits are ever reduced
// (mss_verify reads no other target dist, sampling.py:173-202).
struct LazyWalk {
  double c, M;
  int32_t cur, used, len, done;
};

template <int kCl, bool kMasked, bool kLazy>
__global__ void __launch_bounds__(kWThreads, 2) stochastic_walk_kernel(
    const float *__restrict__ target, const float *__restrict__ draft, int r_max, int vocab, float a,
    const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows, const int32_t *__restrict__ tokens,
    const double *__restrict__ uniforms, int n_uniforms, const RowStats *__restrict__ stats,
    int32_t *__restrict__ path, int32_t *__restrict__ path_len, int64_t *__restrict__ next_token,
    int32_t *__restrict__ uniforms_used, float *__restrict__ residual, int32_t *__restrict__ err,
    const uint32_t *__restrict__ allowed, int n_mw, LazyWalk *__restrict__ lw, int32_t *__restrict__ cur_rows) {
  __shared__ double red[32];
  __shared__ double slots[2];
  __shared__ int s_flag, s_cnt;
  extern __shared__ float2 wlist[];  // kWCap compacted (P, Q) pairs of the current node
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const int b = blockIdx.x / kCl;
  const int n = min(n_rows[b], r_max);
  const int32_t *par = parent + (int64_t)b * r_max;
  const int32_t *tok = tokens + (int64_t)b * r_max;
  const double *uni = uniforms + (int64_t)b * n_uniforms;
  const RowStats *st = stats + (int64_t)b * r_max * 2;
  // this CTA's vocabulary slice (multiple of 4 wide, so 16-byte aligned rows stay aligned)
  const int per = ((vocab + kCl - 1) / kCl + 3) & ~3;
  const int v0 = min(vocab, crank * per), v1 = min(vocab, v0 + per);
  const bool vec = (vocab & 3) == 0 && ((uintptr_t)target & 15) == 0 && ((uintptr_t)draft & 15) == 0;
  int phase = 0;
  double vals[kCl];
  int cur = 0, used = 0, len = 0;
  double c = 0.0, M = 1.0;
  if (kLazy) {
    const LazyWalk s0 = lw[b];
    if (s0.done) return;  // uniform across the cluster: no exchange follows
    cur = s0.cur;
    used = s0.used;
    len = s0.len;
    c = s0.c;
    M = s0.M;
  }
  if (threadIdx.x == 0) {
    s_flag = 0;
    s_cnt = 0;
  }
  __syncthreads();
  if (kLazy) {
    // the visited row (and the q of its children) must be valid
    bool has = false;
    for (int j = cur + 1 + threadIdx.x; j < n; j += kWThreads) has |= par[j] == cur;
    has = __syncthreads_or(has);
    if (threadIdx.x == 0 && (!st[2 * cur].valid || (has && !st[2 * cur + 1].valid))) s_flag = 1;
  } else {
    // any invalid (NaN) row in this sequence aborts it
    for (int r = threadIdx.x; r < n; r += kWThreads)
      if (!st[2 * r].valid) atomicOr(&s_flag, 1);
  }
  __syncthreads();
  if (s_flag) {
    cl.sync();  // uniform across the cluster; lw[b] read by every CTA first
    if (threadIdx.x == 0 && crank == 0) {
      path_len[b] = 0;
      next_token[b] = 0;
      uniforms_used[b] = 0;
      if (kLazy) {
        lw[b].done = 1;
        cur_rows[b] = -1;
      }
    }
    return;
  }
  bool failed = false;
  auto make_row = [&](int r) {
    WalkRow w;
    const RowStats ts = st[2 * r], ds = st[2 * r + 1];
    w.tl = target + ((int64_t)b * r_max + r) * vocab;
    w.dl = ds.valid ? draft + ((int64_t)b * r_max + r) * vocab : nullptr;
    w.p_off = -(ts.m2 + ts.log2_z);
    w.q_off = ds.valid ? -(ds.m2 + ds.log2_z) : 0.f;
    w.keep_all = ts.keep_all;
    w.cut_l = key_to_logit(ts.cut_key);
    w.cut_idx = ts.cut_idx;
    w.mw = kMasked ? allowed + ((int64_t)b * r_max + r) * n_mw : nullptr;
    // this CTA's slices of the node's rows stream into L2 while the
    // (latency-bound) sibling decisions run
    if (vec && threadIdx.x == 0 && v1 > v0) {
      prefetch_l2(w.tl + v0, (uint32_t)(v1 - v0) * 4u);
      if (w.dl) prefetch_l2(w.dl + v0, (uint32_t)(v1 - v0) * 4u);
    }
    return w;
  };
  WalkRow w = make_row(cur);
  int comp = 0;  // 0: no list for this node yet, 1: list valid (cnt pairs), 2: overflowed
  int cnt = 0;
  // children of the current node, a window of kWThreads rows at a time:
  // ordered compaction + every child's p(t), q(t) and uniform fetched in
  // parallel, so the sequential decisions below read shared memory only
  __shared__ int s_wcnt[kWThreads / 32];
  __shared__ int s_child[kWThreads];
  __shared__ float s_pt[kWThreads], s_qt[kWThreads];
  __shared__ double s_u[kWThreads];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    bool descended = false;
    for (int lo = cur + 1; lo < n && !descended && !failed; lo += kWThreads) {
      const int jj = lo + threadIdx.x;
      const bool is_child = jj < n && par[jj] == cur;
      const unsigned bal = __ballot_sync(SDB_FULL_MASK, is_child);
      __syncthreads();  // the previous window's values are consumed
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int off = 0, nch = 0;
#pragma unroll
      for (int q = 0; q < kWThreads / 32; ++q) {
        off += q < warp ? s_wcnt[q] : 0;
        nch += s_wcnt[q];
      }
      if (is_child) {
        const int k = off + __popc(bal & ((1u << lane) - 1u));
        const int t = tok[jj];
        s_child[k] = jj;
        s_pt[k] = p_of(w, a, t);
        s_qt[k] = q_of(w, a, t);
        s_u[k] = used + k < n_uniforms ? uni[used + k] : 0.0;
      }
      __syncthreads();
      for (int k = 0; k < nch; ++k) {
        const int j = s_child[k];
        if (used >= n_uniforms) {
          failed = true;
          break;
        }
        const double u = s_u[k];
        ++used;
        const double pt_full = (double)s_pt[k];
        const double qt = (double)s_qt[k];
        const double pt = fmax(pt_full - c * qt, 0.0) / M;
        const bool acc = qt <= 0.0 ? pt > 0.0 : u < fmin(1.0, pt / qt);
        if (acc) {
          if (threadIdx.x == 0 && crank == 0) path[(int64_t)b * r_max + len] = j - 1;
          ++len;
          cur = j;
          c = 0.0;
          M = 1.0;
          if (kLazy) {  // the next level reduces row j first
            // every CTA of the cluster has read lw[b] (kernel start) and is
            // done with this CTA's exchange slots before lw[b] changes
            cl.sync();
            if (threadIdx.x == 0 && crank == 0) {
              LazyWalk s1;
              s1.c = 0.0;
              s1.M = 1.0;
              s1.cur = j;
              s1.used = used;
              s1.len = len;
              s1.done = 0;
              lw[b] = s1;
              cur_rows[b] = j;
            }
            return;
          }
          w = make_row(cur);
          comp = 0;
          descended = true;
          break;
        }
        // rejection: residual norm(max(p - q, 0)) == max(P - c' Q, 0) / M'
        const double cn = c + M;
        double part;
        if (comp == 0) {
          part = block_sum<kWThreads>(residual_compact(w, a, (float)cn, v0, v1, vec, wlist, &s_cnt), red);
          cnt = s_cnt;  // final: block_sum's barriers follow every append
          comp = cnt <= kWCap ? 1 : 2;
          __syncthreads();
          if (threadIdx.x == 0) s_cnt = 0;  // ordered before the next node's appends by the exchange barrier
        } else if (comp == 1) {
          part = block_sum<kWThreads>(residual_list(wlist, cnt, (float)cn), red);
        } else {
          part = block_sum<kWThreads>(residual_part(w, a, cn, 1.0, v0, v1, vec, nullptr, nullptr), red);
        }
        cluster_exchange<kCl>(part, slots, phase, vals);
        double Mn = 0.0;
#pragma unroll
        for (int q = 0; q < kCl; ++q) Mn += vals[q];
        if (Mn / M <= 1e-12) {
          c = 0.0;  // anchor fallback (sampling.py:193-195)
          M = 1.0;
        } else {
          c = cn;
          M = Mn;
        }
      }
    }
    if (failed || !descended) break;
  }
  if (!failed && used >= n_uniforms) failed = true;
  if (failed) {
    cl.sync();  // (as above: lw[b] read by every CTA, exchange slots free)
    if (threadIdx.x == 0 && crank == 0) {
      atomicOr(err, SDB_ERR_UNIFORMS);
      path_len[b] = len;
      next_token[b] = -1;
      uniforms_used[b] = used;
      if (kLazy) {
        lw[b].done = 1;
        cur_rows[b] = -1;
      }
    }
    return;
  }
  const double u = uni[used++];
  // bonus: inverse CDF of p = max(P - c Q, 0) / M over the vocab in index
  // order (sample_from, sampling.py:105-109): slice masses -> owning CTA.
  float *res_row = residual ? residual + (int64_t)b * vocab : nullptr;
  // the slice's values stay in shared memory (the compaction list is dead)
  // for the owner's inverse CDF
  float *sv = v1 - v0 <= 2 * kWCap ? reinterpret_cast<float *>(wlist) : nullptr;
  __syncthreads();
  const double mine = block_sum<kWThreads>(residual_part(w, a, c, M, v0, v1, vec, res_row, sv), red);
  cluster_exchange<kCl>(mine, slots, phase, vals);
  double base = 0.0, total = 0.0;
  int owner = -1;
#pragma unroll
  for (int q = 0; q < kCl; ++q) {
    if (owner < 0 && total + vals[q] > u) {
      owner = q;
      base = total;
    }
    total += vals[q];
  }
  if (owner < 0 && crank == kCl - 1) {
    if (threadIdx.x == 0) next_token[b] = vocab - 1;
  } else if (owner == crank) {
    // warps own contiguous segments of the slice
    __shared__ double segsum[kWThreads / 32];
    __shared__ double s_prefix;
    __shared__ int s_seg, s_tok;
    // (warp, lane as above)
    constexpr int nw = kWThreads / 32;
    const int seg = (v1 - v0 + nw - 1) / nw;
    const int s0 = v0 + warp * seg, s1 = min(v1, s0 + seg);
    const float cf = (float)c, inv_m = (float)(1.0 / M);
    auto pval = [&](int i) {
      return sv ? (double)sv[i - v0] : (double)(fmaxf(fmaf(-cf, q_of(w, a, i), p_of(w, a, i)), 0.f) * inv_m);
    };
    double wsum = 0.0;
    for (int i = s0 + lane; i < s1; i += 32) wsum += pval(i);
    wsum = warp_sum(wsum);
    if (lane == 0) segsum[warp] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      // searchsorted(cumsum, u, 'right'): first index with cumsum > u
      double cum = base;
      int ws = nw - 1;
      for (int k = 0; k < nw; ++k) {
        if (cum + segsum[k] > u) {
          ws = k;
          break;
        }
        cum += segsum[k];
      }
      s_prefix = cum;  // mass before the chosen segment
      s_seg = ws;
    }
    __syncthreads();
    const int ws = s_seg;
    if (warp == ws) {
      double cum = s_prefix;
      const int a0 = v0 + ws * seg, a1 = min(v1, a0 + seg);
      int found = -1;
      for (int i0 = a0; i0 < a1 && found < 0; i0 += 32) {
        int i = i0 + lane;
        double v = i < a1 ? pval(i) : 0.0;
        double incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          double t = __shfl_up_sync(SDB_FULL_MASK, incl, o);
          if (lane >= o) incl += t;
        }
        unsigned hit = __ballot_sync(SDB_FULL_MASK, i < a1 && cum + incl > u);
        if (hit) found = i0 + __ffs(hit) - 1;
        cum += __shfl_sync(SDB_FULL_MASK, incl, 31);
      }
      if (lane == 0) s_tok = found < 0 ? v1 - 1 : found;
    }
    __syncthreads();
    if (threadIdx.x == 0) next_token[b] = min(s_tok, vocab - 1);
  }
  cl.sync();  // peers may still read this CTA's exchange slots; lw[b] read by all
  if (threadIdx.x == 0 && crank == 0) {
    path_len[b] = len;
    uniforms_used[b] = used;
    if (kLazy) {
      lw[b].done = 1;
      cur_rows[b] = -1;
    }
  }
}

// lazy walk end: a sequence still walking after the planned levels had a
// deeper tree than the host plan (TreeVerifier(tree_levels=) / a captured
// graph): flag it instead of leaving stale outputs
__global__ void lazy_walk_finish_kernel(const LazyWalk *__restrict__ lw, int batch, int32_t *__restrict__ path_len,
                                        int64_t *__restrict__ next_token, int32_t *__restrict__ uniforms_used,
                                        int32_t *__restrict__ err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch || lw[b].done) return;
  path_len[b] = 0;
  next_token[b] = -1;
  uniforms_used[b] = 0;
  atomicOr(err, SDB_ERR_PLAN);
}

// lazy walk start: every sequence at its root row
__global__ void lazy_walk_init_kernel(const int32_t *__restrict__ n_rows, int batch, LazyWalk *__restrict__ lw,
                                      int32_t *__restrict__ cur_rows) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  LazyWalk s;
  s.c = 0.0;
  s.M = 1.0;
  s.cur = 0;
  s.used = 0;
  s.len = 0;
  s.done = n_rows[b] < 1;
  lw[b] = s;
  cur_rows[b] = s.done ? -1 : 0;
}

// Validation scan for the lazy mode: the reference computes target_dist for
// EVERY tree row and the q of every parent row (engine.py:474-475), raising
// on NaN (numcore.py:47-48) or a dead FSM row (sampling.py:96-97) anywhere;
// this streams every such row once (max.NaN) so the error semantics hold
// while the walk only reduces the rows it visits.  HBM-bound, independent
// of the walk: it runs beside it.
template <bool kMasked>
__global__ void __launch_bounds__(kArgmaxThreads) stochastic_validate_kernel(
    const float *__restrict__ target, const float *__restrict__ draft, int r_max, int vocab,
    const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows, const uint32_t *__restrict__ allowed,
    int n_mw, int32_t *__restrict__ err) {
  // one row per CTA, launched at the lowest priority: SMs freed by these
  // short CTAs go to the latency-bound lazy walk's CTAs first
  const int r = blockIdx.x, b = blockIdx.y, z = blockIdx.z;
  const int n = min(n_rows[b], r_max);
  if (r >= n) return;
  if (z) {
    const int32_t *par = parent + (int64_t)b * r_max;
    int has = 0;
    for (int j = r + 1 + threadIdx.x; j < n; j += kArgmaxThreads) has |= par[j] == r;
    if (!__syncthreads_or(has)) return;
  }
  const float *row = (z ? draft : target) + ((int64_t)b * r_max + r) * vocab;
  const uint32_t *mw = kMasked ? allowed + ((int64_t)b * r_max + r) * n_mw : nullptr;
  // NaN only counts at allowed positions (the reference masks first); a
  // masked row needs at least one allowed token
  float nacc = -INFINITY;
  bool any = !kMasked;
  auto one = [&](float x, int j) {
    if (kMasked) {
      if (!((__ldg(mw + (j >> 5)) >> (j & 31)) & 1u)) return;
      any = true;
    }
    nacc = max_nan(nacc, x);
  };
  if ((vocab & 3) == 0 && ((uintptr_t)row & 15) == 0) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    const int n4 = vocab >> 2;
    for (int i0 = 0; i0 < n4; i0 += 4 * kArgmaxThreads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kArgmaxThreads + threadIdx.x;
        v[u] = i < n4 ? __ldcs(r4 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kArgmaxThreads + threadIdx.x;
        if (!kMasked) {
          nacc = max_nan(nacc, max_nan(max_nan3(v[u].x, v[u].y, v[u].z), v[u].w));
        } else if (i < n4) {
          one(v[u].x, 4 * i);
          one(v[u].y, 4 * i + 1);
          one(v[u].z, 4 * i + 2);
          one(v[u].w, 4 * i + 3);
        }
      }
    }
    for (int j = (n4 << 2) + threadIdx.x; j < vocab; j += kArgmaxThreads) one(row[j], j);
  } else {
    for (int j = threadIdx.x; j < vocab; j += kArgmaxThreads) one(row[j], j);
  }
  const bool nan = __syncthreads_or(nacc != nacc);
  const bool alive = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    if (nan) atomicOr(err, SDB_ERR_NAN);
    if (!alive) atomicOr(err, SDB_ERR_NO_ALLOWED);
  }
}

}  // namespace sdb

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
static bool vec_aligned(const void *p, int64_t row_stride, int elem, int vocab) {
  const int lanes = 16 / elem;
  return ((uintptr_t)p % 16 == 0) && (row_stride % lanes == 0) && vocab >= lanes;
}

extern "C" int sdb_argmax_keys(const void *logits, int dtype, int64_t rows, int vocab, int64_t row_stride,
                               int64_t vocab_offset, int64_t *keys, int32_t *err, void *stream) {
  if (!logits || !keys || rows < 0 || vocab < 1 || row_stride < vocab) return SDB_E_INVALID;
  if (vocab_offset < 0 || vocab_offset + vocab > 0xFFFFFFFFll) return SDB_E_INVALID;
  if (rows == 0) return SDB_OK;
  const int64_t gx = rows < 65535 ? rows : 65535;
  const int64_t gy = sdb::cdiv64(rows, gx);
  if (gx * gy != rows) {
    // fall back to a 1-D grid split that tiles exactly
    if (rows > 2147483647ll) return SDB_E_INVALID;
  }
  dim3 grid((unsigned)(gx * gy == rows ? gx : rows), (unsigned)(gx * gy == rows ? gy : 1));
  cudaStream_t s = sdb::as_stream(stream);
  if (dtype == SDB_DTYPE_F32)
    sdb::argmax_keys_kernel<float><<<grid, sdb::kArgmaxThreads, sdb::argmax_smem(), s>>>(
        (const float *)logits, vocab, row_stride, vocab_offset, nullptr, 0, (long long *)keys, err,
        vec_aligned(logits, row_stride, 4, vocab), 1);
  else if (dtype == SDB_DTYPE_BF16)
    sdb::argmax_keys_kernel<__nv_bfloat16><<<grid, sdb::kArgmaxThreads, 0, s>>>(
        (const __nv_bfloat16 *)logits, vocab, row_stride, vocab_offset, nullptr, 0, (long long *)keys, err,
        vec_aligned(logits, row_stride, 2, vocab), 1);
  else
    return SDB_E_UNSUPPORTED;
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_greedy_walk(const int64_t *keys, const int32_t *parent, const int32_t *n_rows,
                               const int32_t *tokens, int batch, int r_max, int32_t *path, int32_t *path_len,
                               int64_t *next_token, int32_t *uniforms_used, void *stream) {
  if (!keys || !parent || !n_rows || !tokens || !path || !path_len || !next_token || !uniforms_used || batch < 0 ||
      r_max < 1)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  sdb::greedy_walk_kernel<<<sdb::cdiv(batch * 32, 128), 128, 0, sdb::as_stream(stream)>>>(
      (const long long *)keys, parent, n_rows, tokens, batch, r_max, path, path_len, next_token, uniforms_used, 1);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_accept_greedy_ex(const float *logits, int batch, int r_max, int vocab, int64_t row_stride,
                                    const int32_t *parent, const int32_t *n_rows, const int32_t *tokens,
                                    const uint32_t *allowed, int allowed_words, int64_t *keys, int32_t *path,
                                    int32_t *path_len, int64_t *next_token, int32_t *uniforms_used, int32_t *err,
                                    void *stream) {
  if (!allowed)
    return sdb_accept_greedy(logits, SDB_DTYPE_F32, batch, r_max, vocab, row_stride, parent, n_rows, tokens, keys,
                             path, path_len, next_token, uniforms_used, err, stream);
  if (!logits || !keys || !parent || !n_rows || !tokens || !err || batch < 0 || r_max < 1 || vocab < 1 ||
      row_stride < vocab || allowed_words < (vocab + 31) / 32)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  cudaStream_t s = sdb::as_stream(stream);
  sdb::argmax_keys_masked_kernel<<<dim3(r_max, batch), sdb::kArgmaxThreads, 0, s>>>(
      logits, vocab, row_stride, n_rows, r_max, allowed, allowed_words, (long long *)keys, err);
  SDB_CHECK_LAUNCH();
  sdb::greedy_walk_kernel<<<sdb::cdiv(batch * 32, 128), 128, 0, s>>>(
      (const long long *)keys, parent, n_rows, tokens, batch, r_max, path, path_len, next_token, uniforms_used, 1);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_accept_greedy(const void *logits, int dtype, int batch, int r_max, int vocab,
                                 int64_t row_stride, const int32_t *parent, const int32_t *n_rows,
                                 const int32_t *tokens, int64_t *keys, int32_t *path, int32_t *path_len,
                                 int64_t *next_token, int32_t *uniforms_used, int32_t *err, void *stream) {
  if (!logits || !keys || !parent || !n_rows || !tokens || batch < 0 || r_max < 1 || vocab < 1 ||
      row_stride < vocab)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  // small batches: cut each row's vocabulary over several CTAs (>= 4096
  // elements each) so that ~4 CTAs per SM stream the logits
  const int64_t rows = (int64_t)batch * r_max;
  int split = (int)std::min<int64_t>(SDB_GREEDY_KEY_SLOTS, std::max<int64_t>(1, (sdb::num_sms() + rows - 1) / rows));
  split = std::max(1, std::min(split, vocab / 16384));
  dim3 grid(r_max * split, batch);
  cudaStream_t s = sdb::as_stream(stream);
  if (dtype == SDB_DTYPE_F32)
    sdb::argmax_keys_kernel<float><<<grid, sdb::kArgmaxThreads, sdb::argmax_smem(), s>>>(
        (const float *)logits, vocab, row_stride, 0, n_rows, r_max, (long long *)keys, err,
        vec_aligned(logits, row_stride, 4, vocab), split);
  else if (dtype == SDB_DTYPE_BF16)
    sdb::argmax_keys_kernel<__nv_bfloat16><<<grid, sdb::kArgmaxThreads, 0, s>>>(
        (const __nv_bfloat16 *)logits, vocab, row_stride, 0, n_rows, r_max, (long long *)keys, err,
        vec_aligned(logits, row_stride, 2, vocab), split);
  else
    return SDB_E_UNSUPPORTED;
  SDB_CHECK_LAUNCH();
  sdb::greedy_walk_kernel<<<sdb::cdiv(batch * 32, 128), 128, 0, s>>>(
      (const long long *)keys, parent, n_rows, tokens, batch, r_max, path, path_len, next_token, uniforms_used, split);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int64_t sdb_accept_stochastic_workspace(int batch, int r_max, int vocab) {
  (void)vocab;
  if (batch < 0 || r_max < 1) return SDB_E_INVALID;
  // RowStats [B][R][2] | LazyWalk [B] | cur_rows [B]
  return (int64_t)batch * r_max * 2 * (int64_t)sizeof(sdb::RowStats) + 256 +
         (int64_t)batch * (int64_t)(sizeof(sdb::LazyWalk) + 4) + 256;
}
extern "C" int sdb_accept_stochastic(const float *target_logits, const float *draft_logits, int batch, int r_max,
                                     int vocab, float temperature, float top_p, const int32_t *parent,
                                     const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                                     int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                                     int32_t *path_len, int64_t *next_token, int32_t *uniforms_used,
                                     float *residual, int32_t *err, void *stream) {
  return sdb_accept_stochastic_ex(target_logits, draft_logits, batch, r_max, vocab, temperature, top_p, parent, n_rows,
                                  tokens, uniforms, n_uniforms, workspace, workspace_bytes, path, path_len,
                                  next_token, uniforms_used, residual, err, nullptr, 0, stream);
}

// co-resident clusters of the walk kernel at cluster size CL (cached per
// process; one device per process)
constexpr int kWalkSmem = sdb::kWCap * (int)sizeof(float2);

template <int CL, bool M, bool L>
static int walk_max_clusters_of() {
  // the smem opt-in is per device: set on every call (cheap); the occupancy
  // query is cached per device
  cudaFuncSetAttribute(sdb::stochastic_walk_kernel<CL, M, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWalkSmem);
  static int cached_per_dev[64] = {0};  // 0: not queried yet (stored + 1)
  int dev = 0;
  cudaGetDevice(&dev);
  int &cached = cached_per_dev[dev & 63];
  if (cached == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * 1024);
    cfg.blockDim = dim3(sdb::kWThreads);
    cfg.dynamicSmemBytes = kWalkSmem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = CL;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, sdb::stochastic_walk_kernel<CL, M, L>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = sdb::num_sms() / CL;
    }
    cached = n + 1;
  }
  return cached - 1;
}

template <int CL>
static int walk_max_clusters(bool lazy, bool masked) {
  if (lazy) return masked ? walk_max_clusters_of<CL, true, true>() : walk_max_clusters_of<CL, false, true>();
  return masked ? walk_max_clusters_of<CL, true, false>() : walk_max_clusters_of<CL, false, false>();
}

static int accept_stochastic_impl(const float *target_logits, const float *draft_logits, int batch, int r_max,
                                  int vocab, float temperature, float top_p, const int32_t *parent,
                                  const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                                  int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                                  int32_t *path_len, int64_t *next_token, int32_t *uniforms_used, float *residual,
                                  int32_t *err, const uint32_t *allowed, int allowed_words, int levels,
                                  void *stream) {
  if (allowed && allowed_words < (vocab + 31) / 32) return SDB_E_INVALID;
  if (!target_logits || !draft_logits || !parent || !n_rows || !tokens || !uniforms || !path || !path_len ||
      !next_token || !uniforms_used || !err || batch < 0 || r_max < 1 || vocab < 1 || n_uniforms < 0 ||
      levels > r_max)
    return SDB_E_INVALID;
  if (!(temperature > 0.0f) || !(top_p > 0.0f) || top_p > 1.0f) return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  if (!workspace || workspace_bytes < sdb_accept_stochastic_workspace(batch, r_max, vocab)) return SDB_E_WORKSPACE;
  const float a = 1.4426950408889634f / temperature;
  sdb::RowStats *stats = reinterpret_cast<sdb::RowStats *>(workspace);
  char *tail = (char *)workspace + (((int64_t)batch * r_max * 2 * (int64_t)sizeof(sdb::RowStats) + 255) & ~255ll);
  sdb::LazyWalk *lw = reinterpret_cast<sdb::LazyWalk *>(tail);
  int32_t *cur_rows = reinterpret_cast<int32_t *>(tail + (((int64_t)batch * sizeof(sdb::LazyWalk) + 15) & ~15ll));
  const bool lazy = levels > 0;
  cudaStream_t s = sdb::as_stream(stream);
  const size_t smem = sizeof(sdb::StSmem);
  cudaFuncSetAttribute(sdb::row_stats_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sdb::row_stats_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sdb::row_stats_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sdb::row_stats_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sdb::row_stats_kernel<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sdb::row_stats_kernel<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // lazy chain: each visited row split over a cluster of st_split CTAs
  // (16-byte aligned rows; SDB_ST_SPLIT = 1 keeps one CTA per row).
  // Measured (tools/cycles/r2_st_split.sh, same box): C5 943 / 910 / 1028 us,
  // C3 stochastic 1191 / 1155 / 1184 us, the C5 chain alone 550 / 516 / 633
  // at 1 / 2 / 4 CTAs per row (4: the first levels' rows need 3.5 waves)
  static int st_split = -1;
  if (st_split < 0) {
    const char *e = getenv("SDB_ST_SPLIT");
    st_split = e ? atoi(e) : 2;
    if (st_split != 2 && st_split != 4) st_split = 1;
  }
  const bool split_rows = lazy && st_split > 1 && (vocab % 4) == 0 && ((uintptr_t)target_logits % 16) == 0 &&
                          ((uintptr_t)draft_logits % 16) == 0;
  // cluster size: the widest (8 = portable maximum) whose clusters for the
  // whole batch fit in two waves -- a wider cluster halves every CTA's
  // full-slice passes, which costs more than a second wave of early-exiting
  // clusters (C5, B 64: 0.94 ms at 8 wide vs 1.18 ms at 4 wide, one wave)
  const int mc8 = walk_max_clusters<8>(lazy, allowed != nullptr);
  const int mc4 = walk_max_clusters<4>(lazy, allowed != nullptr);
  (void)walk_max_clusters<2>(lazy, allowed != nullptr);  // (sets the smem attribute)
  int ncl = batch <= 2 * mc8 ? 8 : batch <= 2 * mc4 ? 4 : 2;
  if (const char *e = getenv("SDB_WALK_CL")) {  // experiments
    const int v = atoi(e);
    if (v == 2 || v == 4 || v == 8) ncl = v;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch * ncl);
  cfg.blockDim = dim3(sdb::kWThreads);
  cfg.dynamicSmemBytes = kWalkSmem;
  cfg.stream = s;
  // lazy mode: the walk's launches at the highest priority (a validation
  // scan may be streaming beside them at the lowest)
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = greatest;
  cfg.attrs = attr;
  cfg.numAttrs = lazy ? 2 : 1;
  cudaLaunchConfig_t scfg = {};
  scfg.blockDim = dim3(sdb::kStThreads);
  scfg.dynamicSmemBytes = smem;
  scfg.stream = s;
  scfg.attrs = &attr[1];
  scfg.numAttrs = lazy ? 1 : 0;
  cudaLaunchAttribute sattr[2];
  sattr[0] = attr[1];  // priority
  sattr[1].id = cudaLaunchAttributeClusterDimension;
  sattr[1].val.clusterDim.x = st_split > 1 ? st_split : 2;
  sattr[1].val.clusterDim.y = 1;
  sattr[1].val.clusterDim.z = 1;
  // the first level (every sequence at its root: 2 B rows) without the row
  // split when its 4 B split CTAs would need more than two waves of the SMs
  // the concurrent validation scan leaves (52 of 148 taken): C5 (B 64) 587 ->
  // 578 us; C3 stochastic (B 32) keeps the split (956 vs 973 us without).
  // SDB_ST_SPLIT0 = 1 / 2 forces it.
  static const int split_lvl0_env = [] {
    const char *e = getenv("SDB_ST_SPLIT0");
    return e ? atoi(e) : 0;
  }();
  int n_sms_dev = 148, dev_id = 0;
  cudaGetDevice(&dev_id);
  cudaDeviceGetAttribute(&n_sms_dev, cudaDevAttrMultiProcessorCount, dev_id);
  const int free_sms = n_sms_dev - (n_sms_dev * sdb::kValSmsPer148 + 74) / 148;
  const int split_lvl0 = split_lvl0_env ? split_lvl0_env : (4 * batch > 2 * free_sms ? 1 : 2);
  auto stats_launch = [&](dim3 grid, const int32_t *rows, bool split_ok = true) {
    scfg.gridDim = grid;
    if (rows && split_rows && split_ok) {
      scfg.gridDim.x = st_split * grid.x;
      scfg.attrs = sattr;
      scfg.numAttrs = 2;
#define SDB_ST_LAUNCH(CS)                                                                                          \
  (allowed ? cudaLaunchKernelEx(&scfg, sdb::row_stats_kernel<true, CS>, target_logits, draft_logits, r_max, vocab, a, \
                                top_p, parent, n_rows, stats, err, allowed, allowed_words, rows)                       \
           : cudaLaunchKernelEx(&scfg, sdb::row_stats_kernel<false, CS>, target_logits, draft_logits, r_max, vocab,   \
                                a, top_p, parent, n_rows, stats, err, (const uint32_t *)nullptr, 0, rows))
      if (st_split == 4)
        SDB_ST_LAUNCH(4);
      else
        SDB_ST_LAUNCH(2);
#undef SDB_ST_LAUNCH
      scfg.attrs = &attr[1];
      scfg.numAttrs = lazy ? 1 : 0;
      return;
    }
    if (allowed)
      cudaLaunchKernelEx(&scfg, sdb::row_stats_kernel<true, 1>, target_logits, draft_logits, r_max, vocab, a, top_p,
                         parent, n_rows, stats, err, allowed, allowed_words, rows);
    else
      cudaLaunchKernelEx(&scfg, sdb::row_stats_kernel<false, 1>, target_logits, draft_logits, r_max, vocab, a, top_p,
                         parent, n_rows, stats, err, (const uint32_t *)nullptr, 0, rows);
  };
#define SDB_WALK(CL, M, L)                                                                                        \
  cudaLaunchKernelEx(&cfg, sdb::stochastic_walk_kernel<CL, M, L>, target_logits, draft_logits, r_max, vocab, a,    \
                     parent, n_rows, tokens, uniforms, n_uniforms, (const sdb::RowStats *)stats, path, path_len,  \
                     next_token, uniforms_used, residual, err, allowed, allowed_words, lw, cur_rows)
  auto walk_launch = [&]() {
    if (lazy) {
      if (ncl == 2) return allowed ? SDB_WALK(2, true, true) : SDB_WALK(2, false, true);
      if (ncl == 4) return allowed ? SDB_WALK(4, true, true) : SDB_WALK(4, false, true);
      return allowed ? SDB_WALK(8, true, true) : SDB_WALK(8, false, true);
    }
    if (ncl == 2) return allowed ? SDB_WALK(2, true, false) : SDB_WALK(2, false, false);
    if (ncl == 4) return allowed ? SDB_WALK(4, true, false) : SDB_WALK(4, false, false);
    return allowed ? SDB_WALK(8, true, false) : SDB_WALK(8, false, false);
  };
#undef SDB_WALK
  if (!lazy) {
    stats_launch(dim3(r_max, batch, 2), nullptr);
    SDB_CHECK_LAUNCH();
    cudaError_t le = walk_launch();
    if (le != cudaSuccess) return sdb::record_cuda_error(le);
    SDB_CHECK_LAUNCH();
    return SDB_OK;
  }
  // lazy: one level per (row stats of the current rows, walk step) pair
  sdb::lazy_walk_init_kernel<<<(batch + 127) / 128, 128, 0, s>>>(n_rows, batch, lw, cur_rows);
  SDB_CHECK_LAUNCH();
  for (int lvl = 0; lvl < levels; ++lvl) {
    stats_launch(dim3(1, batch, 2), cur_rows, lvl > 0 || split_lvl0 > 1);
    SDB_CHECK_LAUNCH();
    cudaError_t le = walk_launch();
    if (le != cudaSuccess) return sdb::record_cuda_error(le);
    SDB_CHECK_LAUNCH();
  }
  sdb::lazy_walk_finish_kernel<<<(batch + 127) / 128, 128, 0, s>>>(lw, batch, path_len, next_token, uniforms_used,
                                                                   err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_accept_stochastic_ex(const float *target_logits, const float *draft_logits, int batch, int r_max,
                                        int vocab, float temperature, float top_p, const int32_t *parent,
                                        const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                                        int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                                        int32_t *path_len, int64_t *next_token, int32_t *uniforms_used,
                                        float *residual, int32_t *err, const uint32_t *allowed, int allowed_words,
                                        void *stream) {
  return accept_stochastic_impl(target_logits, draft_logits, batch, r_max, vocab, temperature, top_p, parent, n_rows,
                                tokens, uniforms, n_uniforms, workspace, workspace_bytes, path, path_len, next_token,
                                uniforms_used, residual, err, allowed, allowed_words, 0, stream);
}

extern "C" int sdb_accept_stochastic_lazy(const float *target_logits, const float *draft_logits, int batch, int r_max,
                                          int vocab, float temperature, float top_p, const int32_t *parent,
                                          const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                                          int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                                          int32_t *path_len, int64_t *next_token, int32_t *uniforms_used,
                                          float *residual, int32_t *err, const uint32_t *allowed, int allowed_words,
                                          int levels, void *stream) {
  if (levels < 1) return SDB_E_INVALID;
  return accept_stochastic_impl(target_logits, draft_logits, batch, r_max, vocab, temperature, top_p, parent, n_rows,
                                tokens, uniforms, n_uniforms, workspace, workspace_bytes, path, path_len, next_token,
                                uniforms_used, residual, err, allowed, allowed_words, levels, stream);
}

namespace sdb {
// Persistent variant of the validation scan (unmasked rows): K CTAs, one
// per SM (the dynamic shared memory request keeps every other CTA off those
// SMs), each streaming its rows as one flat sequence with 8 x 16-byte loads
// per thread in flight (128 KB per SM; ncu alone on 56 SMs: 523 us for
// 2.99 GB = 5.7 TB/s, 102 GB/s per SM -- 579 us with a per-row loop).  The scan then owns K SMs for the whole walk and
// the latency-bound lazy chain runs on the other 148 - K without waiting for
// scan CTAs to drain (a spatial split instead of priorities).
constexpr int kValUnroll = 8;  // (12 measured the same)
constexpr int kValSmem = 150 * 1024;
constexpr int kValFlagBytes = 96 * 1024;                         // has-child flags of up to 96 K (sequence, row) pairs
constexpr int kValListMax = (kValSmem - kValFlagBytes) / 8;      // row pointers of this CTA's listed rows
__global__ void __launch_bounds__(kArgmaxThreads, 1) stochastic_validate_persistent_kernel(
    const float *__restrict__ target, const float *__restrict__ draft, int batch, int r_max, int vocab,
    const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows, int32_t *__restrict__ err) {
  // this CTA's rows (w = blockIdx.x + k * gridDim.x over [target rows |
  // draft rows]) that the reference reads -- target rows r < n_rows[b],
  // draft rows with a child -- are listed in shared memory first, then
  // streamed as ONE flat sequence of 16-byte words, so the loads in flight
  // never drain at a row boundary (per-row loops lost ~25 % of the SM's
  // rate: ncu 5.17 TB/s on 56 SMs vs 6.9 TB/s for a flat stream)
  extern __shared__ __align__(16) unsigned char vsm[];
  const int br_total = batch * r_max, total = 2 * br_total;
  const bool vec = (vocab & 3) == 0 && ((uintptr_t)target & 15) == 0 && ((uintptr_t)draft & 15) == 0;
  const int n_cand = total > (int)blockIdx.x ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const bool listed = vec && br_total <= kValFlagBytes && n_cand <= kValListMax;
  float nacc = -INFINITY;
  if (listed) {
    uint8_t *has_child = vsm;                                                    // [batch * r_max]
    const float4 **list = reinterpret_cast<const float4 **>(vsm + kValFlagBytes);  // [<= kValListMax]
    __shared__ int n_list;
    for (int j = threadIdx.x; j < br_total; j += kArgmaxThreads) has_child[j] = 0;
    if (threadIdx.x == 0) n_list = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < br_total; j += kArgmaxThreads) {
      const int b = j / r_max, r = j % r_max;
      const int pr = parent[j];
      if (r < min(n_rows[b], r_max) && pr >= 0 && pr < r) has_child[b * r_max + pr] = 1;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_cand; t += kArgmaxThreads) {
      const int w = (int)blockIdx.x + t * (int)gridDim.x;
      const int z = w / br_total, br = w % br_total, b = br / r_max, r = br % r_max;
      const bool active = r < min(n_rows[b], r_max) && (z == 0 || has_child[br]);
      if (active) list[atomicAdd(&n_list, 1)] = reinterpret_cast<const float4 *>((z ? draft : target) + (int64_t)br * vocab);
    }
    __syncthreads();
    const int nl = n_list;
    const int n4 = vocab >> 2;
    // this thread's flat position: row li, word off (advanced by 1024 per load)
    int li = 0, off = threadIdx.x;
    while (off >= n4 && li < nl) { off -= n4; ++li; }
    while (li < nl) {
      float4 v[kValUnroll];
#pragma unroll
      for (int u = 0; u < kValUnroll; ++u) {
        v[u] = li < nl ? __ldcs(list[li] + off) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        off += kArgmaxThreads;
        while (off >= n4 && li < nl) { off -= n4; ++li; }
      }
#pragma unroll
      for (int u = 0; u < kValUnroll; ++u) nacc = max_nan(nacc, max_nan(max_nan3(v[u].x, v[u].y, v[u].z), v[u].w));
    }
  } else {
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const int z = w / br_total, br = w % br_total, b = br / r_max, r = br % r_max;
      const int n = min(n_rows[b], r_max);
      if (r >= n) continue;
      if (z) {
        const int32_t *par = parent + (int64_t)b * r_max;
        int has = 0;
        for (int j = r + 1 + threadIdx.x; j < n; j += kArgmaxThreads) has |= par[j] == r;
        if (!__syncthreads_or(has)) continue;
      }
      const float *row = (z ? draft : target) + (int64_t)br * vocab;
      for (int j = threadIdx.x; j < vocab; j += kArgmaxThreads) nacc = max_nan(nacc, row[j]);
    }
  }
  if (__syncthreads_or(nacc != nacc) && threadIdx.x == 0) atomicOr(err, SDB_ERR_NAN);
}
}  // namespace sdb

extern "C" int sdb_stochastic_validate(const float *target_logits, const float *draft_logits, int batch, int r_max,
                                       int vocab, const int32_t *parent, const int32_t *n_rows,
                                       const uint32_t *allowed, int allowed_words, int32_t *err, void *stream) {
  if (!target_logits || !draft_logits || !parent || !n_rows || !err || batch < 0 || r_max < 1 || vocab < 1 ||
      (allowed && allowed_words < (vocab + 31) / 32))
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  // default: the persistent scan on 52 of 148 SMs (scaled to the device),
  // the lazy chain on the rest -- C5 912 -> ~570 us, C3 stochastic 1142 ->
  // ~960 us.  K swept 36..62 on the flat-stream scan (same box, C5 us):
  // 38 703, 42 644, 44 624, 46 603, 48 685 (the chain's clusters place
  // badly), 50 586, 52 593, 54 616, 56 609-618, 60 633; with the unsplit
  // first level: 46 603, 50 578, 52 565-572, 54 592-599, 58 600-606; flat
  // at B <= 32.
  // SDB_VALIDATE_SMS=0 restores the one-row low-priority CTAs
  static const int persist_env = [] {
    const char *e = getenv("SDB_VALIDATE_SMS");
    return e ? atoi(e) : -1;
  }();
  int persist_sms = persist_env;
  if (persist_sms < 0) {
    int dev = 0, n_sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
    persist_sms = (n_sms * sdb::kValSmsPer148 + 74) / 148;
  }
  if (persist_sms > 0 && !allowed) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(sdb::stochastic_validate_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           sdb::kValSmem);
      attr_set = true;
    }
    sdb::stochastic_validate_persistent_kernel<<<persist_sms, sdb::kArgmaxThreads, sdb::kValSmem,
                                                 sdb::as_stream(stream)>>>(target_logits, draft_logits, batch, r_max,
                                                                           vocab, parent, n_rows, err);
    SDB_CHECK_LAUNCH();
    return SDB_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(r_max, batch, 2);
  cfg.blockDim = dim3(sdb::kArgmaxThreads);
  cfg.stream = sdb::as_stream(stream);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributePriority;
  attr.val.priority = least;  // below the lazy walk's launches
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaError_t le =
      allowed ? cudaLaunchKernelEx(&cfg, sdb::stochastic_validate_kernel<true>, target_logits, draft_logits, r_max,
                                   vocab, parent, n_rows, allowed, allowed_words, err)
              : cudaLaunchKernelEx(&cfg, sdb::stochastic_validate_kernel<false>, target_logits, draft_logits, r_max,
                                   vocab, parent, n_rows, (const uint32_t *)nullptr, 0, err);
  if (le != cudaSuccess) return sdb::record_cuda_error(le);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

#ifdef SDB_TRACE
extern "C" int sdb_debug_st_trace(unsigned long long *host_out, unsigned int *count) {
  if (cudaMemcpyFromSymbol(host_out, sdb::g_st_trace, sizeof(sdb::g_st_trace)) != cudaSuccess) return -4;
  return cudaMemcpyFromSymbol(count, sdb::g_st_launch, sizeof(unsigned int)) == cudaSuccess ? 0 : -4;
}
#endif
