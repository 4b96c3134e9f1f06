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
#include <math.h>

#include "accept_common.cuh"

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
    // 4 independent 16-byte loads in flight per thread
    for (; i + 3 * kArgmaxThreads < n4; i += 4 * kArgmaxThreads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(r4 + i + u * kArgmaxThreads);
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
      const float4 v = __ldcs(r4 + i);
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
      const uint4 v = __ldcs(r8 + i);
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

// grid.x = rows (flat) or (r_max, batch) with n_rows gating.
template <typename T>
__global__ void __launch_bounds__(kArgmaxThreads, 2) argmax_keys_kernel(const T *__restrict__ logits, int vocab,
                                                                     int64_t row_stride, int64_t vocab_offset,
                                                                     const int32_t *__restrict__ n_rows,
                                                                     int r_max, long long *__restrict__ keys,
                                                                     int32_t *__restrict__ err, bool vec_ok) {
  __shared__ long long red[kArgmaxThreads / 32];
  int64_t row;
  if (n_rows) {
    const int r = blockIdx.x, b = blockIdx.y;
    if (r >= n_rows[b]) return;
    row = (int64_t)b * r_max + r;
  } else {
    row = blockIdx.x + (int64_t)blockIdx.y * gridDim.x;
  }
  long long best = LLONG_MIN;
  bool nan = false;
  argmax_row<T>(logits + row * row_stride, vocab, vocab_offset, vec_ok, best, nan);
  best = block_max_i64<kArgmaxThreads>(best, red);
  if (__syncthreads_or(nan) && threadIdx.x == 0 && err) atomicOr(err, SDB_ERR_NAN);
  if (threadIdx.x == 0) keys[row] = best;
}

// One warp per sequence: the argmax walk in the augmented frame (row 0 =
// root; children of row r = rows j > r with parent[j] == r, index order).
__global__ void greedy_walk_kernel(const long long *__restrict__ keys, const int32_t *__restrict__ parent,
                                   const int32_t *__restrict__ n_rows, const int32_t *__restrict__ tokens,
                                   int batch, int r_max, int32_t *__restrict__ path, int32_t *__restrict__ path_len,
                                   int64_t *__restrict__ next_token, int32_t *__restrict__ uniforms_used) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= batch) return;
  const int n = min(n_rows[b], r_max);
  const int32_t *par = parent + (int64_t)b * r_max;
  const int32_t *tok = tokens + (int64_t)b * r_max;
  const long long *key = keys + (int64_t)b * r_max;
  int cur = 0, used = 0, len = 0;
  while (true) {
    const int want = (int)key_index(key[cur]);
    int accepted = -1, examined = 0;
    for (int j0 = cur + 1; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool child = j < n && par[j] == cur;
      const bool hit = child && tok[j] == want;
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
    next_token[b] = (int64_t)key_index(key[cur]);
    uniforms_used[b] = used + 1;
  }
}

// ---------------------------------------------------------------------------
// stochastic
// ---------------------------------------------------------------------------
constexpr int kStThreads = 1024;
constexpr int kHistBins = 1024;        // width 1/16 log2 unit below the row max
constexpr float kHistScale = 16.0f;
constexpr int kHistCopies = 16;        // warp-pair private histograms
constexpr int kCandCap = 4096;         // exact-sort capacity around the cut


__device__ __forceinline__ int hist_bin(float x2, float m2) {
  float d = (m2 - x2) * kHistScale;
  return d >= (float)(kHistBins - 1) ? kHistBins - 1 : (int)d;
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
  float hist[kHistCopies][kHistBins];
  unsigned long long cand[kCandCap];
  double red[32];
  float redf[32];
  double cum[kHistBins];
  int count;
  int pad[3];
};

// Phase A.  grid (r_max, batch, 2): z = 0 target rows (nucleus), z = 1 draft
// rows that have children (full softmax).
__global__ void __launch_bounds__(kStThreads, 1) row_stats_kernel(
    const float *__restrict__ target, const float *__restrict__ draft, int r_max, int vocab, float a,
    float top_p, const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows,
    RowStats *__restrict__ stats, int32_t *__restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StSmem &sm = *reinterpret_cast<StSmem *>(smem_raw);
  const int r = blockIdx.x, b = blockIdx.y, is_draft = blockIdx.z;
  const int n = min(n_rows[b], r_max);
  RowStats *out = stats + ((int64_t)b * r_max + r) * 2 + is_draft;
  if (r >= n) {
    if (threadIdx.x == 0) out->valid = 0;
    return;
  }
  if (is_draft) {
    // only parent rows carry a q (their children's proposal distribution)
    const int32_t *par = parent + (int64_t)b * r_max;
    int has = 0;
    for (int j = r + 1 + threadIdx.x; j < n; j += kStThreads) has |= par[j] == r;
    if (!__syncthreads_or(has)) {
      if (threadIdx.x == 0) out->valid = 0;
      return;
    }
  }
  const float *row = (is_draft ? draft : target) + ((int64_t)b * r_max + r) * vocab;
  const bool vec = (vocab & 3) == 0 && ((uintptr_t)row & 15) == 0;
  // pass 1: max + NaN
  float mx = -INFINITY;
  bool nan = false;
  if (vec) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    for (int i = threadIdx.x; i < (vocab >> 2); i += kStThreads) {
      float4 v = r4[i];
      nan |= (v.x != v.x) | (v.y != v.y) | (v.z != v.z) | (v.w != v.w);
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
  } else {
    for (int i = threadIdx.x; i < vocab; i += kStThreads) {
      float v = row[i];
      nan |= v != v;
      mx = fmaxf(mx, v);
    }
  }
  if (__syncthreads_or(nan)) {
    if (threadIdx.x == 0) {
      atomicOr(err, SDB_ERR_NAN);
      out->valid = 0;
    }
    return;
  }
  mx = block_max<kStThreads>(mx, sm.redf);
  const float m2 = mx * a;
  const bool nucleus = !is_draft && top_p < 1.0f;
  // pass 2: normaliser (+ value histogram for nucleus rows)
  if (nucleus) {
    for (int i = threadIdx.x; i < kHistCopies * kHistBins; i += kStThreads) (&sm.hist[0][0])[i] = 0.f;
    __syncthreads();
  }
  float *hist = sm.hist[(threadIdx.x >> 6) % kHistCopies];
  float s_loc = 0.f;
  for (int i = threadIdx.x; i < vocab; i += kStThreads) {
    float x2 = row[i] * a;
    float w = exp2f(x2 - m2);
    s_loc += w;
    if (nucleus) atomicAdd(&hist[hist_bin(x2, m2)], w);
  }
  const double s = block_sum<kStThreads>((double)s_loc, sm.red);
  if (!nucleus) {
    if (threadIdx.x == 0) {
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
  // cumulative mass by bin (bin 0 = largest values)
  for (int bb = threadIdx.x; bb < kHistBins; bb += kStThreads) {
    float t = 0.f;
#pragma unroll
    for (int c = 0; c < kHistCopies; ++c) t += sm.hist[c][bb];
    sm.cum[bb] = t;
  }
  __syncthreads();
  double cv = block_inclusive_scan(threadIdx.x < kHistBins ? sm.cum[threadIdx.x] : 0.0, sm.red);
  if (threadIdx.x < kHistBins) sm.cum[threadIdx.x] = cv;  // inclusive
  __syncthreads();
  const double tau = ((double)top_p - 1e-12) * s;
  // window of bins whose inclusive cumulative could straddle tau given fp32
  // bin sums (relative error << 1e-5)
  int lo = kHistBins - 1, hi = kHistBins - 1;
  {
    // first bin with cum >= threshold: parallel min over bins
    __shared__ int s_lo, s_hi;
    if (threadIdx.x == 0) {
      s_lo = kHistBins - 1;
      s_hi = kHistBins - 1;
    }
    __syncthreads();
    for (int bb = threadIdx.x; bb < kHistBins; bb += kStThreads) {
      if (sm.cum[bb] >= tau * (1.0 - 1e-5)) atomicMin(&s_lo, bb);
      if (sm.cum[bb] >= tau * (1.0 + 1e-5)) atomicMin(&s_hi, bb);
    }
    __syncthreads();
    lo = s_lo;
    hi = max(s_hi, lo);
  }
  double mass_above = lo > 0 ? sm.cum[lo - 1] : 0.0;
  // pass 3+: collect the window [key range]; refine in key space until the
  // candidates fit the exact-sort buffer or only ties remain.
  uint32_t klo = 0xffffffffu, khi = 0u;
  {
    uint32_t kl = 0xffffffffu, kh = 0u;
    for (int i = threadIdx.x; i < vocab; i += kStThreads) {
      float l = row[i];
      int bin = hist_bin(l * a, m2);
      if (bin >= lo && bin <= hi) {
        uint32_t k = orderable_u32(l);
        kl = min(kl, k);
        kh = max(kh, k);
      }
    }
    // block min/max through the float reducer reinterpreted as unsigned
    __shared__ unsigned s_kl, s_kh;
    if (threadIdx.x == 0) {
      s_kl = 0xffffffffu;
      s_kh = 0u;
    }
    __syncthreads();
    atomicMin(&s_kl, kl);
    atomicMax(&s_kh, kh);
    __syncthreads();
    klo = s_kl;
    khi = s_kh;
  }
  uint32_t cut_key = 0;
  int cut_idx = -1;
  double z = 0.0;
  for (int level = 0; level < 8; ++level) {
    if (threadIdx.x == 0) sm.count = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < vocab; i += kStThreads) {
      uint32_t k = orderable_u32(row[i]);
      if (k >= klo && k <= khi) {
        int slot = atomicAdd(&sm.count, 1);
        if (slot < kCandCap) sm.cand[slot] = ((unsigned long long)k << 32) | (0xffffffffu - (uint32_t)i);
      }
    }
    __syncthreads();
    const int count = sm.count;
    if (count <= kCandCap) {
      // exact: sort descending by (key, -index), scan masses from mass_above
      int np2 = 1;
      while (np2 < count) np2 <<= 1;
      for (int i = count + threadIdx.x; i < np2; i += kStThreads) sm.cand[i] = 0ull;
      __syncthreads();
      for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int i = threadIdx.x; i < np2; i += kStThreads) {
            int j = i ^ stride;
            if (j > i) {
              bool desc = (i & size) == 0;
              unsigned long long x = sm.cand[i], y = sm.cand[j];
              if (desc ? (x < y) : (x > y)) {
                sm.cand[i] = y;
                sm.cand[j] = x;
              }
            }
          }
          __syncthreads();
        }
      }
      // per-thread chunk of 4 consecutive sorted candidates
      double loc[4];
      double tot = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = threadIdx.x * 4 + u;
        double w = 0.0;
        if (i < count) {
          uint32_t k = (uint32_t)(sm.cand[i] >> 32);
          uint32_t bits = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
          w = (double)exp2f(__uint_as_float(bits) * a - m2);
        }
        tot += w;
        loc[u] = tot;
      }
      double incl = block_inclusive_scan(tot, sm.red);
      double base = mass_above + incl - tot;
      __shared__ int s_cut;
      if (threadIdx.x == 0) s_cut = count - 1;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = threadIdx.x * 4 + u;
        if (i < count && base + loc[u] >= tau) atomicMin(&s_cut, i);
      }
      __syncthreads();
      const int cpos = s_cut;
      // kept mass = mass_above + candidates[0..cpos]
      double zz = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = threadIdx.x * 4 + u;
        if (i <= cpos && i < count) {
          uint32_t k = (uint32_t)(sm.cand[i] >> 32);
          uint32_t bits = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
          zz += (double)exp2f(__uint_as_float(bits) * a - m2);
        }
      }
      z = mass_above + block_sum<kStThreads>(zz, sm.red);
      if (count > 0) {
        cut_key = (uint32_t)(sm.cand[cpos] >> 32);
        cut_idx = (int)(0xffffffffu - (uint32_t)(sm.cand[cpos] & 0xffffffffu));
      } else {
        // empty window: everything above is kept
        cut_key = khi;
        cut_idx = INT_MAX;
        z = mass_above;
      }
      break;
    }
    if (klo == khi) {
      // only ties remain: all candidates share the weight w*; the first j by
      // index are kept, j = ceil((tau - mass_above) / w*)
      uint32_t bits = (klo & 0x80000000u) ? (klo & 0x7fffffffu) : ~klo;
      double w = (double)exp2f(__uint_as_float(bits) * a - m2);
      long long need = (long long)ceil((tau - mass_above) / w);
      need = need < 1 ? 1 : (need > count ? count : need);
      // index of the need-th tied element in index order: chunked prefix count
      __shared__ int s_idx;
      __shared__ double s_tot;
      if (threadIdx.x == 0) s_idx = vocab - 1;
      __syncthreads();
      long long seen = 0;
      for (int c0 = 0; c0 < vocab; c0 += kStThreads) {
        int i = c0 + threadIdx.x;
        bool t = i < vocab && orderable_u32(row[i]) == klo;
        double pre = block_inclusive_scan(t ? 1.0 : 0.0, sm.red);
        if (t && seen + (long long)pre == need) s_idx = i;
        if (threadIdx.x == kStThreads - 1) s_tot = pre;
        __syncthreads();
        seen += (long long)s_tot;
        __syncthreads();
        if (seen >= need) break;
      }
      __syncthreads();
      cut_key = klo;
      cut_idx = s_idx;
      z = mass_above + w * (double)need;
      break;
    }
    // refine: 1024 sub-ranges of [klo, khi] by key (bin 0 = highest keys)
    for (int i = threadIdx.x; i < kHistBins; i += kStThreads) sm.hist[0][i] = 0.f;
    __syncthreads();
    const unsigned long long span = (unsigned long long)(khi - klo) + 1ull;
    for (int i = threadIdx.x; i < vocab; i += kStThreads) {
      float l = row[i];
      uint32_t k = orderable_u32(l);
      if (k >= klo && k <= khi) {
        int bin = (int)(((unsigned long long)(khi - k) * kHistBins) / span);
        atomicAdd(&sm.hist[0][bin], exp2f(l * a - m2));
      }
    }
    __syncthreads();
    double c2 = block_inclusive_scan(threadIdx.x < kHistBins ? (double)sm.hist[0][threadIdx.x] : 0.0, sm.red);
    if (threadIdx.x < kHistBins) sm.cum[threadIdx.x] = mass_above + c2;
    __syncthreads();
    __shared__ int s_lo2, s_hi2;
    if (threadIdx.x == 0) {
      s_lo2 = kHistBins - 1;
      s_hi2 = kHistBins - 1;
    }
    __syncthreads();
    for (int bb = threadIdx.x; bb < kHistBins; bb += kStThreads) {
      if (sm.cum[bb] >= tau * (1.0 - 1e-5)) atomicMin(&s_lo2, bb);
      if (sm.cum[bb] >= tau * (1.0 + 1e-5)) atomicMin(&s_hi2, bb);
    }
    __syncthreads();
    const int blo = s_lo2, bhi = max(s_hi2, s_lo2);
    mass_above = blo > 0 ? sm.cum[blo - 1] : mass_above;
    // key range of bins [blo, bhi]: bin(k) = floor((khi - k) * B / span)
    const uint32_t nkhi = khi - (uint32_t)(((unsigned long long)blo * span + kHistBins - 1) / kHistBins);
    const uint32_t nklo_off = (uint32_t)((((unsigned long long)(bhi + 1)) * span + kHistBins - 1) / kHistBins) - 1u;
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

// p_k(t) = max(P(t) - c Q(t), 0) / M at row `cur` (Q from draft row cur).
struct WalkRow {
  const float *tl;  // target logits row
  const float *dl;  // draft logits row (nullptr when cur has no children)
  RowStats ts, ds;
};

__device__ __forceinline__ float p_of(const WalkRow &w, float a, int t) {
  float l = w.tl[t];
  return kept(w.ts, l, t) ? exp2f(l * a - w.ts.m2 - w.ts.log2_z) : 0.f;
}
__device__ __forceinline__ float q_of(const WalkRow &w, float a, int t) {
  return w.dl ? exp2f(w.dl[t] * a - w.ds.m2 - w.ds.log2_z) : 0.f;
}

// Phase B: one CTA per sequence.
__global__ void __launch_bounds__(kStThreads, 1) stochastic_walk_kernel(
    const float *__restrict__ target, const float *__restrict__ draft, int r_max, int vocab, float a,
    const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows, const int32_t *__restrict__ tokens,
    const double *__restrict__ uniforms, int n_uniforms, const RowStats *__restrict__ stats,
    int32_t *__restrict__ path, int32_t *__restrict__ path_len, int64_t *__restrict__ next_token,
    int32_t *__restrict__ uniforms_used, float *__restrict__ residual, int32_t *__restrict__ err) {
  __shared__ double red[32];
  __shared__ int s_flag;
  const int b = blockIdx.x;
  const int n = min(n_rows[b], r_max);
  const int32_t *par = parent + (int64_t)b * r_max;
  const int32_t *tok = tokens + (int64_t)b * r_max;
  const double *uni = uniforms + (int64_t)b * n_uniforms;
  const RowStats *st = stats + (int64_t)b * r_max * 2;
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  // any invalid (NaN) row in this sequence aborts it
  for (int r = threadIdx.x; r < n; r += kStThreads)
    if (!st[2 * r].valid) atomicOr(&s_flag, 1);
  __syncthreads();
  if (s_flag) {
    if (threadIdx.x == 0) {
      path_len[b] = 0;
      next_token[b] = 0;
      uniforms_used[b] = 0;
    }
    return;
  }
  int cur = 0, used = 0, len = 0;
  double c = 0.0, M = 1.0;
  bool failed = false;
  auto make_row = [&](int r) {
    WalkRow w;
    w.tl = target + ((int64_t)b * r_max + r) * vocab;
    w.ts = st[2 * r];
    w.ds = st[2 * r + 1];
    w.dl = w.ds.valid ? draft + ((int64_t)b * r_max + r) * vocab : nullptr;
    return w;
  };
  WalkRow w = make_row(cur);
  while (true) {
    bool descended = false;
    for (int j = cur + 1; j < n; ++j) {
      if (par[j] != cur) continue;
      if (used >= n_uniforms) {
        failed = true;
        break;
      }
      const double u = uni[used++];
      const int t = tok[j];
      const double pt_full = (double)p_of(w, a, t);
      const double qt = (double)q_of(w, a, t);
      const double pt = fmax(pt_full - c * qt, 0.0) / M;
      const bool acc = qt <= 0.0 ? pt > 0.0 : u < fmin(1.0, pt / qt);
      if (acc) {
        if (threadIdx.x == 0) path[(int64_t)b * r_max + len] = j - 1;
        ++len;
        cur = j;
        c = 0.0;
        M = 1.0;
        w = make_row(cur);
        descended = true;
        break;
      }
      // rejection: residual norm(max(p - q, 0)) == max(P - c' Q, 0) / M'
      const double cn = c + M;
      double part = 0.0;
      for (int i = threadIdx.x; i < vocab; i += kStThreads) {
        double v = (double)p_of(w, a, i) - cn * (double)q_of(w, a, i);
        part += v > 0.0 ? v : 0.0;
      }
      const double Mn = block_sum<kStThreads>(part, red);
      if (Mn / M <= 1e-12) {
        c = 0.0;  // anchor fallback (sampling.py:193-195)
        M = 1.0;
      } else {
        c = cn;
        M = Mn;
      }
    }
    if (failed || !descended) break;
  }
  if (!failed && used >= n_uniforms) failed = true;
  if (failed) {
    if (threadIdx.x == 0) {
      atomicOr(err, SDB_ERR_UNIFORMS);
      path_len[b] = len;
      next_token[b] = -1;
      uniforms_used[b] = used;
    }
    return;
  }
  const double u = uni[used++];
  // bonus: inverse CDF of p = max(P - c Q, 0) / M over the vocab in index
  // order (sample_from, sampling.py:105-109).  Warps own contiguous segments.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = kStThreads / 32;
  const int seg = (vocab + nw - 1) / nw;
  const int s0 = warp * seg, s1 = min(vocab, s0 + seg);
  auto pval = [&](int i) {
    double v = (double)p_of(w, a, i) - c * (double)q_of(w, a, i);
    return (v > 0.0 ? v : 0.0) / M;
  };
  double wsum = 0.0;
  for (int i = s0 + lane; i < s1; i += 32) {
    double v = pval(i);
    wsum += v;
    if (residual) residual[(int64_t)b * vocab + i] = (float)v;
  }
  wsum = warp_sum(wsum);
  __shared__ double segsum[32];
  __shared__ double s_prefix;
  if (lane == 0) segsum[warp] = wsum;
  __syncthreads();
  __shared__ int s_tok;
  if (threadIdx.x == 0) {
    // searchsorted(cumsum, u, 'right'): first index with cumsum > u
    double cum = 0.0;
    int ws = nw - 1;
    for (int k = 0; k < nw; ++k) {
      if (cum + segsum[k] > u) {
        ws = k;
        break;
      }
      cum += segsum[k];
    }
    s_prefix = cum;  // mass before the chosen segment
    s_tok = ws;
  }
  __syncthreads();
  const int ws = s_tok;
  if (warp == ws) {
    double cum = s_prefix;
    const int a0 = ws * seg, a1 = min(vocab, a0 + seg);
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
    if (lane == 0) s_tok = found < 0 ? vocab - 1 : found;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    path_len[b] = len;
    next_token[b] = min(s_tok, vocab - 1);
    uniforms_used[b] = used;
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
    sdb::argmax_keys_kernel<float><<<grid, sdb::kArgmaxThreads, 0, s>>>(
        (const float *)logits, vocab, row_stride, vocab_offset, nullptr, 0, (long long *)keys, err,
        vec_aligned(logits, row_stride, 4, vocab));
  else if (dtype == SDB_DTYPE_BF16)
    sdb::argmax_keys_kernel<__nv_bfloat16><<<grid, sdb::kArgmaxThreads, 0, s>>>(
        (const __nv_bfloat16 *)logits, vocab, row_stride, vocab_offset, nullptr, 0, (long long *)keys, err,
        vec_aligned(logits, row_stride, 2, vocab));
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
      (const long long *)keys, parent, n_rows, tokens, batch, r_max, path, path_len, next_token, uniforms_used);
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
  dim3 grid(r_max, batch);
  cudaStream_t s = sdb::as_stream(stream);
  if (dtype == SDB_DTYPE_F32)
    sdb::argmax_keys_kernel<float><<<grid, sdb::kArgmaxThreads, 0, s>>>(
        (const float *)logits, vocab, row_stride, 0, n_rows, r_max, (long long *)keys, err,
        vec_aligned(logits, row_stride, 4, vocab));
  else if (dtype == SDB_DTYPE_BF16)
    sdb::argmax_keys_kernel<__nv_bfloat16><<<grid, sdb::kArgmaxThreads, 0, s>>>(
        (const __nv_bfloat16 *)logits, vocab, row_stride, 0, n_rows, r_max, (long long *)keys, err,
        vec_aligned(logits, row_stride, 2, vocab));
  else
    return SDB_E_UNSUPPORTED;
  SDB_CHECK_LAUNCH();
  return sdb_greedy_walk(keys, parent, n_rows, tokens, batch, r_max, path, path_len, next_token, uniforms_used,
                         stream);
}

extern "C" int64_t sdb_accept_stochastic_workspace(int batch, int r_max, int vocab) {
  (void)vocab;
  if (batch < 0 || r_max < 1) return SDB_E_INVALID;
  return (int64_t)batch * r_max * 2 * (int64_t)sizeof(sdb::RowStats) + 256;
}

extern "C" int sdb_accept_stochastic(const float *target_logits, const float *draft_logits, int batch, int r_max,
                                     int vocab, float temperature, float top_p, const int32_t *parent,
                                     const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                                     int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                                     int32_t *path_len, int64_t *next_token, int32_t *uniforms_used,
                                     float *residual, int32_t *err, void *stream) {
  if (!target_logits || !draft_logits || !parent || !n_rows || !tokens || !uniforms || !path || !path_len ||
      !next_token || !uniforms_used || !err || batch < 0 || r_max < 1 || vocab < 1 || n_uniforms < 0)
    return SDB_E_INVALID;
  if (!(temperature > 0.0f) || !(top_p > 0.0f) || top_p > 1.0f) return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  if (!workspace || workspace_bytes < sdb_accept_stochastic_workspace(batch, r_max, vocab)) return SDB_E_WORKSPACE;
  const float a = 1.4426950408889634f / temperature;
  sdb::RowStats *stats = reinterpret_cast<sdb::RowStats *>(workspace);
  cudaStream_t s = sdb::as_stream(stream);
  const size_t smem = sizeof(sdb::StSmem);
  cudaFuncSetAttribute(sdb::row_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  sdb::row_stats_kernel<<<dim3(r_max, batch, 2), sdb::kStThreads, smem, s>>>(
      target_logits, draft_logits, r_max, vocab, a, top_p, parent, n_rows, stats, err);
  SDB_CHECK_LAUNCH();
  sdb::stochastic_walk_kernel<<<batch, sdb::kStThreads, 0, s>>>(target_logits, draft_logits, r_max, vocab, a,
                                                                 parent, n_rows, tokens, uniforms, n_uniforms,
                                                                 stats, path, path_len, next_token, uniforms_used,
                                                                 residual, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
