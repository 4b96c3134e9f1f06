// Vocab-sharded stochastic (T > 0) acceptance: SURVEY.md section 8(e).
//
// Each rank holds a contiguous vocabulary slice [vocab_offset, +vocab_local)
// of every target and draft logits row (a column-parallel LM head leaves them
// that way).  The reference semantics are those of the unsharded path
// (accept.cu, sampling.py:87-202): target_dist with the exact top-p nucleus
// for every tree row, the draft q of every parent row, the MSS walk, the
// inverse-CDF bonus draw.  The decomposition needs these exchanges, every one
// batched over all B*R rows (never per row), issued by the host between the
// phases below (see paper_2508_08192_b200/sharding.py):
//
//   PARTIALS   local (max, sum) per row            -> all-gather
//   COMBINE    global max / normaliser
//   NUCLEUS k  k = 0..3: 256-bin mass histogram over byte k of the
//              orderable fp32 key, restricted to the prefix found so far
//                                                  -> all-reduce SUM (x4)
//   CUT        exact cut key, per-rank tie counts  -> all-reduce SUM
//   FINISH     per-rank (key, index) cut; kept mass Z
//   TOKEN_PQ   p(t), q(t) of every drafted token   -> all-reduce SUM
//   RESIDUAL k k = 1..max_children: the rejection chain of every parent row,
//              M_k = sum max(P - c_k Q, 0)          -> all-reduce SUM (each)
//   WALK       identical MSS walk on every rank + local bonus mass
//                                                  -> all-reduce SUM
//   PICK       the owning rank draws the bonus token -> all-reduce MAX
//
// The rejection chain needs no token: siblings share their parent's q
// (engine.py:405-407), so after k rejections at a node the residual is
// max(P - c_k Q, 0) / M_k with c_{k+1} = c_k + M_k, M_{k+1} = sum max(P -
// c_{k+1} Q, 0) (anchor reset c = 0, M = 1 when M_{k+1} / M_k <= 1e-12,
// sampling.py:193-195).  It is therefore precomputed level-synchronously for
// every parent row, and the walk itself is collective-free and identical on
// every rank (same uniforms, same reduced values).
#include "accept_common.cuh"

namespace sdb {

constexpr int kShThreads = 512;
constexpr int kShBins = 256;

struct ShNuc {
  double tau;         // (top_p - 1e-12) * S in weight units
  double mass_above;  // mass of keys strictly above the current prefix range
  double w;           // weight of the cut key
  uint32_t prefix;    // cut-key bytes found so far
  uint32_t cut_key;
  int32_t active;     // target row with a nucleus (top_p < 1)
  int32_t need;       // tied elements kept (global)
};

struct ShWalk {
  double c, M;  // residual state at the final node
  int32_t cur, k, used, len, failed;
  double u;     // bonus uniform
};

struct ShScratch {
  RowStats *stats;  // [B][R][2]
  ShNuc *nuc;       // [B][R]
  int32_t *cnt;     // [B][R][256] local element counts of the last byte pass
  double2 *chain;   // [B][R][levels + 1] (c_k, M_k)
  ShWalk *walk;     // [B]
};

__host__ __device__ inline int64_t align_up(int64_t x) { return (x + 255) & ~int64_t(255); }

__host__ __device__ inline int64_t scratch_bytes(int batch, int r_max, int levels) {
  const int64_t rows = (int64_t)batch * r_max;
  return align_up(rows * 2 * (int64_t)sizeof(RowStats)) + align_up(rows * (int64_t)sizeof(ShNuc)) +
         align_up(rows * kShBins * 4) + align_up(rows * (levels + 1) * (int64_t)sizeof(double2)) +
         align_up((int64_t)batch * (int64_t)sizeof(ShWalk));
}

__host__ __device__ inline ShScratch carve(void *base, int batch, int r_max, int levels) {
  const int64_t rows = (int64_t)batch * r_max;
  char *p = (char *)base;
  ShScratch s;
  s.stats = (RowStats *)p;
  p += align_up(rows * 2 * (int64_t)sizeof(RowStats));
  s.nuc = (ShNuc *)p;
  p += align_up(rows * (int64_t)sizeof(ShNuc));
  s.cnt = (int32_t *)p;
  p += align_up(rows * kShBins * 4);
  s.chain = (double2 *)p;
  p += align_up(rows * (levels + 1) * (int64_t)sizeof(double2));
  s.walk = (ShWalk *)p;
  return s;
}

__device__ __forceinline__ float key_to_float(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// number of children of row r (rows j > r with parent[j] == r), block-wide;
// every thread of the block must call it
__device__ int block_children(const int32_t *par, int r, int n) {
  int c = 0;
  for (int j = r + 1 + threadIdx.x; j < n; j += blockDim.x) c += par[j] == r;
  return __syncthreads_count(c) ? [&] {
    __shared__ int s_c;
    if (threadIdx.x == 0) s_c = 0;
    __syncthreads();
    if (c) atomicAdd(&s_c, c);
    __syncthreads();
    return s_c;
  }() : 0;
}

struct ShParams {
  const float *target, *draft;
  int batch, r_max, vl;
  int64_t v_lo, vocab;
  int world, rank;
  float a, top_p;
  int levels;
  const int32_t *parent, *n_rows, *tokens;
  const double *uniforms;
  int n_uniforms;
  double *partials, *gathered, *hist;
  int32_t *tie;
  double *pq, *chain_x, *bonus_mass;
  long long *bonus_token;
  ShScratch s;
  int32_t *path, *path_len, *uniforms_used;
  float *residual;
  int32_t *err;
};

__device__ __forceinline__ const float *row_ptr(const float *base, const ShParams &p, int b, int r) {
  return base + ((int64_t)b * p.r_max + r) * p.vl;
}

// ---- PARTIALS: grid (r_max, B, 2) ----------------------------------------
__global__ void __launch_bounds__(kShThreads) sh_partials_kernel(ShParams p) {
  __shared__ float redf[32];
  __shared__ double red[32];
  const int r = blockIdx.x, b = blockIdx.y, z = blockIdx.z;
  const int n = min(p.n_rows[b], p.r_max);
  double *out = p.partials + (((int64_t)b * p.r_max + r) * 2 + z) * 2;
  bool use = r < n;
  if (use && z == 1) use = block_children(p.parent + (int64_t)b * p.r_max, r, n) > 0;
  if (!use) {
    if (threadIdx.x == 0) {
      out[0] = -INFINITY;
      out[1] = 0.0;
    }
    return;
  }
  const float *row = row_ptr(z ? p.draft : p.target, p, b, r);
  float mx = -INFINITY;
  bool nan = false;
  for (int i = threadIdx.x; i < p.vl; i += kShThreads) {
    const float v = row[i];
    nan |= v != v;
    mx = fmaxf(mx, v);
  }
  if (__syncthreads_or(nan)) {
    if (threadIdx.x == 0) {
      atomicOr(p.err, SDB_ERR_NAN);
      out[0] = NAN;
      out[1] = 0.0;
    }
    return;
  }
  mx = block_max<kShThreads>(mx, redf);
  const float m2 = mx * p.a;
  float s = 0.f;
  for (int i = threadIdx.x; i < p.vl; i += kShThreads) s += exp2f(row[i] * p.a - m2);
  const double S = block_sum<kShThreads>((double)s, red);
  if (threadIdx.x == 0) {
    out[0] = (double)m2;
    out[1] = S;
  }
}

// ---- COMBINE: one thread per (b, r) ------------------------------------------
__global__ void sh_combine_kernel(ShParams p) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.batch * p.r_max) return;
  const int b = (int)(idx / p.r_max), r = (int)(idx % p.r_max);
  const int n = min(p.n_rows[b], p.r_max);
  for (int z = 0; z < 2; ++z) {
    RowStats st;
    st.valid = 0;
    st.keep_all = 1;
    st.cut_key = 0;
    st.cut_idx = 0;
    double M = -INFINITY;
    bool nan = false;
    for (int g = 0; g < p.world; ++g) {
      const double m = p.gathered[(((int64_t)g * p.batch + b) * p.r_max + r) * 4 + z * 2];
      nan |= m != m;
      M = fmax(M, m);
    }
    if (nan) atomicOr(p.err, SDB_ERR_NAN);
    if (r < n && !nan && M > -INFINITY) {
      // the global max is one rank's local m2 (a float), bit-exact
      const float m2 = (float)M;
      double S = 0.0;
      for (int g = 0; g < p.world; ++g) {
        const double *q = p.gathered + (((int64_t)g * p.batch + b) * p.r_max + r) * 4 + z * 2;
        if (q[0] > -INFINITY) S += q[1] * exp2(q[0] - M);
      }
      st.m2 = m2;
      st.s = S;
      st.z = S;
      st.log2_z = (float)log2(S);
      st.valid = 1;
    }
    p.s.stats[idx * 2 + z] = st;
    if (z == 0) {
      ShNuc nu;
      nu.active = st.valid && p.top_p < 1.0f;
      nu.tau = ((double)p.top_p - 1e-12) * st.s;
      nu.mass_above = 0.0;
      nu.prefix = 0;
      nu.cut_key = 0;
      nu.w = 0.0;
      nu.need = 0;
      p.s.nuc[idx] = nu;
    }
  }
  // a NaN anywhere in the sequence invalidates it on every rank
}

// Scan a reduced 256-bin histogram from the top: the bin where the running
// mass crosses tau (or the lowest non-empty bin if rounding keeps it below).
__device__ void scan_hist(const double *h, ShNuc &nu, int &bin_out, double &above_out) {
  double cum = nu.mass_above;
  int last_nz = -1;
  for (int bb = kShBins - 1; bb >= 0; --bb) {
    const double m = h[bb];
    if (m > 0.0) last_nz = bb;
    if (m > 0.0 && cum + m >= nu.tau) {
      bin_out = bb;
      above_out = cum;
      return;
    }
    cum += m;
  }
  // not reached: keep everything down to the lowest non-empty bin
  bin_out = last_nz < 0 ? 0 : last_nz;
  above_out = cum - (last_nz < 0 ? 0.0 : h[last_nz]);
}

// ---- NUCLEUS pass k: grid (r_max, B) ------------------------------------------
__global__ void __launch_bounds__(kShThreads) sh_nucleus_kernel(ShParams p, int k) {
  __shared__ double hist[kShBins];
  __shared__ int cnt[kShBins];
  __shared__ ShNuc s_nu;
  const int r = blockIdx.x, b = blockIdx.y;
  const int64_t idx = (int64_t)b * p.r_max + r;
  double *hout = p.hist + idx * kShBins;
  if (threadIdx.x == 0) {
    ShNuc nu = p.s.nuc[idx];
    if (nu.active && k > 0) {
      int bin;
      double above;
      scan_hist(hout, nu, bin, above);  // reduced histogram of pass k-1
      nu.prefix = (nu.prefix << 8) | (uint32_t)bin;
      nu.mass_above = above;
      p.s.nuc[idx] = nu;
    }
    s_nu = nu;
  }
  for (int i = threadIdx.x; i < kShBins; i += kShThreads) {
    hist[i] = 0.0;
    cnt[i] = 0;
  }
  __syncthreads();
  const ShNuc nu = s_nu;
  if (nu.active) {
    const RowStats st = p.s.stats[idx * 2];
    const float *row = row_ptr(p.target, p, b, r);
    const int hi_shift = 32 - 8 * k, shift = 24 - 8 * k;
    for (int i = threadIdx.x; i < p.vl; i += kShThreads) {
      const float l = row[i];
      const uint32_t key = prob_key(l);
      if (k > 0 && (key >> hi_shift) != nu.prefix) continue;
      const int bin = (key >> shift) & 0xff;
      atomicAdd(&hist[bin], (double)exp2f(l * p.a - st.m2));
      if (k == 3) atomicAdd(&cnt[bin], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kShBins; i += kShThreads) {
    hout[i] = hist[i];
    if (k == 3) p.s.cnt[idx * kShBins + i] = cnt[i];
  }
}

// ---- CUT: grid covers (b, r), one thread each -----------------------------------
__global__ void sh_cut_kernel(ShParams p) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.batch * p.r_max) return;
  ShNuc nu = p.s.nuc[idx];
  int32_t *tie = p.tie + idx * p.world;
  for (int g = 0; g < p.world; ++g) tie[g] = 0;
  if (!nu.active) return;
  int bin;
  double above;
  scan_hist(p.hist + idx * kShBins, nu, bin, above);
  nu.cut_key = (nu.prefix << 8) | (uint32_t)bin;
  nu.mass_above = above;
  const RowStats st = p.s.stats[idx * 2];
  nu.w = (double)exp2f(key_to_float(nu.cut_key) * p.a - st.m2);
  p.s.nuc[idx] = nu;
  tie[p.rank] = p.s.cnt[idx * kShBins + bin];
}

// ---- FINISH: grid (r_max, B) -------------------------------------------------------
__global__ void __launch_bounds__(kShThreads) sh_finish_kernel(ShParams p) {
  __shared__ double red[32];
  __shared__ int s_idx;
  __shared__ int s_seen;
  const int r = blockIdx.x, b = blockIdx.y;
  const int64_t idx = (int64_t)b * p.r_max + r;
  const ShNuc nu0 = p.s.nuc[idx];
  if (!nu0.active) return;
  const int32_t *tie = p.tie + idx * p.world;
  long long total = 0, before = 0;
  for (int g = 0; g < p.world; ++g) {
    total += tie[g];
    if (g < p.rank) before += tie[g];
  }
  long long need = (long long)ceil((nu0.tau - nu0.mass_above) / nu0.w);
  need = need < 1 ? 1 : (need > total ? total : need);
  const long long mine = tie[p.rank];
  long long kept_local = need - before;
  kept_local = kept_local < 0 ? 0 : (kept_local > mine ? mine : kept_local);
  int cut_idx;
  if (kept_local == 0) {
    cut_idx = -1;
  } else if (kept_local == mine) {
    cut_idx = INT_MAX;
  } else {
    // local index of the kept_local-th tied element in index order
    const float *row = row_ptr(p.target, p, b, r);
    if (threadIdx.x == 0) {
      s_idx = p.vl - 1;
      s_seen = 0;
    }
    __syncthreads();
    for (int c0 = 0; c0 < p.vl; c0 += kShThreads) {
      const int i = c0 + threadIdx.x;
      const bool t = i < p.vl && prob_key(row[i]) == nu0.cut_key;
      const unsigned bal = __ballot_sync(SDB_FULL_MASK, t);
      // block-wide exclusive prefix of tied flags (warp ballots)
      __shared__ int wcnt[kShThreads / 32];
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      int pre = s_seen;
      for (int w = 0; w < warp; ++w) pre += wcnt[w];
      pre += __popc(bal & ((1u << lane) - 1u));
      if (t && pre + 1 == kept_local) s_idx = i;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < kShThreads / 32; ++w) tot += wcnt[w];
        s_seen += tot;
      }
      __syncthreads();
      if (s_seen >= kept_local) break;
    }
    cut_idx = s_idx;
  }
  (void)red;
  if (threadIdx.x == 0) {
    RowStats st = p.s.stats[idx * 2];
    st.z = nu0.mass_above + nu0.w * (double)need;
    st.log2_z = (float)log2(st.z);
    st.cut_key = nu0.cut_key;
    st.cut_idx = cut_idx;
    st.keep_all = 0;
    p.s.stats[idx * 2] = st;
  }
}

__device__ __forceinline__ float sh_p(const RowStats &ts, const float *tl, float a, int i) {
  const float l = tl[i];
  return kept(ts, l, i) ? exp2f(l * a - ts.m2 - ts.log2_z) : 0.f;
}
__device__ __forceinline__ float sh_q(const RowStats &ds, const float *dl, float a, int i) {
  return exp2f(dl[i] * a - ds.m2 - ds.log2_z);
}

// ---- TOKEN_PQ: one thread per (b, row j) ---------------------------------------------
__global__ void sh_token_pq_kernel(ShParams p) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.batch * p.r_max) return;
  const int b = (int)(idx / p.r_max), j = (int)(idx % p.r_max);
  const int n = min(p.n_rows[b], p.r_max);
  double P = 0.0, Q = 0.0;
  if (j >= 1 && j < n) {
    const int pr = p.parent[idx];
    const int64_t t = p.tokens[idx];
    if (pr >= 0 && pr < j && t >= p.v_lo && t < p.v_lo + p.vl) {
      const int64_t pidx = (int64_t)b * p.r_max + pr;
      const RowStats ts = p.s.stats[pidx * 2], ds = p.s.stats[pidx * 2 + 1];
      if (ts.valid && ds.valid) {
        const int i = (int)(t - p.v_lo);
        P = (double)sh_p(ts, row_ptr(p.target, p, b, pr), p.a, i);
        Q = (double)sh_q(ds, row_ptr(p.draft, p, b, pr), p.a, i);
      }
    }
  }
  p.pq[idx * 2] = P;
  p.pq[idx * 2 + 1] = Q;
  double2 *ch = p.s.chain + idx * (p.levels + 1);
  ch[0] = make_double2(0.0, 1.0);
}

// chain[k] from the reduced level-k mass X_k (sampling.py:190-195)
__device__ __forceinline__ double2 chain_step(double2 prev, double X) {
  const double cn = prev.x + prev.y;
  return X / prev.y <= 1e-12 ? make_double2(0.0, 1.0) : make_double2(cn, X);
}

// ---- RESIDUAL level k (1-based): grid (r_max, B) --------------------------------------
// Finalises chain[k-1] from the reduced X_{k-1} (rows with >= k-1 children),
// then, for rows with >= k children, the local X_k = sum max(P - c' Q, 0)
// with c' = c_{k-1} + M_{k-1}.
__global__ void __launch_bounds__(kShThreads) sh_residual_kernel(ShParams p, int k) {
  __shared__ double red[32];
  const int r = blockIdx.x, b = blockIdx.y;
  const int64_t idx = (int64_t)b * p.r_max + r;
  const int n = min(p.n_rows[b], p.r_max);
  if (r >= n) return;
  const int nch = block_children(p.parent + (int64_t)b * p.r_max, r, n);
  double2 *ch = p.s.chain + idx * (p.levels + 1);
  if (k >= 2 && nch >= k - 1) {
    if (threadIdx.x == 0) ch[k - 1] = chain_step(ch[k - 2], p.chain_x[idx]);
    __syncthreads();
  }
  if (nch < k) return;
  const RowStats ts = p.s.stats[idx * 2], ds = p.s.stats[idx * 2 + 1];
  double X = 0.0;
  if (ts.valid && ds.valid) {
    const double2 prev = ch[k - 1];
    const double cn = prev.x + prev.y;
    const float *tl = row_ptr(p.target, p, b, r), *dl = row_ptr(p.draft, p, b, r);
    double part = 0.0;
    for (int i = threadIdx.x; i < p.vl; i += kShThreads) {
      const double v = (double)sh_p(ts, tl, p.a, i) - cn * (double)sh_q(ds, dl, p.a, i);
      part += v > 0.0 ? v : 0.0;
    }
    X = block_sum<kShThreads>(part, red);
  }
  if (threadIdx.x == 0) p.chain_x[idx] = X;
}

// ---- WALK (+ local bonus mass): grid B ---------------------------------------------------
__global__ void __launch_bounds__(kShThreads) sh_walk_kernel(ShParams p) {
  __shared__ double red[32];
  __shared__ ShWalk s_w;
  __shared__ int s_bad;
  const int b = blockIdx.x;
  const int n = min(p.n_rows[b], p.r_max);
  const int32_t *par = p.parent + (int64_t)b * p.r_max;
  const int32_t *tok = p.tokens + (int64_t)b * p.r_max;
  (void)tok;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  // finalise chain[levels] and check row validity
  for (int r = threadIdx.x; r < n; r += kShThreads) {
    const int64_t idx = (int64_t)b * p.r_max + r;
    if (!p.s.stats[idx * 2].valid) atomicOr(&s_bad, 1);
    int nch = 0;
    for (int j = r + 1; j < n; ++j) nch += par[j] == r;
    if (p.levels >= 1 && nch >= p.levels) {
      double2 *ch = p.s.chain + idx * (p.levels + 1);
      ch[p.levels] = chain_step(ch[p.levels - 1], p.chain_x[idx]);
    }
  }
  __syncthreads();
  double *bm = p.bonus_mass + (int64_t)b * p.world;
  if (s_bad) {
    if (threadIdx.x == 0) {
      for (int g = 0; g < p.world; ++g) bm[g] = 0.0;
      ShWalk w;
      w.failed = 2;
      w.len = 0;
      w.used = 0;
      w.cur = 0;
      w.k = 0;
      w.c = 0.0;
      w.M = 1.0;
      w.u = 0.0;
      p.s.walk[b] = w;
    }
    return;
  }
  if (threadIdx.x == 0) {
    const double *uni = p.uniforms + (int64_t)b * p.n_uniforms;
    int cur = 0, k = 0, used = 0, len = 0, failed = 0;
    while (true) {
      bool descended = false;
      for (int j = cur + 1; j < n; ++j) {
        if (par[j] != cur) continue;
        if (used >= p.n_uniforms) {
          failed = 1;
          break;
        }
        const double u = uni[used++];
        const int64_t jdx = (int64_t)b * p.r_max + j;
        const double P = p.pq[jdx * 2], Q = p.pq[jdx * 2 + 1];
        if (k > p.levels) {  // more siblings than the planned chain (max_children): no clamped guess
          failed = 3;
          break;
        }
        const double2 cm = p.s.chain[((int64_t)b * p.r_max + cur) * (p.levels + 1) + k];
        const double pt = fmax(P - cm.x * Q, 0.0) / cm.y;
        const bool acc = Q <= 0.0 ? pt > 0.0 : u < fmin(1.0, pt / Q);
        if (acc) {
          p.path[(int64_t)b * p.r_max + len++] = j - 1;
          cur = j;
          k = 0;
          descended = true;
          break;
        }
        ++k;
      }
      if (failed || !descended) break;
    }
    if (!failed && used >= p.n_uniforms) failed = 1;
    if (!failed && k > p.levels) failed = 3;
    ShWalk w;
    const double2 cm = p.s.chain[((int64_t)b * p.r_max + cur) * (p.levels + 1) + min(k, p.levels)];
    w.c = cm.x;
    w.M = cm.y;
    w.cur = cur;
    w.k = k;
    w.len = len;
    w.failed = failed;
    w.u = failed ? 0.0 : uni[used];
    w.used = failed ? used : used + 1;
    s_w = w;
    p.s.walk[b] = w;
    if (failed) atomicOr(p.err, failed == 3 ? SDB_ERR_PLAN : SDB_ERR_UNIFORMS);
  }
  __syncthreads();
  const ShWalk w = s_w;
  double part = 0.0;
  if (!w.failed) {
    const int64_t idx = (int64_t)b * p.r_max + w.cur;
    const RowStats ts = p.s.stats[idx * 2], ds = p.s.stats[idx * 2 + 1];
    const float *tl = row_ptr(p.target, p, b, w.cur), *dl = row_ptr(p.draft, p, b, w.cur);
    const bool hasq = ds.valid && w.c != 0.0;
    for (int i = threadIdx.x; i < p.vl; i += kShThreads) {
      double v = (double)sh_p(ts, tl, p.a, i) - (hasq ? w.c * (double)sh_q(ds, dl, p.a, i) : 0.0);
      part += (v > 0.0 ? v : 0.0) / w.M;
    }
  }
  const double tot = block_sum<kShThreads>(part, red);
  if (threadIdx.x == 0)
    for (int g = 0; g < p.world; ++g) bm[g] = g == p.rank ? tot : 0.0;
}

// ---- PICK: grid B -----------------------------------------------------------------------------
__global__ void __launch_bounds__(kShThreads) sh_pick_kernel(ShParams p) {
  __shared__ double segsum[kShThreads / 32];
  __shared__ double s_prefix;
  __shared__ int s_seg, s_tok;
  const int b = blockIdx.x;
  const ShWalk w = p.s.walk[b];
  const double *bm = p.bonus_mass + (int64_t)b * p.world;
  double base = 0.0, total = 0.0;
  for (int g = 0; g < p.world; ++g) {
    if (g < p.rank) base += bm[g];
    total += bm[g];
  }
  const double mine = bm[p.rank];
  // owner: the first rank whose inclusive cumulative mass exceeds u; if
  // rounding leaves every rank at or below u, the last rank clips to V - 1
  const bool owner = !w.failed && ((base <= w.u && base + mine > w.u) || (p.rank == p.world - 1 && total <= w.u));
  const int64_t idx = (int64_t)b * p.r_max + w.cur;
  const RowStats ts = p.s.stats[idx * 2], ds = p.s.stats[idx * 2 + 1];
  const float *tl = row_ptr(p.target, p, b, w.cur), *dl = row_ptr(p.draft, p, b, w.cur);
  const bool hasq = ds.valid && w.c != 0.0;
  auto pval = [&](int i) {
    double v = (double)sh_p(ts, tl, p.a, i) - (hasq ? w.c * (double)sh_q(ds, dl, p.a, i) : 0.0);
    return (v > 0.0 ? v : 0.0) / w.M;
  };
  if (p.residual && !w.failed)
    for (int i = threadIdx.x; i < p.vl; i += kShThreads) p.residual[(int64_t)b * p.vl + i] = (float)pval(i);
  long long tok = -1;
  if (owner) {
    if (!(base + mine > w.u)) {
      tok = p.vocab - 1;
    } else {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kShThreads / 32;
      const int seg = (p.vl + nw - 1) / nw;
      const int s0 = warp * seg, s1 = min(p.vl, s0 + seg);
      double ws = 0.0;
      for (int i = s0 + lane; i < s1; i += 32) ws += pval(i);
      ws = warp_sum(ws);
      if (lane == 0) segsum[warp] = ws;
      __syncthreads();
      if (threadIdx.x == 0) {
        double cum = base;
        int sel = nw - 1;
        for (int q = 0; q < nw; ++q) {
          if (cum + segsum[q] > w.u) {
            sel = q;
            break;
          }
          cum += segsum[q];
        }
        s_prefix = cum;
        s_seg = sel;
      }
      __syncthreads();
      if (warp == s_seg) {
        double cum = s_prefix;
        const int a0 = s_seg * seg, a1 = min(p.vl, a0 + seg);
        int found = -1;
        for (int i0 = a0; i0 < a1 && found < 0; i0 += 32) {
          const int i = i0 + lane;
          double incl = i < a1 ? pval(i) : 0.0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(SDB_FULL_MASK, incl, o);
            if (lane >= o) incl += t;
          }
          const unsigned hit = __ballot_sync(SDB_FULL_MASK, i < a1 && cum + incl > w.u);
          if (hit) found = i0 + __ffs(hit) - 1;
          cum += __shfl_sync(SDB_FULL_MASK, incl, 31);
        }
        if (lane == 0) s_tok = found < 0 ? p.vl - 1 : found;
      }
      __syncthreads();
      tok = p.v_lo + s_tok;
    }
  }
  if (threadIdx.x == 0) {
    p.bonus_token[b] = tok;
    p.path_len[b] = w.failed >= 2 ? 0 : w.len;
    p.uniforms_used[b] = w.failed >= 2 ? 0 : w.used;
  }
}

}  // namespace sdb

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
static int sh_params(const sdb_sharded_accept_args *a, sdb::ShParams &p) {
  if (!a || !a->target_logits || !a->draft_logits || !a->parent || !a->n_rows || !a->tokens || !a->err)
    return SDB_E_INVALID;
  if (a->batch < 0 || a->batch > 65535 || a->r_max < 1 || a->r_max > 65535 || a->vocab_local < 1 ||
      a->world < 1 || a->rank < 0 || a->rank >= a->world || a->max_children < 0 || a->max_children > a->r_max ||
      a->vocab_offset < 0 || a->vocab_offset + a->vocab_local > a->vocab || a->vocab > 0x7fffffffll)
    return SDB_E_INVALID;
  if (!(a->temperature > 0.0f) || !(a->top_p > 0.0f) || a->top_p > 1.0f) return SDB_E_INVALID;
  if (!a->scratch || a->scratch_bytes < sdb::scratch_bytes(a->batch, a->r_max, a->max_children))
    return SDB_E_WORKSPACE;
  p.target = a->target_logits;
  p.draft = a->draft_logits;
  p.batch = a->batch;
  p.r_max = a->r_max;
  p.vl = a->vocab_local;
  p.v_lo = a->vocab_offset;
  p.vocab = a->vocab;
  p.world = a->world;
  p.rank = a->rank;
  p.a = 1.4426950408889634f / a->temperature;
  p.top_p = a->top_p;
  p.levels = a->max_children;
  p.parent = a->parent;
  p.n_rows = a->n_rows;
  p.tokens = a->tokens;
  p.uniforms = a->uniforms;
  p.n_uniforms = a->n_uniforms;
  p.partials = a->xchg_partials;
  p.gathered = a->gathered;
  p.hist = a->hist;
  p.tie = a->tie;
  p.pq = a->pq;
  p.chain_x = a->chain_x;
  p.bonus_mass = a->bonus_mass;
  p.bonus_token = (long long *)a->bonus_token;
  p.s = sdb::carve(a->scratch, a->batch, a->r_max, a->max_children);
  p.path = a->path;
  p.path_len = a->path_len;
  p.uniforms_used = a->uniforms_used;
  p.residual = a->residual;
  p.err = a->err;
  return SDB_OK;
}

extern "C" int sdb_sharded_accept_sizes(const sdb_sharded_accept_args *a, int64_t *sizes) {
  if (!a || !sizes || a->batch < 0 || a->r_max < 1 || a->world < 1 || a->max_children < 0) return SDB_E_INVALID;
  const int64_t rows = (int64_t)a->batch * a->r_max;
  sizes[SDB_SH_BUF_PARTIALS] = rows * 4;               // doubles
  sizes[SDB_SH_BUF_GATHERED] = rows * 4 * a->world;    // doubles
  sizes[SDB_SH_BUF_HIST] = rows * sdb::kShBins;         // doubles
  sizes[SDB_SH_BUF_TIE] = rows * a->world;              // int32
  sizes[SDB_SH_BUF_PQ] = rows * 2;                      // doubles
  sizes[SDB_SH_BUF_CHAIN_X] = rows;                     // doubles
  sizes[SDB_SH_BUF_BONUS_MASS] = (int64_t)a->batch * a->world;  // doubles
  sizes[SDB_SH_BUF_BONUS_TOKEN] = a->batch;             // int64
  sizes[SDB_SH_BUF_SCRATCH] = sdb::scratch_bytes(a->batch, a->r_max, a->max_children);  // bytes
  return SDB_OK;
}

extern "C" int sdb_sharded_accept_phase(const sdb_sharded_accept_args *a, int phase, int level, void *stream) {
  sdb::ShParams p;
  int rc = sh_params(a, p);
  if (rc != SDB_OK) return rc;
  if (p.batch == 0) return SDB_OK;
  cudaStream_t s = sdb::as_stream(stream);
  const int64_t rows = (int64_t)p.batch * p.r_max;
  const int rb = (int)((rows + 255) / 256);
  const dim3 rgrid(p.r_max, p.batch);
  switch (phase) {
    case SDB_SH_PARTIALS:
      if (!p.partials) return SDB_E_INVALID;
      sdb::sh_partials_kernel<<<dim3(p.r_max, p.batch, 2), sdb::kShThreads, 0, s>>>(p);
      break;
    case SDB_SH_COMBINE:
      if (!p.gathered) return SDB_E_INVALID;
      sdb::sh_combine_kernel<<<rb, 256, 0, s>>>(p);
      break;
    case SDB_SH_NUCLEUS:
      if (!p.hist || level < 0 || level > 3) return SDB_E_INVALID;
      sdb::sh_nucleus_kernel<<<rgrid, sdb::kShThreads, 0, s>>>(p, level);
      break;
    case SDB_SH_CUT:
      if (!p.hist || !p.tie) return SDB_E_INVALID;
      sdb::sh_cut_kernel<<<rb, 256, 0, s>>>(p);
      break;
    case SDB_SH_FINISH:
      if (!p.tie) return SDB_E_INVALID;
      sdb::sh_finish_kernel<<<rgrid, sdb::kShThreads, 0, s>>>(p);
      break;
    case SDB_SH_TOKEN_PQ:
      if (!p.pq) return SDB_E_INVALID;
      sdb::sh_token_pq_kernel<<<rb, 256, 0, s>>>(p);
      break;
    case SDB_SH_RESIDUAL:
      if (!p.chain_x || level < 1 || level > p.levels) return SDB_E_INVALID;
      sdb::sh_residual_kernel<<<rgrid, sdb::kShThreads, 0, s>>>(p, level);
      break;
    case SDB_SH_WALK:
      if (!p.pq || !p.chain_x || !p.bonus_mass || !p.uniforms || !p.path) return SDB_E_INVALID;
      sdb::sh_walk_kernel<<<p.batch, sdb::kShThreads, 0, s>>>(p);
      break;
    case SDB_SH_PICK:
      if (!p.bonus_mass || !p.bonus_token || !p.path_len || !p.uniforms_used) return SDB_E_INVALID;
      sdb::sh_pick_kernel<<<p.batch, sdb::kShThreads, 0, s>>>(p);
      break;
    default:
      return SDB_E_INVALID;
  }
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
