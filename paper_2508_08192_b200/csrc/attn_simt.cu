// Attention on CUDA cores:
//   * sdb_attend_heads_f64 / sdb_merge_partials_f64 -- the drop-in
//     reference-precision (float64) attention core and LSE merge
//     (kernels.py:40-92, attention.py:108-124);
//   * the SIMT instantiation of the batched paged GQA tree-verify attention
//     (any head_dim <= 256, multiple of 4; bf16 or fp32 I/O) used for fp32
//     inputs, unusual head dims and as an on-device cross-check of the
//     tcgen05 kernel (attn_sm100.cu);
//   * the split-KV LSE combine shared by both tree-verify kernels.
#include <math.h>

#include "attn_internal.cuh"

namespace sdb {

// ---------------------------------------------------------------------------
// float64 drop-in: one warp per (head, query row); lanes own output dims
// (<= 8 per lane, head_dim <= 256).  Two passes over keys: row max, then
// exp-weights and the weighted V sum -- the same arithmetic as
// _attend_numba (kernels.py:57-92) with fully masked rows -> 0 / -inf.
// ---------------------------------------------------------------------------
__global__ void attend_heads_f64_kernel(const double *__restrict__ q, const double *__restrict__ k,
                                        const double *__restrict__ v, const uint8_t *__restrict__ mask,
                                        int heads, int m, int n, int d, double scale, double *__restrict__ out,
                                        double *__restrict__ lse) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= heads * m) return;
  const int h = warp / m, i = warp % m;
  const double *qr = q + ((int64_t)h * m + i) * d;
  const double *kh = k + (int64_t)h * n * d;
  const double *vh = v + (int64_t)h * n * d;
  double qv[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) qv[t] = (lane + 32 * t < d) ? qr[lane + 32 * t] : 0.0;
  auto score = [&](int j) {
    const double *kr = kh + (int64_t)j * d;
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < d) s += qv[t] * kr[lane + 32 * t];
    return warp_sum(s) * scale;
  };
  double smax = -INFINITY;
  for (int j = 0; j < n; ++j) {
    if (mask && !mask[(int64_t)i * n + j]) continue;
    smax = fmax(smax, score(j));
  }
  double *orow = out + ((int64_t)h * m + i) * d;
  if (smax == -INFINITY) {
    for (int t = lane; t < d; t += 32) orow[t] = 0.0;
    if (lane == 0) lse[(int64_t)h * m + i] = -INFINITY;
    return;
  }
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double denom = 0.0;
  for (int j = 0; j < n; ++j) {
    if (mask && !mask[(int64_t)i * n + j]) continue;
    double w = exp(score(j) - smax);
    denom += w;
    const double *vr = vh + (int64_t)j * d;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < d) acc[t] += w * vr[lane + 32 * t];
  }
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (lane + 32 * t < d) orow[lane + 32 * t] = acc[t] / denom;
  if (lane == 0) lse[(int64_t)h * m + i] = smax + log(denom);
}

// merge_partials (attention.py:108-124): one thread per (head, row).
__global__ void merge_partials_f64_kernel(const double *__restrict__ outs, const double *__restrict__ lses,
                                          int parts, int heads, int m, int d, double *__restrict__ out,
                                          double *__restrict__ lse, int32_t *__restrict__ err) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= heads * m) return;
  const int64_t hm = (int64_t)heads * m;
  double mx = -INFINITY;
  for (int p = 0; p < parts; ++p) mx = fmax(mx, lses[p * hm + idx]);
  double *orow = out + (int64_t)idx * d;
  if (!(mx > -INFINITY && mx < INFINITY)) {
    if (err) atomicOr(err, SDB_ERR_ALL_MASKED);
    for (int t = 0; t < d; ++t) orow[t] = 0.0;
    lse[idx] = -INFINITY;
    return;
  }
  double denom = 0.0;
  for (int p = 0; p < parts; ++p) denom += exp(lses[p * hm + idx] - mx);
  for (int t = 0; t < d; ++t) {
    double s = 0.0;
    for (int p = 0; p < parts; ++p) s += exp(lses[p * hm + idx] - mx) * outs[(p * hm + idx) * d + t];
    orow[t] = s / denom;
  }
  lse[idx] = mx + log(denom);
}

// ---------------------------------------------------------------------------
// SIMT batched paged GQA tree-verify attention (split-KV partials).
//
// CTA = 4 warps = 32 query rows of one (sequence, kv head); rows are ordered
// rho = node * g + j (q head = kvh * g + j) so a node's g heads are adjacent.
// Keys: [0, C) committed prefix read through the block table (no mask),
// [C, C + n_rows) fresh tree rows under the ancestor bitmask.  Key tiles of
// 32 (one key per lane for QK^T, lanes over head dims for PV); online
// softmax in log2 units.
// ---------------------------------------------------------------------------
constexpr int kSimtRowsPerWarp = 8;
constexpr int kSimtWarps = 4;
constexpr int kSimtRows = kSimtRowsPerWarp * kSimtWarps;
constexpr int kSimtKeys = 32;

template <typename T>
__global__ void __launch_bounds__(kSimtWarps * 32) tree_attn_simt_kernel(TreeAttnParams p) {
  extern __shared__ float sm[];
  const int D = p.head_dim, DP = D + 4;
  float *sQ = sm;                       // [32 rows][D]
  float *sK = sQ + kSimtRows * D;       // [32 keys][D+4]
  float *sV = sK + kSimtKeys * DP;      // [32 keys][D]
  float *sP = sV + kSimtKeys * D;       // [warps][32 keys][8 rows]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, row_tile = blockIdx.y;
  const int b = blockIdx.z / p.hkv, kvh = blockIdx.z % p.hkv;
  const int g = p.hq / p.hkv;
  const int n_nodes = min(p.n_rows[b], p.r_max);
  const int q0 = q_first(p, b, n_nodes);  // query rows: nodes [q0, n_nodes)
  const int rows_total = (n_nodes - q0) * g;
  const int row0 = row_tile * kSimtRows;
  if (row0 >= rows_total) {
    // padding rows of an unsplit launch still get zeros / -inf
    if (p.num_splits == 1) {
      for (int r = warp; r < kSimtRows; r += kSimtWarps) {
        int rho = row0 + r;
        if (q0 * g + rho < p.r_max * g)
          store_partial<T>(p, 0, b, q0 + rho / g, kvh * g + rho % g, -INFINITY, [&](int) { return 0.f; }, lane);
      }
    }
    return;
  }
  const int C = p.ctx_len[b];
  const int kstart = prefix_start(p, C);  // iRoPE: prefix keys [kstart, C)
  const int T_keys = C + n_nodes;
  // split range, tile aligned
  const int tiles = cdiv(T_keys, kSimtKeys);
  const int tiles_per = cdiv(tiles, p.num_splits);
  const int k_begin = split * tiles_per * kSimtKeys;
  const int k_end = min(T_keys, k_begin + tiles_per * kSimtKeys);
  const T *q = reinterpret_cast<const T *>(p.q);
  // stage Q rows (fp32)
  for (int idx = threadIdx.x; idx < kSimtRows * D; idx += blockDim.x) {
    int r = idx / D, c = idx % D;
    int rho = row0 + r;
    float val = 0.f;
    if (rho < rows_total) {
      int node = q0 + rho / g, j = rho % g;
      val = to_f32<T>(q[(((int64_t)b * p.r_max + node) * p.hq + kvh * g + j) * D + c]);
    }
    sQ[idx] = val;
  }
  const float sl2 = p.scale * 1.4426950408889634f;  // scores in log2 units
  float m_r[kSimtRowsPerWarp], l_r[kSimtRowsPerWarp], acc[kSimtRowsPerWarp][8];
#pragma unroll
  for (int r = 0; r < kSimtRowsPerWarp; ++r) {
    m_r[r] = -INFINITY;
    l_r[r] = 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[r][t] = 0.f;
  }
  const T *kc = reinterpret_cast<const T *>(p.k_cache);
  const T *vc = reinterpret_cast<const T *>(p.v_cache);
  const T *tk = reinterpret_cast<const T *>(p.tree_k);
  const T *tv = reinterpret_cast<const T *>(p.tree_v);
  const int wrow0 = warp * kSimtRowsPerWarp;  // first row of this warp within the CTA tile
  for (int kt = k_begin; kt < k_end; kt += kSimtKeys) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSimtKeys * D; idx += blockDim.x) {
      int j = idx / D, c = idx % D;
      int key = kt + j;
      float kv = 0.f, vv = 0.f;
      if (key < C) {
        int page = p.block_table[(int64_t)b * p.max_blocks + key / p.block_size];
        int64_t off = (((int64_t)page * p.hkv + kvh) * p.block_size + key % p.block_size) * D + c;
        kv = to_f32<T>(kc[off]);
        vv = to_f32<T>(vc[off]);
      } else if (key < T_keys) {
        int64_t off = (((int64_t)b * p.r_max + (key - C)) * p.hkv + kvh) * D + c;
        kv = to_f32<T>(tk[off]);
        vv = to_f32<T>(tv[off]);
      }
      sK[j * DP + c] = kv;
      sV[j * D + c] = vv;
    }
    __syncthreads();
    // scores: lane = key
    const int key = kt + lane;
    float s[kSimtRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kSimtRowsPerWarp; ++r) s[r] = 0.f;
    for (int c = 0; c < D; c += 4) {
      float4 kk = *reinterpret_cast<const float4 *>(&sK[lane * DP + c]);
#pragma unroll
      for (int r = 0; r < kSimtRowsPerWarp; ++r) {
        float4 qq = *reinterpret_cast<const float4 *>(&sQ[(wrow0 + r) * D + c]);
        s[r] = fmaf(qq.x, kk.x, fmaf(qq.y, kk.y, fmaf(qq.z, kk.z, fmaf(qq.w, kk.w, s[r]))));
      }
    }
#pragma unroll
    for (int r = 0; r < kSimtRowsPerWarp; ++r) {
      int rho = row0 + wrow0 + r;
      bool vis = key < T_keys && rho < rows_total && key >= kstart;
      if (vis && key >= C) {
        int node = q0 + rho / g, j = key - C;
        uint32_t w = p.mask_words[((int64_t)b * p.r_max + node) * p.n_words + (j >> 5)];
        vis = (w >> (j & 31)) & 1u;
      }
      float sv = vis ? s[r] * sl2 : -INFINITY;
      float mx = warp_max(sv);
      float m_new = fmaxf(m_r[r], mx);
      float pr = (sv == -INFINITY) ? 0.f : exp2f(sv - m_new);
      float corr = (m_r[r] == -INFINITY) ? 0.f : exp2f(m_r[r] - m_new);
      if (m_new == -INFINITY) corr = 1.f;
      l_r[r] = l_r[r] * corr + warp_sum(pr);
      m_r[r] = m_new;
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[r][t] *= corr;
      sP[(warp * kSimtKeys + lane) * kSimtRowsPerWarp + r] = pr;
    }
    __syncwarp();
    for (int j = 0; j < kSimtKeys; ++j) {
      float4 p0 = *reinterpret_cast<const float4 *>(&sP[(warp * kSimtKeys + j) * kSimtRowsPerWarp]);
      float4 p1 = *reinterpret_cast<const float4 *>(&sP[(warp * kSimtKeys + j) * kSimtRowsPerWarp + 4]);
      float pj[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        int c = lane + 32 * t;
        if (c < D) {
          float vv = sV[j * D + c];
#pragma unroll
          for (int r = 0; r < kSimtRowsPerWarp; ++r) acc[r][t] = fmaf(pj[r], vv, acc[r][t]);
        }
      }
    }
    __syncwarp();
  }
  // epilogue: normalised partial (out, lse) per row
#pragma unroll
  for (int r = 0; r < kSimtRowsPerWarp; ++r) {
    int rho = row0 + wrow0 + r;
    if (rho >= rows_total) {
      if (p.num_splits == 1 && q0 * g + rho < p.r_max * g)
        store_partial<T>(p, 0, b, q0 + rho / g, kvh * g + rho % g, -INFINITY, [&](int) { return 0.f; }, lane);
      continue;
    }
    int node = q0 + rho / g, hq_idx = kvh * g + rho % g;
    float inv = l_r[r] > 0.f ? 1.f / l_r[r] : 0.f;
    float lse2 = l_r[r] > 0.f ? m_r[r] + log2f(l_r[r]) : -INFINITY;
    float lse_n = lse2 * 0.6931471805599453f;
    store_partial<T>(p, split, b, node, hq_idx, lse_n, [&](int t) { return acc[r][t] * inv; }, lane);
  }
}

// Split-KV combine (same math as merge_partials, attention.py:108-124):
// one warp per (b, node, q head).
template <typename T>
__global__ void tree_attn_combine_kernel(TreeAttnParams p) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)p.batch * p.r_max * p.hq;
  if (wid >= total) return;
  const int hq_idx = (int)(wid % p.hq);
  const int node = (int)((wid / p.hq) % p.r_max);
  const int b = (int)(wid / ((int64_t)p.hq * p.r_max));
  const int D = p.head_dim;
  T *out = reinterpret_cast<T *>(p.out) + (((int64_t)b * p.r_max + node) * p.hq + hq_idx) * D;
  const int n_nodes = min(p.n_rows[b], p.r_max);
  if (node < q_first(p, b, n_nodes)) return;  // not a query row of this call
  if (node >= n_nodes) {
    for (int c = lane; c < D; c += 32) out[c] = from_f32<T>(0.f);
    if (p.lse && lane == 0) p.lse[((int64_t)b * p.hq + hq_idx) * p.r_max + node] = -INFINITY;
    return;
  }
  const int64_t stride_split = total;
  const float *lp = p.ws_lse + (((int64_t)b * p.hq + hq_idx) * p.r_max + node);
  const int64_t lstride = (int64_t)p.batch * p.hq * p.r_max;
  float mx = -INFINITY;
  for (int s = 0; s < p.num_splits; ++s) mx = fmaxf(mx, lp[s * lstride]);
  float wsum = 0.f;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int s = 0; s < p.num_splits; ++s) {
    float l = lp[s * lstride];
    if (l == -INFINITY) continue;
    float w = __expf(l - mx);
    wsum += w;
    const float *o = p.ws_out + ((s * stride_split) + wid) * D;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < D) acc[t] = fmaf(w, o[lane + 32 * t], acc[t]);
  }
  float inv = wsum > 0.f ? 1.f / wsum : 0.f;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (lane + 32 * t < D) out[lane + 32 * t] = from_f32<T>(acc[t] * inv);
  if (p.lse && lane == 0)
    p.lse[((int64_t)b * p.hq + hq_idx) * p.r_max + node] = wsum > 0.f ? mx + logf(wsum) : -INFINITY;
}

template <typename T>
int launch_tree_attn_simt(const TreeAttnParams &p, cudaStream_t stream) {
  if (p.head_dim % 4 != 0 || p.head_dim > 256) return SDB_E_UNSUPPORTED;
  const int g = p.hq / p.hkv;
  const int row_tiles = cdiv(p.max_q_nodes * g, kSimtRows);
  dim3 grid(p.num_splits, row_tiles, p.batch * p.hkv);
  const int D = p.head_dim;
  size_t smem = sizeof(float) * ((size_t)kSimtRows * D + (size_t)kSimtKeys * (D + 4) + (size_t)kSimtKeys * D +
                                 (size_t)kSimtWarps * kSimtKeys * kSimtRowsPerWarp);
  cudaFuncSetAttribute(tree_attn_simt_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tree_attn_simt_kernel<T><<<grid, kSimtWarps * 32, smem, stream>>>(p);
  SDB_CHECK_LAUNCH();
  if (p.num_splits > 1) {
    int64_t warps = (int64_t)p.batch * p.r_max * p.hq;
    tree_attn_combine_kernel<T><<<(unsigned)cdiv64(warps * 32, 256), 256, 0, stream>>>(p);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

template int launch_tree_attn_simt<float>(const TreeAttnParams &, cudaStream_t);
template int launch_tree_attn_simt<__nv_bfloat16>(const TreeAttnParams &, cudaStream_t);
template __global__ void tree_attn_combine_kernel<__nv_bfloat16>(TreeAttnParams);
template __global__ void tree_attn_combine_kernel<float>(TreeAttnParams);

int launch_tree_attn_combine_bf16(const TreeAttnParams &p, cudaStream_t stream) {
  int64_t warps = (int64_t)p.batch * p.r_max * p.hq;
  tree_attn_combine_kernel<__nv_bfloat16><<<(unsigned)cdiv64(warps * 32, 256), 256, 0, stream>>>(p);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

}  // namespace sdb

extern "C" int sdb_attend_heads_f64(const double *q, const double *k, const double *v, const uint8_t *mask,
                                    int heads, int m, int n, int head_dim, double scale, double *out, double *lse,
                                    void *stream) {
  if (!q || !out || !lse || heads < 1 || m < 0 || n < 0 || head_dim < 1 || head_dim > 256) return SDB_E_INVALID;
  if (n > 0 && (!k || !v)) return SDB_E_INVALID;
  if (m == 0) return SDB_OK;
  int64_t threads = (int64_t)heads * m * 32;
  sdb::attend_heads_f64_kernel<<<(unsigned)sdb::cdiv64(threads, 128), 128, 0, sdb::as_stream(stream)>>>(
      q, k, v, mask, heads, m, n, head_dim, scale, out, lse);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_merge_partials_f64(const double *outs, const double *lses, int parts, int heads, int m,
                                      int head_dim, double *out, double *lse, int32_t *err, void *stream) {
  if (!outs || !lses || !out || !lse || parts < 1 || heads < 1 || m < 0 || head_dim < 1) return SDB_E_INVALID;
  if (m == 0) return SDB_OK;
  int n = heads * m;
  sdb::merge_partials_f64_kernel<<<sdb::cdiv(n, 128), 128, 0, sdb::as_stream(stream)>>>(
      outs, lses, parts, heads, m, head_dim, out, lse, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
