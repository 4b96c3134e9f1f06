// Internal parameter block shared by the tree-verify attention kernels.
#pragma once

#include "sdb_common.cuh"

namespace sdb {

struct TreeAttnParams {
  const void *q, *k_cache, *v_cache, *tree_k, *tree_v;
  const int32_t *block_table, *ctx_len, *n_rows;
  const int32_t *q_row0;  // [B] first query row (draft-side rectangular attention) or nullptr = 0
  const uint32_t *mask_words;
  void *out;
  float *lse;
  float *ws_out;  // [splits][B][r_max][hq][D]
  float *ws_lse;  // [splits][B][hq][r_max]
  int batch, r_max, n_words, hq, hkv, head_dim, block_size, num_blocks, max_blocks, max_ctx;
  int max_q_nodes;  // query nodes per sequence (<= r_max); plans the row blocks
  int chunk_len;    // iRoPE local chunk: prefix keys [floor(C / chunk) * chunk, C); 0 = all
  int pdl;          // launch the tcgen05 kernel as a programmatic dependent of the previous kernel
  // fused greedy-acceptance scan (idle warp of the pair kernel): packed
  // argmax keys of the fp32 logits rows [B][r_max][vocab] (n_rows gated)
  const float *fa_logits;
  int64_t fa_row_stride, fa_vocab_offset;
  int fa_vocab;
  long long *fa_keys;
  int32_t *err;     // SDB_ERR_CACHE when ctx_len > max_ctx (tcgen05 plan), or nullptr
  int32_t *fa_err;
  float scale;
  int num_splits;
};

// First query row of sequence b: rows [q0, n_rows) attend, keys are all the
// tree rows [0, n_rows) (the draft stage's depth step, engine.py:424-432).
__device__ __forceinline__ int prefix_start(const TreeAttnParams &p, int ctx) {
  return p.chunk_len > 0 ? (ctx / p.chunk_len) * p.chunk_len : 0;
}

__device__ __forceinline__ int q_first(const TreeAttnParams &p, int b, int n_nodes) {
  return p.q_row0 ? min(max(p.q_row0[b], 0), n_nodes) : 0;
}

// Write one row's attention result: the final output when the KV range is
// not split, otherwise the fp32 partial for the combine kernel.
template <typename T, typename F>
__device__ __forceinline__ void store_partial(const TreeAttnParams &p, int split, int b, int node, int hq_idx,
                                              float lse_nat, F &&val, int lane) {
  const int D = p.head_dim;
  if (p.num_splits == 1) {
    T *o = reinterpret_cast<T *>(p.out) + (((int64_t)b * p.r_max + node) * p.hq + hq_idx) * D;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < D) o[lane + 32 * t] = from_f32<T>(val(t));
    if (p.lse && lane == 0) p.lse[((int64_t)b * p.hq + hq_idx) * p.r_max + node] = lse_nat;
  } else {
    const int64_t wid = ((int64_t)b * p.r_max + node) * p.hq + hq_idx;
    const int64_t total = (int64_t)p.batch * p.r_max * p.hq;
    float *o = p.ws_out + (split * total + wid) * D;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < D) o[lane + 32 * t] = val(t);
    if (lane == 0) p.ws_lse[(int64_t)split * total + ((int64_t)b * p.hq + hq_idx) * p.r_max + node] = lse_nat;
  }
}

template <typename T>
int launch_tree_attn_simt(const TreeAttnParams &p, cudaStream_t stream);
int launch_tree_attn_combine_bf16(const TreeAttnParams &p, cudaStream_t stream);
int launch_tree_attn_sm100(const TreeAttnParams &p, int ctas_override, void *workspace, cudaStream_t stream);
int64_t tree_attn_sm100_workspace(const TreeAttnParams &p, int ctas_override);
int tree_attn_sm100_sms(const TreeAttnParams &p, int ctas_override);
int tree_attn_sm100_group(const TreeAttnParams &p, int ctas_override);
bool tree_attn_sm100_supported(const TreeAttnParams &p);

}  // namespace sdb
