// C ABI of the batched tree-verify attention: argument checks, split-KV
// sizing, workspace carving and kernel selection (tcgen05 for bf16/d=128,
// SIMT otherwise).
#include "attn_internal.cuh"

namespace sdb {

static int auto_splits(const sdb_tree_attn_args *a, int rows_per_cta) {
  const int g = a->hq / a->hkv;
  const int qn = (a->max_q_nodes > 0 && a->max_q_nodes < a->r_max) ? a->max_q_nodes : a->r_max;
  const int row_tiles = cdiv(qn * g, rows_per_cta);
  const int64_t units = (int64_t)a->batch * a->hkv * row_tiles;
  const int max_ctx = a->max_ctx > 0 ? a->max_ctx : a->max_blocks * a->block_size;
  const int target = 2 * num_sms();
  int s = (int)cdiv64(target, units);
  // keep at least ~512 keys per split
  int cap = max(1, (max_ctx + a->r_max) / 512);
  return max(1, min(s, min(cap, 64)));
}

static bool fill_params(const sdb_tree_attn_args *a, TreeAttnParams &p) {
  p.q = a->q;
  p.k_cache = a->k_cache;
  p.v_cache = a->v_cache;
  p.tree_k = a->tree_k;
  p.tree_v = a->tree_v;
  p.block_table = a->block_table;
  p.ctx_len = a->ctx_len;
  p.n_rows = a->n_rows;
  p.q_row0 = a->q_row0;
  p.max_q_nodes = (a->max_q_nodes > 0 && a->max_q_nodes < a->r_max) ? a->max_q_nodes : a->r_max;
  p.pdl = (a->flags & SDB_ATTN_FLAG_PDL) != 0;
  p.chunk_len = a->chunk_len > 0 ? a->chunk_len : 0;
  p.fa_logits = nullptr;
  p.fa_keys = nullptr;
  p.fa_err = nullptr;
  p.err = a->err;
  p.mask_words = a->mask_words;
  p.out = a->out;
  p.lse = a->lse;
  p.batch = a->batch;
  p.r_max = a->r_max;
  p.n_words = a->n_words;
  p.hq = a->hq;
  p.hkv = a->hkv;
  p.head_dim = a->head_dim;
  p.block_size = a->block_size;
  p.num_blocks = a->num_blocks;
  p.max_blocks = a->max_blocks;
  p.max_ctx = a->max_ctx > 0 ? a->max_ctx : a->max_blocks * a->block_size;
  p.scale = a->scale;
  return true;
}

static bool use_sm100(const sdb_tree_attn_args *a, const TreeAttnParams &p) {
  if (a->kernel == 2) return false;
  if (a->dtype != SDB_DTYPE_BF16) return false;
  return tree_attn_sm100_supported(p);
}

static int64_t workspace_for(const TreeAttnParams &p, bool sm100, int ctas_override) {
  if (sm100) return tree_attn_sm100_workspace(p, ctas_override);
  if (p.num_splits <= 1) return 0;
  const int64_t rows = (int64_t)p.batch * p.r_max * p.hq;
  return (int64_t)p.num_splits * rows * (p.head_dim + 1) * (int64_t)sizeof(float) + 256;
}

static int resolve(const sdb_tree_attn_args *a, TreeAttnParams &p, bool &sm100) {
  if (!a || !a->q || !a->k_cache || !a->v_cache || !a->block_table || !a->ctx_len || !a->tree_k || !a->tree_v ||
      !a->mask_words || !a->n_rows || !a->out)
    return SDB_E_INVALID;
  if (a->batch < 0 || a->r_max < 1 || a->hq < 1 || a->hkv < 1 || a->hq % a->hkv != 0 || a->head_dim < 1 ||
      a->block_size < 1 || a->max_blocks < 1 || a->n_words < cdiv(a->r_max, 32))
    return SDB_E_INVALID;
  if (a->dtype != SDB_DTYPE_BF16 && a->dtype != SDB_DTYPE_F32) return SDB_E_UNSUPPORTED;
  fill_params(a, p);
  p.num_splits = 1;
  sm100 = use_sm100(a, p);
  if (a->kernel == 1 && !sm100) return SDB_E_UNSUPPORTED;
  // SIMT: uniform split-KV; tcgen05: num_splits overrides the persistent CTA count
  p.num_splits = sm100 ? 1 : (a->num_splits > 0 ? a->num_splits : auto_splits(a, 32));
  return SDB_OK;
}

}  // namespace sdb

extern "C" int64_t sdb_tree_attn_workspace(const sdb_tree_attn_args *a) {
  sdb::TreeAttnParams p;
  bool sm100 = false;
  int rc = sdb::resolve(a, p, sm100);
  if (rc != SDB_OK) return rc;
  return sdb::workspace_for(p, sm100, a->num_splits);
}

extern "C" int sdb_tree_attn_sms(const sdb_tree_attn_args *a) {
  sdb::TreeAttnParams p;
  bool sm100 = false;
  int rc = sdb::resolve(a, p, sm100);
  if (rc != SDB_OK) return rc;
  if (sm100) return sdb::tree_attn_sm100_sms(p, a->num_splits);
  return sdb::num_sms();  // SIMT: a full-device grid
}

extern "C" int sdb_tree_attn(const sdb_tree_attn_args *a, void *stream) {
  sdb::TreeAttnParams p;
  bool sm100 = false;
  int rc = sdb::resolve(a, p, sm100);
  if (rc != SDB_OK) return rc;
  if (a->batch == 0) return SDB_OK;
  int64_t need = sdb::workspace_for(p, sm100, a->num_splits);
  if (need > 0) {
    if (!a->workspace || a->workspace_bytes < need) return SDB_E_WORKSPACE;
  }
  cudaStream_t s = sdb::as_stream(stream);
  // fused greedy acceptance scan: inside the pair kernel when it runs,
  // otherwise a separate argmax launch right after the attention
  bool fa_separate = false;
  if (a->fused_keys) {
    const bool ok = a->fused_logits && a->fused_vocab > 0 && a->fused_row_stride >= a->fused_vocab &&
                    a->fused_vocab_offset >= 0 && a->fused_vocab_offset + a->fused_vocab <= 0xFFFFFFFFll;
    if (!ok) return SDB_E_INVALID;
    const bool vec = (a->fused_vocab % 4) == 0 && (a->fused_row_stride % 4) == 0 &&
                     ((uintptr_t)a->fused_logits % 16) == 0;
    if (sm100 && vec && sdb::tree_attn_sm100_group(p, a->num_splits) == 2) {
      p.fa_logits = reinterpret_cast<const float *>(a->fused_logits);
      p.fa_row_stride = a->fused_row_stride;
      p.fa_vocab = a->fused_vocab;
      p.fa_vocab_offset = a->fused_vocab_offset;
      p.fa_keys = reinterpret_cast<long long *>(a->fused_keys);
      p.fa_err = a->fused_err;
    } else {
      fa_separate = true;
    }
  }
  if (sm100) {
    rc = sdb::launch_tree_attn_sm100(p, a->num_splits, a->workspace, s);
    if (rc != SDB_OK || !fa_separate) return rc;
    return sdb_argmax_keys(a->fused_logits, SDB_DTYPE_F32, (int64_t)a->batch * a->r_max, a->fused_vocab,
                           a->fused_row_stride, a->fused_vocab_offset, a->fused_keys, a->fused_err, stream);
  }
  if (need > 0) {
    const int64_t rows = (int64_t)p.batch * p.r_max * p.hq;
    p.ws_out = reinterpret_cast<float *>(a->workspace);
    p.ws_lse = p.ws_out + (int64_t)p.num_splits * rows * p.head_dim;
  } else {
    p.ws_out = nullptr;
    p.ws_lse = nullptr;
  }
  rc = a->dtype == SDB_DTYPE_BF16 ? sdb::launch_tree_attn_simt<__nv_bfloat16>(p, s)
                                  : sdb::launch_tree_attn_simt<float>(p, s);
  if (rc != SDB_OK || !fa_separate) return rc;
  return sdb_argmax_keys(a->fused_logits, SDB_DTYPE_F32, (int64_t)a->batch * a->r_max, a->fused_vocab,
                         a->fused_row_stride, a->fused_vocab_offset, a->fused_keys, a->fused_err, stream);
}
