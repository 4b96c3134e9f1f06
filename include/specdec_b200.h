/*
 * specdec_b200 -- C ABI of the B200-native EAGLE tree-verification hot path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void*), enqueues work on that stream and returns without a host
 * synchronisation.  No torch types cross this boundary.  Return value: 0 on
 * success, a negative SDB_E* code on bad arguments (nothing is enqueued then);
 * data errors found on the device (invalid parent index, NaN logits, invalid
 * distribution) are reported through the caller-provided int32 `err` words.
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/specdec/<file>:<line>).  The Python host mirror
 * (paper_2508_08192_b200/) keeps the reference's names and error behaviour
 * on top of these calls; INTEGRATION.md shows the ctypes binding.
 *
 * Layout conventions
 *   tree rows   : "augmented" order -- row 0 is the root (last committed
 *                 token), row 1+i is draft node i (engine.py:170-173); any
 *                 parent array with parent[i] in {-1} U [0, i) is accepted.
 *   mask words  : uint32 [B][R][n_words], bit j of row i = row i sees row j
 *                 (LSB = row 0) -- the ancestor-or-self closure.
 *   KV pages    : bf16 [num_blocks][n_kv_heads][block_size][head_dim], one
 *                 pool per layer; block_table int32 [B][max_blocks].
 *   LSE         : natural log, fp32 [B][Hq][R] (reference PartialAttention.lse).
 */
#ifndef SPECDEC_B200_H
#define SPECDEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDB_OK 0
#define SDB_E_INVALID (-1)     /* bad shape / null pointer / unsupported size   */
#define SDB_E_UNSUPPORTED (-2) /* dtype or head_dim not supported by a kernel   */
#define SDB_E_WORKSPACE (-3)   /* workspace too small                           */
#define SDB_E_CUDA (-4)        /* a CUDA launch failed (see sdb_last_cuda_error) */

/* device-side error bits written into `err` words */
#define SDB_ERR_BAD_PARENT 1      /* TreeError: parent must precede node (drafttree.py:31-34) */
#define SDB_ERR_NAN 2             /* ValueError: NaN in logits (numcore.py:47-48)             */
#define SDB_ERR_BAD_DIST 4        /* SamplingError: dist not >= 0 / sum != 1 (sampling.py:47) */
#define SDB_ERR_UNIFORMS 8        /* SamplingError: uniform stream exhausted (sampling.py:179) */
#define SDB_ERR_ALL_MASKED 16     /* AttentionError: row masked in every part (attention.py:117) */
#define SDB_ERR_NO_ALLOWED 32     /* SamplingError: no token allowed (sampling.py:96-97)       */
#define SDB_ERR_CACHE 64          /* CacheError: block pool exhausted / tape or table overflow */
#define SDB_ERR_PLAN 128          /* SamplingError: tree deeper / wider than the host-planned walk */

#define SDB_DTYPE_BF16 0
#define SDB_DTYPE_F32 1
#define SDB_DTYPE_F64 2

int sdb_version(void);
const char *sdb_strerror(int code);
const char *sdb_last_cuda_error(void);

/* Clear `bytes` (a multiple of 4, 4-byte aligned) of device memory on
 * `stream` with a small kernel -- the per-call error words (the reference
 * raises per call: sampling.py:43-49, engine.py:474-475). */
int sdb_clear_async(void *ptr, int64_t bytes, void *stream);

/* ---- K0: tree mask, depth and positions -------------------------------
 * Replaces TreeSpec.__post_init__ depth + validation (drafttree.py:26-35),
 * suffix_mask (drafttree.py:102-111) and the row positions
 * L-2+depth_aug (engine.py:456) / ctx+depth-1 (attention.py:142).
 * parent int32 [B][r_max]; n_rows int32 [B]; ctx_len int32 [B] (may be NULL
 * -> 0).  Outputs mask_words uint32 [B][r_max][n_words], positions int32
 * [B][r_max] (= ctx + depth - 1), depth int32 [B][r_max]; err int32 [B]
 * gets SDB_ERR_BAD_PARENT for an invalid sequence.  Rows >= n_rows are 0. */
int sdb_tree_build(const int32_t *parent, const int32_t *n_rows, const int32_t *ctx_len,
                   int batch, int r_max, int n_words, uint32_t *mask_words,
                   int32_t *positions, int32_t *depth, int32_t *err, void *stream);

/* ---- drop-in attention core (float64, reference precision) ------------
 * Replaces kernels.attend_heads -> _attend_numpy / _attend_numba
 * (kernels.py:40-92, 195-203).  q [heads][m][d], k/v [heads][n][d],
 * mask uint8 [m][n] or NULL (all visible).  out [heads][m][d], lse
 * [heads][m]; fully masked rows give out 0 and lse -inf. */
int sdb_attend_heads_f64(const double *q, const double *k, const double *v,
                         const uint8_t *mask, int heads, int m, int n, int head_dim,
                         double scale, double *out, double *lse, void *stream);

/* Replaces attention.merge_partials (attention.py:108-124).  outs
 * [parts][heads][m][d], lses [parts][heads][m] -> out [heads][m][d], lse
 * [heads][m]; a row masked in every part sets SDB_ERR_ALL_MASKED in err[0]. */
int sdb_merge_partials_f64(const double *outs, const double *lses, int parts, int heads,
                           int m, int head_dim, double *out, double *lse, int32_t *err,
                           void *stream);

/* ---- K1-K3: batched paged GQA tree-verify attention -------------------
 * Replaces, per layer, the attention block of model.forward
 * (model.py:252-272): cache.gather (kvstore.py:235-246) +
 * attend(CausalPrefix) + attend(TreeSuffix(mask)) + merge_attentions
 * (attention.py:92-128), i.e. tree_attention (attention.py:131-151) with
 * GQA (q head h reads kv head h / (hq/hkv)). */
typedef struct sdb_tree_attn_args {
  const void *q;              /* [B][r_max][hq][head_dim]  (dtype)           */
  const void *k_cache;        /* [num_blocks][hkv][block_size][head_dim]     */
  const void *v_cache;
  const int32_t *block_table; /* [B][max_blocks]                             */
  const int32_t *ctx_len;     /* [B] committed rows C = L-1 in the cache      */
  const void *tree_k;         /* [B][r_max][hkv][head_dim] fresh tree K/V     */
  const void *tree_v;
  const uint32_t *mask_words; /* [B][r_max][n_words] from sdb_tree_build      */
  const int32_t *n_rows;      /* [B] valid tree rows (<= r_max)               */
  void *out;                  /* [B][r_max][hq][head_dim] (dtype)             */
  float *lse;                 /* [B][hq][r_max] natural log, may be NULL      */
  void *workspace;            /* split-KV partials, see sdb_tree_attn_workspace */
  int64_t workspace_bytes;
  int batch, r_max, n_words, hq, hkv, head_dim;
  int block_size, num_blocks, max_blocks;
  int max_ctx;                /* upper bound of ctx_len (host-known), sizes the grid */
  float scale;
  int dtype;                  /* SDB_DTYPE_BF16 (tcgen05 path) or SDB_DTYPE_F32 */
  int num_splits;             /* 0 = auto                                     */
  int kernel;                 /* 0 = auto, 1 = tcgen05 (sm_100a), 2 = SIMT    */
  const int32_t *q_row0;      /* [B] or NULL: only rows [q_row0, n_rows) query
                                 (written); keys stay all tree rows [0, n_rows).
                                 The draft stage's depth step: new nodes attend
                                 the carried + new suffix under a rectangular
                                 mask (engine.py:424-432, model.py:265-270) */
  int max_q_nodes;            /* host bound of n_rows - q_row0 over the batch
                                 (sizes the work plan); 0 = r_max            */
  int flags;                  /* SDB_ATTN_FLAG_*                              */
  /* optional fused greedy-acceptance scan (sdb_argmax_keys semantics over the
   * flat rows [batch * r_max] of fp32 logits): when fused_keys is set, the
   * call also produces keys[b * r_max + r] -- inside the CTA-pair attention
   * kernel (an otherwise idle warp streams the logits through TMA while the
   * tensor pipe works), else by a separate launch after it.  Feed the keys
   * to sdb_greedy_walk (replaces argmax_keys_kernel of sdb_accept_greedy). */
  const float *fused_logits;  /* [batch][r_max][row_stride], this rank's vocab slice */
  int64_t fused_row_stride, fused_vocab_offset;
  int fused_vocab;
  int64_t *fused_keys;        /* [batch * r_max]                              */
  int32_t *fused_err;         /* NaN -> SDB_ERR_NAN                           */
  int chunk_len;              /* iRoPE local attention (attention.py:33-40,
                                 76-84): 0 = none; else every tree row sees the
                                 prefix keys [floor(C / chunk) * chunk, C) --
                                 exact when the tree was truncated at the
                                 chunk boundary (truncate_draft_at_boundary,
                                 attention.py:189-206; engine.py:486-487).
                                 tcgen05 path: chunk % 128 == 0 and
                                 chunk % block_size == 0, else SIMT */
  int32_t *err;               /* optional [1]: SDB_ERR_CACHE (OR-ed) when a
                                 sequence's ctx_len exceeds max_ctx -- the
                                 tcgen05 plan covers max_ctx keys, so the keys
                                 past it would be dropped (kvstore.py CacheError
                                 contract: fail, never truncate silently) */
} sdb_tree_attn_args;

/* The kernel launched just before on the stream is sdb_tree_build (the only
 * producer of mask_words this call must wait for): launch the tcgen05 kernel
 * as its programmatic dependent, so its prologue and K/V streaming overlap
 * tree_build (sm_100 PDL; captured as a programmatic graph edge). */
#define SDB_ATTN_FLAG_PDL 1

int64_t sdb_tree_attn_workspace(const sdb_tree_attn_args *a);
/* SMs the launch plan of these arguments occupies (the persistent grid);
 * callers that run independent work concurrently (acceptance) use the rest. */
int sdb_tree_attn_sms(const sdb_tree_attn_args *a);
int sdb_tree_attn(const sdb_tree_attn_args *a, void *stream);

/* ---- K4/K5: greedy (T = 0) acceptance ----------------------------------
 * Replaces target_dist(row, 0, top_p) (sampling.py:87-102, numcore.py:51-55)
 * for every tree row + mss_verify (sampling.py:149-202) at temperature 0,
 * which is exactly the argmax walk.
 *
 * Step 1 (vocab-shardable): per-row packed argmax keys over this rank's
 * vocab slice [vocab_offset, vocab_offset + vocab): int64 key =
 * (int32(orderable(max)) << 32) | (0xFFFFFFFF - global_index) -- signed int64
 * MAX over ranks (NCCL/torch all_reduce MAX) yields the global argmax with the
 * lowest index on ties.  logits [rows][row_stride] of dtype f32 or bf16. */
int sdb_argmax_keys(const void *logits, int dtype, int64_t rows, int vocab, int64_t row_stride,
                    int64_t vocab_offset, int64_t *keys, int32_t *err, void *stream);

/* Step 2: the tree walk on global keys.  parent/tokens int32 [B][r_max]
 * (tokens[b][1+i] = draft token of node i; row 0 unused), keys int64
 * [B][r_max].  Outputs path int32 [B][r_max] (draft-node indices, the
 * reference accepted_path), path_len int32 [B], next_token int64 [B],
 * uniforms_used int32 [B] (= candidates examined + 1, as mss_verify counts). */
int sdb_greedy_walk(const int64_t *keys, const int32_t *parent, const int32_t *n_rows,
                    const int32_t *tokens, int batch, int r_max, int32_t *path,
                    int32_t *path_len, int64_t *next_token, int32_t *uniforms_used,
                    void *stream);

/* Steps 1+2 (single GPU, unsharded vocab).  keys is scratch of
 * batch * r_max * SDB_GREEDY_KEY_SLOTS int64 (small batches split each
 * row's vocabulary over several CTAs, one partial key each). */
#define SDB_GREEDY_KEY_SLOTS 8
int sdb_accept_greedy(const void *logits, int dtype, int batch, int r_max, int vocab,
                      int64_t row_stride, const int32_t *parent, const int32_t *n_rows,
                      const int32_t *tokens, int64_t *keys, int32_t *path, int32_t *path_len,
                      int64_t *next_token, int32_t *uniforms_used, int32_t *err,
                      void *stream);

/* Greedy acceptance over FSM-masked rows (guided decoding: target_dist(row,
 * 0, ., allowed), sampling.py:94-99 -- the argmax of the ALLOWED logits;
 * engine.py:465-475 gives each tree row the FSM state after its token).
 * allowed uint32 [B][r_max][allowed_words], bit j of word w = token 32 w + j
 * allowed; NULL = sdb_accept_greedy (fp32).  A row with no allowed token sets
 * SDB_ERR_NO_ALLOWED.  keys: batch * r_max int64. */
int sdb_accept_greedy_ex(const float *logits, int batch, int r_max, int vocab, int64_t row_stride,
                         const int32_t *parent, const int32_t *n_rows, const int32_t *tokens,
                         const uint32_t *allowed, int allowed_words, int64_t *keys, int32_t *path,
                         int32_t *path_len, int64_t *next_token, int32_t *uniforms_used, int32_t *err,
                         void *stream);

/* ---- K4/K5: stochastic (T > 0) acceptance ------------------------------
 * Replaces target_dist(row, T, top_p) for every tree row, the draft q
 * target_dist(draft_row, T, 1.0) (engine.py:266-269; siblings share their
 * parent's q, engine.py:405-407) and mss_verify (sampling.py:149-202) with
 * uniforms[b][0..] (rank_sliced_uniforms row, engine.py:251-254, 498-503).
 * target/draft logits fp32 [B][r_max][vocab]; uniforms f64 [B][n_uniforms].
 * residual (optional, f32 [B][vocab]) receives the distribution the bonus
 * token was drawn from (MssResult.residual). */
int64_t sdb_accept_stochastic_workspace(int batch, int r_max, int vocab);
int sdb_accept_stochastic(const float *target_logits, const float *draft_logits, int batch,
                          int r_max, int vocab, float temperature, float top_p,
                          const int32_t *parent, const int32_t *n_rows, const int32_t *tokens,
                          const double *uniforms, int n_uniforms, void *workspace,
                          int64_t workspace_bytes, int32_t *path, int32_t *path_len,
                          int64_t *next_token, int32_t *uniforms_used, float *residual,
                          int32_t *err, void *stream);

/* ---- K4/K5 (sharded): vocab-sharded stochastic acceptance ----------------
 * The T > 0 acceptance of sdb_accept_stochastic with the vocabulary split
 * over `world` ranks; same reference semantics
 * (sampling.py:87-202, engine.py:266-269, 405-407, 498-503).  The host runs
 * the phases in order and performs, after the phases marked below, one
 * collective on the named exchange buffer (identical on every rank):
 *   SDB_SH_PARTIALS      -> all-gather xchg_partials into gathered [world][...]
 *   SDB_SH_COMBINE
 *   SDB_SH_NUCLEUS k=0..3 -> all-reduce SUM hist   (only when top_p < 1)
 *   SDB_SH_CUT           -> all-reduce SUM tie     (only when top_p < 1)
 *   SDB_SH_FINISH                                  (only when top_p < 1)
 *   SDB_SH_TOKEN_PQ      -> all-reduce SUM pq
 *   SDB_SH_RESIDUAL k=1..max_children -> all-reduce SUM chain_x (each)
 *   SDB_SH_WALK          -> all-reduce SUM bonus_mass
 *   SDB_SH_PICK          -> all-reduce MAX bonus_token (= next_token)
 * path / path_len / uniforms_used are identical on every rank after WALK /
 * PICK; residual (optional) receives this rank's vocab slice. */
#define SDB_SH_PARTIALS 0
#define SDB_SH_COMBINE 1
#define SDB_SH_NUCLEUS 2
#define SDB_SH_CUT 3
#define SDB_SH_FINISH 4
#define SDB_SH_TOKEN_PQ 5
#define SDB_SH_RESIDUAL 6
#define SDB_SH_WALK 7
#define SDB_SH_PICK 8

/* indices of sdb_sharded_accept_sizes' output (element counts; scratch in bytes) */
#define SDB_SH_BUF_PARTIALS 0     /* f64 */
#define SDB_SH_BUF_GATHERED 1     /* f64 */
#define SDB_SH_BUF_HIST 2         /* f64 */
#define SDB_SH_BUF_TIE 3          /* int32 */
#define SDB_SH_BUF_PQ 4           /* f64 */
#define SDB_SH_BUF_CHAIN_X 5      /* f64 */
#define SDB_SH_BUF_BONUS_MASS 6   /* f64 */
#define SDB_SH_BUF_BONUS_TOKEN 7  /* int64 */
#define SDB_SH_BUF_SCRATCH 8      /* bytes */
#define SDB_SH_N_BUFS 9

typedef struct sdb_sharded_accept_args {
  const float *target_logits; /* [B][r_max][vocab_local]: this rank's vocab slice */
  const float *draft_logits;
  int batch, r_max, vocab_local;
  int64_t vocab_offset, vocab; /* slice start, global vocabulary size      */
  int world, rank;
  float temperature, top_p;
  int max_children;            /* >= children of any node (residual levels) */
  const int32_t *parent, *n_rows, *tokens; /* as sdb_accept_stochastic; tokens global ids */
  const double *uniforms;      /* [B][n_uniforms], identical on every rank   */
  int n_uniforms;
  double *xchg_partials, *gathered, *hist;
  int32_t *tie;
  double *pq, *chain_x, *bonus_mass;
  int64_t *bonus_token;
  void *scratch;               /* private per-rank state                     */
  int64_t scratch_bytes;
  int32_t *path, *path_len, *uniforms_used;
  float *residual;             /* optional [B][vocab_local]                  */
  int32_t *err;
} sdb_sharded_accept_args;

int sdb_sharded_accept_sizes(const sdb_sharded_accept_args *a, int64_t *sizes /* [SDB_SH_N_BUFS] */);
int sdb_sharded_accept_phase(const sdb_sharded_accept_args *a, int phase, int level, void *stream);

/* sdb_accept_stochastic with FSM masks: allowed (as in sdb_accept_greedy_ex)
 * masks row r's target dist AND the q its children were drafted from (the
 * same FSM state, engine.py:266-269, 465-475); NULL = unmasked. */
int sdb_accept_stochastic_ex(const float *target_logits, const float *draft_logits, int batch, int r_max,
                             int vocab, float temperature, float top_p, const int32_t *parent,
                             const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                             int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                             int32_t *path_len, int64_t *next_token, int32_t *uniforms_used, float *residual,
                             int32_t *err, const uint32_t *allowed, int allowed_words, void *stream);

/* Lazy stochastic acceptance: the same results as sdb_accept_stochastic_ex,
 * but only the rows the walk visits are reduced (mss_verify reads the target
 * dist of the nodes on its path and the q of their children only,
 * sampling.py:173-202): `levels` (>= the tree's max depth + 1) rounds of
 * {row stats of each sequence's current node, one walk step}.  Pair it with
 * sdb_stochastic_validate (may run concurrently on another stream) to keep
 * the reference's error behaviour, which checks EVERY row (engine.py:474-475:
 * NaN -> SDB_ERR_NAN, dead FSM row -> SDB_ERR_NO_ALLOWED). */
int sdb_accept_stochastic_lazy(const float *target_logits, const float *draft_logits, int batch, int r_max,
                               int vocab, float temperature, float top_p, const int32_t *parent,
                               const int32_t *n_rows, const int32_t *tokens, const double *uniforms,
                               int n_uniforms, void *workspace, int64_t workspace_bytes, int32_t *path,
                               int32_t *path_len, int64_t *next_token, int32_t *uniforms_used, float *residual,
                               int32_t *err, const uint32_t *allowed, int allowed_words, int levels, void *stream);
int sdb_stochastic_validate(const float *target_logits, const float *draft_logits, int batch, int r_max, int vocab,
                            const int32_t *parent, const int32_t *n_rows, const uint32_t *allowed,
                            int allowed_words, int32_t *err, void *stream);

/* ---- uniforms: device Philox4x64-10 ----------------------------------------
 * Replaces rank_sliced_uniforms (sampling.py:112-124) as the engine consumes
 * it (engine.py:251-254): out[b][i] = element (row, i) of the (padded_batch,
 * width) matrix numpy's Generator(Philox(key=(seeds[b], steps[b]))).random()
 * returns -- bit-identical.  seeds/steps int64 [B] (uint64 bit patterns), out
 * f64 [B][width].  The engine uses row 0, seed = sampler.seed + seq, step =
 * 2*round + 2 for acceptance (engine.py:234-235, 499). */
int sdb_philox_uniforms(const int64_t *seeds, const int64_t *steps, int batch, int64_t row, int width,
                        double *out, void *stream);

/* ---- drop-in sampling ops (float64, reference precision) ---------------
 * target_dist (sampling.py:87-102): logits f64 [rows][vocab] -> dist f64,
 * allowed uint8 [rows][vocab] or NULL (guided-decoding mask, applied first). */
int sdb_target_dist_f64(const double *logits, const uint8_t *allowed, int64_t rows, int vocab,
                        double temperature, double top_p, double *dist, int32_t *err,
                        void *stream);

/* mss_verify on explicit distributions (sampling.py:149-202): parent int32
 * [n] (non-augmented draft tree, ROOT = -1), tokens int32 [n], node_dists f64
 * [n][vocab], target_dists f64 [n+1][vocab], uniforms f64 [n_uniforms].
 * out_path int32 [n], out_scalars int64 [3] = {path_len, next_token,
 * uniforms_used}, residual f64 [vocab]. */
int sdb_mss_verify_f64(const int32_t *parent, const int32_t *tokens, int n_nodes, int vocab,
                       const double *node_dists, const double *target_dists,
                       const double *uniforms, int n_uniforms, int32_t *out_path,
                       int64_t *out_scalars, double *residual, int32_t *err, void *stream);

/* ---- K7: KV write-back ---------------------------------------------------
 * Replaces the bookkeeping write-back (engine.py:504-523): for every layer
 * and sequence, tree rows [0] + [1 + a for a in path[:n_keep-1]] are written
 * to positions ctx_len[b] .. of the sequence's pages
 * (PagedKvCache.write / compact_accepted, kvstore.py:217-233).
 * tree_k/v: bf16 [n_layers][B][r_max][hkv][head_dim]; caches: per layer
 * pool, layer stride layer_stride elements.  n_keep int32 [B] may be NULL
 * (-> path_len + 1).  A position past the sequence's mapped blocks (table
 * entry < 0 or beyond max_blocks: the reference's CacheError "write past
 * allocated blocks", kvstore.py:220-221) is not written and sets SDB_ERR_CACHE in
 * err[0] (err may be NULL). */
int sdb_compact_kv(const void *tree_k, const void *tree_v, void *k_cache, void *v_cache,
                   int64_t cache_layer_stride, const int32_t *block_table, int max_blocks,
                   const int32_t *ctx_len, const int32_t *path, const int32_t *path_len,
                   const int32_t *n_keep, int n_layers, int batch, int r_max, int hkv,
                   int head_dim, int block_size, int elem_bytes, int32_t *err, void *stream);

/* ---- bookkeeping either side of the step ----------
 * Draft-cache write-back (engine.py:524-531): rows path[:n_keep-1] of the
 * draft's carried suffix K/V suffix_k/v [n_layers][B][n_src][hkv][head_dim]
 * (realized draft nodes in node order, no root row) written at positions
 * ctx_len[b] + 1 .. (L; the alignment token already sits at L - 1).  Unmapped
 * positions are skipped with SDB_ERR_CACHE, as in sdb_compact_kv. */
int sdb_compact_draft_kv(const void *suffix_k, const void *suffix_v, void *k_cache, void *v_cache,
                         int64_t cache_layer_stride, const int32_t *block_table, int max_blocks,
                         const int32_t *ctx_len, const int32_t *path, const int32_t *path_len,
                         const int32_t *n_keep, int n_layers, int batch, int r_max, int n_src, int hkv,
                         int head_dim, int block_size, int elem_bytes, int32_t *err, void *stream);

/* Hidden tape append (engine.py:532-533 -> HiddenTape.append_rows,
 * kvstore.py:405-409): rows [0] + [1 + a for a in path[:n_keep-1]] of hidden
 * [B][r_max][row_bytes] appended to tape [B][tape_cap][row_bytes] at
 * tape_len[b], which advances; overflow sets SDB_ERR_CACHE. */
int sdb_tape_append(const void *hidden, void *tape, int64_t tape_cap, int32_t *tape_len, const int32_t *path,
                    const int32_t *path_len, const int32_t *n_keep, int batch, int r_max, int row_bytes,
                    int32_t *err, void *stream);

/* Device block allocator (PagedKvCache.ensure / alloc_for_step / rewind,
 * kvstore.py:195-203, 248-258): free_stack int32 [num_blocks] holds free block
 * ids in [0, *free_top); n_mapped int32 [B] counts each sequence's mapped
 * blocks (block_table[b][0..n_mapped)).  sdb_paged_alloc maps blocks until
 * n_mapped * block_size >= need[b] (alloc_for_step: need = length +
 * n_draft_nodes + 1); exhaustion sets SDB_ERR_CACHE.  sdb_paged_rewind
 * unmaps the blocks beyond ceil(new_len / block_size) (entries -> -1). */
int sdb_paged_alloc(int32_t *block_table, int max_blocks, int32_t *n_mapped, const int32_t *need, int batch,
                    int block_size, int32_t *free_stack, int32_t *free_top, int32_t *err, void *stream);
int sdb_paged_rewind(int32_t *block_table, int max_blocks, int32_t *n_mapped, const int32_t *new_len, int batch,
                     int block_size, int32_t *free_stack, int32_t *free_top, void *stream);

/* Generic row scatter / gather on one sequence's pages (PagedKvCache.write /
 * gather, kvstore.py:217-225, 235-246): rows [n][hkv*head_dim] <-> pages at
 * positions start.. .  elem_bytes 2, 4 or 8. */
int sdb_paged_write(void *pool, const int32_t *block_table, int64_t start, const void *rows,
                    int64_t n, int hkv, int head_dim, int block_size, int elem_bytes,
                    void *stream);
int sdb_paged_gather(const void *pool, const int32_t *block_table, int64_t start, void *rows,
                     int64_t n, int hkv, int head_dim, int block_size, int elem_bytes,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECDEC_B200_H */
