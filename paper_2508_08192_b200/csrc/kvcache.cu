// K7: paged KV write-back of the accepted path, plus the generic per-sequence
// row scatter/gather of PagedKvCache.
//
// Reference: engine.py:504-523 (rows = [0] + [1+a for a in path[:n_keep-1]]
// written at L-1 = ctx_len for every layer), PagedKvCache.write / gather /
// compact_accepted (kvstore.py:207-246).  Device page layout
// [num_blocks][hkv][block_size][head_dim]: one (page, head) slab per row of
// head_dim elements, so every copy here is a 16-byte-vectorised memcpy of
// head_dim*elem_bytes per (row, head).
#include "sdb_common.cuh"

namespace sdb {

// Page of position pos of sequence b, or -1 when the position lies past the
// sequence's mapped blocks (unmapped table entry or beyond max_blocks).
__device__ __forceinline__ int mapped_page(const int32_t *__restrict__ block_table, int b, int max_blocks,
                                           int64_t pos, int block_size) {
  if (pos < 0 || pos / block_size >= max_blocks) return -1;
  return block_table[(int64_t)b * max_blocks + pos / block_size];
}

// One CTA per (row slot, sequence, layer); threads stride over hkv*head_dim
// in 16-byte chunks, K and V in the same pass.
__global__ void compact_kv_kernel(const uint8_t *__restrict__ tree_k, const uint8_t *__restrict__ tree_v,
                                  uint8_t *__restrict__ k_cache, uint8_t *__restrict__ v_cache,
                                  int64_t layer_stride_bytes, const int32_t *__restrict__ block_table,
                                  int max_blocks, const int32_t *__restrict__ ctx_len,
                                  const int32_t *__restrict__ path, const int32_t *__restrict__ path_len,
                                  const int32_t *__restrict__ n_keep, int batch, int r_max, int hkv,
                                  int row_bytes, int block_size, int32_t *__restrict__ err) {
  const int slot = blockIdx.x, b = blockIdx.y, layer = blockIdx.z;
  int len = path_len[b];
  int keep = n_keep ? n_keep[b] : len + 1;
  int n_write = min(keep - 1, len) + 1;  // root + write_path
  if (slot >= n_write) return;
  int row = slot == 0 ? 0 : 1 + path[(int64_t)b * r_max + slot - 1];
  int64_t pos = (int64_t)ctx_len[b] + slot;
  int page = mapped_page(block_table, b, max_blocks, pos, block_size);
  if (page < 0) {  // CacheError "write past allocated blocks" (kvstore.py:220-221)
    if (threadIdx.x == 0 && layer == 0 && err) atomicOr(err, SDB_ERR_CACHE);
    return;
  }
  int off = (int)(pos % block_size);
  const int64_t src_row = (((int64_t)layer * batch + b) * r_max + row) * hkv;  // in units of head rows
  const int chunks = row_bytes / 16;
  for (int idx = threadIdx.x; idx < hkv * chunks; idx += blockDim.x) {
    int h = idx / chunks, c = idx % chunks;
    int64_t src = (src_row + h) * row_bytes + (int64_t)c * 16;
    int64_t dst = layer * layer_stride_bytes + ((((int64_t)page * hkv + h) * block_size + off) * row_bytes) +
                  (int64_t)c * 16;
    *reinterpret_cast<int4 *>(k_cache + dst) = *reinterpret_cast<const int4 *>(tree_k + src);
    *reinterpret_cast<int4 *>(v_cache + dst) = *reinterpret_cast<const int4 *>(tree_v + src);
  }
}

template <bool kWrite>
__global__ void paged_rows_kernel(uint8_t *__restrict__ pool, const int32_t *__restrict__ block_table,
                                  int64_t start, uint8_t *__restrict__ rows, int64_t n, int hkv,
                                  int row_bytes, int block_size) {
  const int chunks = row_bytes / 16;
  const int64_t total = n * hkv * chunks;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx / (hkv * chunks);
    int rem = (int)(idx % (hkv * chunks));
    int h = rem / chunks, c = rem % chunks;
    int64_t pos = start + r;
    int page = block_table[pos / block_size];
    int off = (int)(pos % block_size);
    int64_t pidx = (((int64_t)page * hkv + h) * block_size + off) * row_bytes + (int64_t)c * 16;
    int64_t ridx = (r * hkv + h) * row_bytes + (int64_t)c * 16;
    if (kWrite)
      *reinterpret_cast<int4 *>(pool + pidx) = *reinterpret_cast<const int4 *>(rows + ridx);
    else
      *reinterpret_cast<int4 *>(rows + ridx) = *reinterpret_cast<const int4 *>(pool + pidx);
  }
}

}  // namespace sdb

extern "C" int sdb_compact_kv(const void *tree_k, const void *tree_v, void *k_cache, void *v_cache,
                              int64_t cache_layer_stride, const int32_t *block_table, int max_blocks,
                              const int32_t *ctx_len, const int32_t *path, const int32_t *path_len,
                              const int32_t *n_keep, int n_layers, int batch, int r_max, int hkv,
                              int head_dim, int block_size, int elem_bytes, int32_t *err, void *stream) {
  if (!tree_k || !tree_v || !k_cache || !v_cache || !block_table || !ctx_len || !path || !path_len)
    return SDB_E_INVALID;
  if (n_layers < 1 || batch < 0 || r_max < 1 || hkv < 1 || head_dim < 1 || block_size < 1)
    return SDB_E_INVALID;
  int row_bytes = head_dim * elem_bytes;
  if (row_bytes % 16 != 0) return SDB_E_UNSUPPORTED;
  if (batch == 0) return SDB_OK;
  dim3 grid(r_max, batch, n_layers);
  int threads = min(256, max(32, hkv * (row_bytes / 16)));
  threads = (threads + 31) / 32 * 32;
  sdb::compact_kv_kernel<<<grid, threads, 0, sdb::as_stream(stream)>>>(
      (const uint8_t *)tree_k, (const uint8_t *)tree_v, (uint8_t *)k_cache, (uint8_t *)v_cache,
      cache_layer_stride * elem_bytes, block_table, max_blocks, ctx_len, path, path_len, n_keep, batch, r_max,
      hkv, row_bytes, block_size, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

static int paged_rows(bool write, void *pool, const int32_t *block_table, int64_t start, void *rows, int64_t n,
                      int hkv, int head_dim, int block_size, int elem_bytes, void *stream) {
  if (!pool || !block_table || !rows || n < 0 || start < 0 || hkv < 1 || head_dim < 1 || block_size < 1)
    return SDB_E_INVALID;
  int row_bytes = head_dim * elem_bytes;
  if (row_bytes % 16 != 0) return SDB_E_UNSUPPORTED;
  if (n == 0) return SDB_OK;
  int64_t total = n * hkv * (row_bytes / 16);
  int threads = 256;
  int blocks = (int)std::min<int64_t>(sdb::cdiv64(total, threads), 4096);
  if (write)
    sdb::paged_rows_kernel<true><<<blocks, threads, 0, sdb::as_stream(stream)>>>(
        (uint8_t *)pool, block_table, start, (uint8_t *)rows, n, hkv, row_bytes, block_size);
  else
    sdb::paged_rows_kernel<false><<<blocks, threads, 0, sdb::as_stream(stream)>>>(
        (uint8_t *)pool, block_table, start, (uint8_t *)rows, n, hkv, row_bytes, block_size);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_paged_write(void *pool, const int32_t *block_table, int64_t start, const void *rows,
                               int64_t n, int hkv, int head_dim, int block_size, int elem_bytes, void *stream) {
  return paged_rows(true, pool, block_table, start, const_cast<void *>(rows), n, hkv, head_dim, block_size,
                    elem_bytes, stream);
}

extern "C" int sdb_paged_gather(const void *pool, const int32_t *block_table, int64_t start, void *rows,
                                int64_t n, int hkv, int head_dim, int block_size, int elem_bytes,
                                void *stream) {
  return paged_rows(false, const_cast<void *>(pool), block_table, start, rows, n, hkv, head_dim, block_size,
                    elem_bytes, stream);
}

// ---------------------------------------------------------------------------
// Bookkeeping either side of the verify step
// ---------------------------------------------------------------------------
namespace sdb {

// Draft-cache write-back (engine.py:524-531): rows write_path =
// path[:n_keep-1] of the draft's carried suffix K/V (realized draft nodes, no
// root row) at positions ctx_len + 1 .. (the draft cache holds the root --
// the alignment token -- at ctx_len = L - 1 already).
__global__ void compact_draft_kv_kernel(const uint8_t *__restrict__ suf_k, const uint8_t *__restrict__ suf_v,
                                        uint8_t *__restrict__ k_cache, uint8_t *__restrict__ v_cache,
                                        int64_t layer_stride_bytes, const int32_t *__restrict__ block_table,
                                        int max_blocks, const int32_t *__restrict__ ctx_len,
                                        const int32_t *__restrict__ path, const int32_t *__restrict__ path_len,
                                        const int32_t *__restrict__ n_keep, int batch, int r_max, int n_src,
                                        int hkv, int row_bytes, int block_size, int32_t *__restrict__ err) {
  const int slot = blockIdx.x, b = blockIdx.y, layer = blockIdx.z;
  const int len = path_len[b];
  const int keep = n_keep ? n_keep[b] : len + 1;
  if (slot >= min(keep - 1, len)) return;
  const int row = path[(int64_t)b * r_max + slot];
  const int64_t pos = (int64_t)ctx_len[b] + 1 + slot;
  const int page = mapped_page(block_table, b, max_blocks, pos, block_size);
  if (page < 0) {
    if (threadIdx.x == 0 && layer == 0 && err) atomicOr(err, SDB_ERR_CACHE);
    return;
  }
  const int off = (int)(pos % block_size);
  const int64_t src_row = (((int64_t)layer * batch + b) * n_src + row) * hkv;
  const int chunks = row_bytes / 16;
  for (int idx = threadIdx.x; idx < hkv * chunks; idx += blockDim.x) {
    const int h = idx / chunks, c = idx % chunks;
    const int64_t src = (src_row + h) * row_bytes + (int64_t)c * 16;
    const int64_t dst = layer * layer_stride_bytes + ((((int64_t)page * hkv + h) * block_size + off) * row_bytes) +
                        (int64_t)c * 16;
    *reinterpret_cast<int4 *>(k_cache + dst) = *reinterpret_cast<const int4 *>(suf_k + src);
    *reinterpret_cast<int4 *>(v_cache + dst) = *reinterpret_cast<const int4 *>(suf_v + src);
  }
}

// Hidden tape append (engine.py:532-533, HiddenTape.append_rows
// kvstore.py:405-409): rows [0] + [1 + a for a in write_path] of the
// verify step's hidden states appended at tape_len[b]; tape_len advances.
__global__ void tape_append_kernel(const uint8_t *__restrict__ hidden, uint8_t *__restrict__ tape, int64_t tape_cap,
                                   int32_t *__restrict__ tape_len, const int32_t *__restrict__ path,
                                   const int32_t *__restrict__ path_len, const int32_t *__restrict__ n_keep,
                                   int r_max, int row_bytes, int32_t *__restrict__ err) {
  const int slot = blockIdx.x, b = blockIdx.y;
  const int len = path_len[b];
  const int keep = n_keep ? n_keep[b] : len + 1;
  const int n_write = min(keep - 1, len) + 1;
  const int base = tape_len[b];
  if (slot >= n_write) return;
  if (base + n_write > tape_cap) {
    if (slot == 0 && threadIdx.x == 0) atomicOr(err, SDB_ERR_CACHE);
    return;
  }
  const int row = slot == 0 ? 0 : 1 + path[(int64_t)b * r_max + slot - 1];
  const uint8_t *src = hidden + ((int64_t)b * r_max + row) * row_bytes;
  uint8_t *dst = tape + ((int64_t)b * tape_cap + base + slot) * row_bytes;
  for (int c = threadIdx.x; c < row_bytes / 16; c += blockDim.x)
    reinterpret_cast<int4 *>(dst)[c] = reinterpret_cast<const int4 *>(src)[c];
}

__global__ void tape_advance_kernel(int32_t *__restrict__ tape_len, int64_t tape_cap,
                                    const int32_t *__restrict__ path_len, const int32_t *__restrict__ n_keep,
                                    int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int len = path_len[b];
  const int keep = n_keep ? n_keep[b] : len + 1;
  const int n_write = min(keep - 1, len) + 1;
  if (tape_len[b] + n_write <= tape_cap) tape_len[b] += n_write;
}

// Device block allocator (PagedKvCache.ensure / alloc_for_step / rewind,
// kvstore.py:195-203, 248-258): a free stack of block ids (top = count) and
// per-sequence mapped-block counts.  alloc: map blocks until
// n_mapped * bs >= need[b]; rewind: unmap blocks beyond ceil(new_len / bs).
// One thread per sequence; the stack is shared through atomics (block ids
// differ from the reference's list order; the logical mapping does not).
__global__ void paged_alloc_kernel(int32_t *__restrict__ block_table, int max_blocks, int32_t *__restrict__ n_mapped,
                                   const int32_t *__restrict__ need, int batch, int block_size,
                                   int32_t *__restrict__ free_stack, int32_t *__restrict__ free_top,
                                   int32_t *__restrict__ err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int want = min(max_blocks, (need[b] + block_size - 1) / block_size);
  if ((int64_t)need[b] > (int64_t)max_blocks * block_size) atomicOr(err, SDB_ERR_CACHE);
  int have = n_mapped[b];
  while (have < want) {
    const int t = atomicSub(free_top, 1) - 1;
    if (t < 0) {  // pool exhausted (CacheError "block pool exhausted")
      atomicAdd(free_top, 1);
      atomicOr(err, SDB_ERR_CACHE);
      break;
    }
    block_table[(int64_t)b * max_blocks + have++] = free_stack[t];
  }
  n_mapped[b] = have;
}

__global__ void paged_rewind_kernel(int32_t *__restrict__ block_table, int max_blocks, int32_t *__restrict__ n_mapped,
                                    const int32_t *__restrict__ new_len, int batch, int block_size,
                                    int32_t *__restrict__ free_stack, int32_t *__restrict__ free_top) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int keep = (new_len[b] + block_size - 1) / block_size;
  const int have = n_mapped[b];
  if (have <= keep) return;
  const int t = atomicAdd(free_top, have - keep);
  for (int i = keep; i < have; ++i) {
    free_stack[t + i - keep] = block_table[(int64_t)b * max_blocks + i];
    block_table[(int64_t)b * max_blocks + i] = -1;
  }
  n_mapped[b] = keep;
}

}  // namespace sdb

extern "C" int sdb_compact_draft_kv(const void *suffix_k, const void *suffix_v, void *k_cache, void *v_cache,
                                    int64_t cache_layer_stride, const int32_t *block_table, int max_blocks,
                                    const int32_t *ctx_len, const int32_t *path, const int32_t *path_len,
                                    const int32_t *n_keep, int n_layers, int batch, int r_max, int n_src, int hkv,
                                    int head_dim, int block_size, int elem_bytes, int32_t *err, void *stream) {
  if (!suffix_k || !suffix_v || !k_cache || !v_cache || !block_table || !ctx_len || !path || !path_len ||
      n_layers < 1 || batch < 0 || r_max < 1 || n_src < 1 || hkv < 1 || block_size < 1 || max_blocks < 1)
    return SDB_E_INVALID;
  const int row_bytes = head_dim * elem_bytes;
  if (row_bytes % 16 != 0) return SDB_E_UNSUPPORTED;
  if (batch == 0) return SDB_OK;
  dim3 grid(r_max, batch, n_layers);
  sdb::compact_draft_kv_kernel<<<grid, 128, 0, sdb::as_stream(stream)>>>(
      (const uint8_t *)suffix_k, (const uint8_t *)suffix_v, (uint8_t *)k_cache, (uint8_t *)v_cache,
      cache_layer_stride * elem_bytes, block_table, max_blocks, ctx_len, path, path_len, n_keep, batch, r_max, n_src,
      hkv, row_bytes, block_size, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_tape_append(const void *hidden, void *tape, int64_t tape_cap, int32_t *tape_len,
                               const int32_t *path, const int32_t *path_len, const int32_t *n_keep, int batch,
                               int r_max, int row_bytes, int32_t *err, void *stream) {
  if (!hidden || !tape || !tape_len || !path || !path_len || !err || batch < 0 || r_max < 1 || tape_cap < 1 ||
      row_bytes < 16 || row_bytes % 16 != 0)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  cudaStream_t s = sdb::as_stream(stream);
  sdb::tape_append_kernel<<<dim3(r_max, batch), 128, 0, s>>>((const uint8_t *)hidden, (uint8_t *)tape, tape_cap,
                                                            tape_len, path, path_len, n_keep, r_max, row_bytes, err);
  SDB_CHECK_LAUNCH();
  sdb::tape_advance_kernel<<<(batch + 127) / 128, 128, 0, s>>>(tape_len, tape_cap, path_len, n_keep, batch);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_paged_alloc(int32_t *block_table, int max_blocks, int32_t *n_mapped, const int32_t *need,
                               int batch, int block_size, int32_t *free_stack, int32_t *free_top, int32_t *err,
                               void *stream) {
  if (!block_table || !n_mapped || !need || !free_stack || !free_top || !err || batch < 0 || max_blocks < 1 ||
      block_size < 1)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  sdb::paged_alloc_kernel<<<(batch + 127) / 128, 128, 0, sdb::as_stream(stream)>>>(
      block_table, max_blocks, n_mapped, need, batch, block_size, free_stack, free_top, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_paged_rewind(int32_t *block_table, int max_blocks, int32_t *n_mapped, const int32_t *new_len,
                                int batch, int block_size, int32_t *free_stack, int32_t *free_top, void *stream) {
  if (!block_table || !n_mapped || !new_len || !free_stack || !free_top || batch < 0 || max_blocks < 1 ||
      block_size < 1)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  sdb::paged_rewind_kernel<<<(batch + 127) / 128, 128, 0, sdb::as_stream(stream)>>>(
      block_table, max_blocks, n_mapped, new_len, batch, block_size, free_stack, free_top);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
