// K0: on-device tree structure -- depth, validation, ancestor-or-self mask
// words and absolute positions from a parent array.
//
// Reference: TreeSpec.__post_init__ (drafttree.py:26-35), suffix_mask
// (drafttree.py:102-111), positions L-2+depth_aug (engine.py:456) =
// ctx+depth-1 (attention.py:142).
//
// One warp per sequence.  Parents are staged in shared memory; each lane owns
// rows lane, lane+32, ... and builds its row by walking the ancestor chain
// (O(depth) per row, fully parallel across rows -- no row-to-row dependency).
#include "sdb_common.cuh"

namespace sdb {

constexpr int kTreeMaxRows = 4096;

__global__ void __launch_bounds__(128) tree_build_kernel(
    const int32_t *__restrict__ parent, const int32_t *__restrict__ n_rows,
    const int32_t *__restrict__ ctx_len, int batch, int r_max, int n_words,
    uint32_t *__restrict__ mask_words, int32_t *__restrict__ positions,
    int32_t *__restrict__ depth_out, int32_t *__restrict__ err) {
  extern __shared__ int32_t smem_par[];  // [warps][r_max]
  // a programmatic-dependent attention launch may start its prologue now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + warp;
  if (b >= batch) return;
  int32_t *par = smem_par + warp * r_max;
  const int n = min(max(n_rows[b], 0), r_max);
  const int ctx = ctx_len ? ctx_len[b] : 0;
  const int32_t *pb = parent + (int64_t)b * r_max;
  bool bad = false;
  for (int i = lane; i < r_max; i += 32) {
    int p = i < n ? pb[i] : -1;
    if (i < n && !(p == -1 || (p >= 0 && p < i))) bad = true;
    par[i] = p;
  }
  bad = __any_sync(SDB_FULL_MASK, bad);
  __syncwarp();
  uint32_t *mw = mask_words + (int64_t)b * r_max * n_words;
  for (int i = lane; i < r_max; i += 32) {
    int d = 0;
    if (i < n && !bad) {
      for (int w = 0; w < n_words; ++w) {
        uint32_t word = 0;
        int lo = w * 32, hi = lo + 32;
        if (lo <= i) {
          // walk i, parent(i), ... ; parents strictly decrease so stop below lo
          for (int a = i; a >= lo; a = par[a]) {
            if (a < hi) word |= 1u << (a - lo);
            if (par[a] < 0) break;
          }
        }
        mw[(int64_t)i * n_words + w] = word;
      }
      for (int a = i; a >= 0; a = par[a]) ++d;
    } else {
      for (int w = 0; w < n_words; ++w) mw[(int64_t)i * n_words + w] = 0u;
    }
    if (depth_out) depth_out[(int64_t)b * r_max + i] = d;
    if (positions) positions[(int64_t)b * r_max + i] = d > 0 ? ctx + d - 1 : 0;
  }
  if (lane == 0 && err) err[b] = bad ? SDB_ERR_BAD_PARENT : 0;
}

}  // namespace sdb

extern "C" int sdb_tree_build(const int32_t *parent, const int32_t *n_rows, const int32_t *ctx_len,
                              int batch, int r_max, int n_words, uint32_t *mask_words,
                              int32_t *positions, int32_t *depth, int32_t *err, void *stream) {
  if (batch < 0 || r_max < 1 || r_max > sdb::kTreeMaxRows || n_words < sdb::cdiv(r_max, 32) || !parent ||
      !n_rows || !mask_words)
    return SDB_E_INVALID;
  if (batch == 0) return SDB_OK;
  const int warps = 4;
  dim3 grid(sdb::cdiv(batch, warps));
  size_t smem = (size_t)warps * r_max * sizeof(int32_t);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(sdb::tree_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  sdb::tree_build_kernel<<<grid, warps * 32, smem, sdb::as_stream(stream)>>>(
      parent, n_rows, ctx_len, batch, r_max, n_words, mask_words, positions, depth, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
