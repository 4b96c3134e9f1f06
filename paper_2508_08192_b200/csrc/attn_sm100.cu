// tcgen05 / TMEM / TMA tree-verify attention for sm_100a (work in progress:
// the dispatcher falls back to the SIMT kernel until this path is enabled).
#include "attn_internal.cuh"

namespace sdb {
bool tree_attn_sm100_supported(const TreeAttnParams &) { return false; }
int launch_tree_attn_sm100(const TreeAttnParams &, cudaStream_t) { return SDB_E_UNSUPPORTED; }
}  // namespace sdb
