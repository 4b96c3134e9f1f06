// Tree-verify attention on CTA pairs: tcgen05.mma.cta_group::2 (M = 256).
//
// A cluster of 2 CTAs (one TPC) processes 256 query rows per MMA: each CTA
// holds 128 of the rows (its Q tile, its S / P / O in its own TMEM) and HALF
// of every KV tile -- K split by keys (64 of the 128), V split by head-dim
// columns (64 of 128) -- so each SM's shared memory is read for 6 KB per
// 64-clock QK^T instruction instead of 8 KB, and each K/V byte crosses
// L2 -> SM once per pair.  At the 70B shapes (R*g = 512 rows per KV head) a
// unit is the whole GQA group x tree of one (sequence, KV head).
//
// Roles per CTA (NT = 2: 384 threads): warp 0 TMA producer (both CTAs load
// their own halves; completion bytes land on the leader's barriers), warp 1
// TMEM allocator (both) + single-thread MMA issuer (leader only), warps 4..
// softmax of the CTA's 128 rows of each query tile.  Commits are multicast to
// both CTAs; the softmax -> MMA handshakes (P written, O consumed) arrive on
// the leader's barriers (256 arrivals: 128 local + 128 remote).
#include "sm100_common.cuh"

namespace sdb {
namespace sm100 {

constexpr int kStages2 = 3;

#ifdef SDB_TRACE
// [event][iteration] clock64 stamps of worker 0 (debug builds only)
__device__ unsigned long long g_trace[16][256];
#define TRACE(ev, it)                                                                   \
  do {                                                                                  \
    if (worker == 0 && (it) < 256) g_trace[ev][it] = clock64();                         \
  } while (0)
#else
#define TRACE(ev, it) \
  do {                \
  } while (0)
#endif
constexpr int kHalfBytes = kTileBytes / 2;    // 16 KB: K half [64 keys][128 d] or V half [128 keys][64 d]
constexpr int kKChunk = kHalfBytes / 2;       // 8 KB: one 64-column chunk of the K half

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void *p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, 0;\n"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA into this CTA's smem, completion bytes counted on the leader's barrier
__device__ __forceinline__ void tma2_2d(void *dst, const CUtensorMap *m, uint32_t lbar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lbar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma2_3d(void *dst, const CUtensorMap *m, uint32_t lbar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lbar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma2_4d(void *dst, const CUtensorMap *m, uint32_t lbar, int c0, int c1, int c2,
                                        int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lbar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tc_commit2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// kind::f16, bf16 x bf16 -> fp32, M = 256 (pair), N = 128
__host__ __device__ constexpr uint32_t make_idesc2(bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(kTileN >> 3) << 17) |
         ((uint32_t)(256 >> 4) << 24);
}

template <int NT>
struct alignas(1024) Smem2 {
  uint8_t q[NT][kTileBytes];
  uint8_t k[kStages2][kHalfBytes];
  uint8_t v[kStages2][kHalfBytes];
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages2], k_empty[kStages2], v_full[kStages2], v_empty[kStages2];
  uint64_t s_full[NT], p_full[NT], o_done[NT], o_free[NT];
  uint32_t tmem_base;
  float xch[NT][3][2][128];  // half-row exchange: [0/1] row max by tile parity, [2] row sum
};

template <int NT, int EMU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + NT * 256, 1)
    tree_attn_tcgen05_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tk,
                                  const __grid_constant__ CUtensorMap tm_tv, const Sm100Params sp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem2<NT> &sm = *reinterpret_cast<Smem2<NT> *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TreeAttnParams &p = sp.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.hq / p.hkv;
  const float sl2 = p.scale * 1.4426950408889634f;
  const uint32_t rank = cta_rank();
  const int worker = blockIdx.x >> 1;

  if (threadIdx.x == 0) {
    if (rank == 0) {
      sp.seg[worker] = seg_begin(sp, worker);
      if (worker == 0) sp.seg[sp.n_workers] = sp.total;
    }
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 512);  // 2 CTAs x 256 softmax threads
      mbar_init(&sm.o_done[t], 1);
      mbar_init(&sm.o_free[t], 512);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      tma_prefetch(&tm_tk);
      tma_prefetch(&tm_tv);
      const int bs = p.block_size;
      const int seg_rows = bs < 64 ? bs : 64;
      const uint32_t l_qfull = leader_addr(&sm.q_full);
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, worker);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        mbar_wait(&sm.q_empty, (g_q & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(&sm.q_full, 2 * NT * kTileBytes);
        for (int t = 0; t < NT; ++t) {
          const int node0 = (geo.row0 + t * 2 * kTileM + (int)rank * kTileM) / g;
          for (int c = 0; c < 2; ++c)
            tma2_4d(sm.q[t] + c * kChunkBytes, &tm_q, l_qfull, c * 64, 0, geo.kvh, geo.b * p.r_max + node0);
        }
        ++g_q;
        const int n_valid_pages = (geo.C + bs - 1) / bs;
        const int32_t *bt = p.block_table + (int64_t)geo.b * p.max_blocks;
        for (int it = 0; it < geo.n_tiles; ++it, ++g_tile) {
          const int s = g_tile % kStages2;
          const uint32_t ph = (g_tile / kStages2) & 1;
          const bool pref = it < geo.n_pref;
          const int tile = pref ? geo.pa + it : geo.sa + (it - geo.n_pref);
          // K half: keys [tile*128 + rank*64, +64), all 128 head-dim columns
          mbar_wait(&sm.k_empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&sm.k_full[s], 2 * kHalfBytes);
          const uint32_t l_kfull = leader_addr(&sm.k_full[s]);
          if (pref) {
            for (int r0 = 0; r0 < 64; r0 += seg_rows) {
              const int key = tile * kTileN + (int)rank * 64 + r0;
              const int lp = key / bs;
              const int page = lp < n_valid_pages ? bt[lp] : p.num_blocks;  // OOB page -> zero fill
              const int rowc = (page * p.hkv + geo.kvh) * bs + key % bs;
              for (int c = 0; c < 2; ++c) tma2_2d(sm.k[s] + c * kKChunk + r0 * 128, &tm_k, l_kfull, c * 64, rowc);
            }
          } else {
            for (int c = 0; c < 2; ++c)
              tma2_3d(sm.k[s] + c * kKChunk, &tm_tk, l_kfull, c * 64, geo.kvh,
                      geo.b * p.r_max + tile * kTileN + (int)rank * 64);
          }
          // V half: all 128 keys, head-dim columns [rank*64, +64)
          mbar_wait(&sm.v_empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&sm.v_full[s], 2 * kHalfBytes);
          const uint32_t l_vfull = leader_addr(&sm.v_full[s]);
          if (pref) {
            for (int r0 = 0; r0 < kTileN; r0 += seg_rows) {
              const int key = tile * kTileN + r0;
              const int lp = key / bs;
              const int page = lp < n_valid_pages ? bt[lp] : p.num_blocks;
              const int rowc = (page * p.hkv + geo.kvh) * bs + key % bs;
              tma2_2d(sm.v[s] + r0 * 128, &tm_v, l_vfull, (int)rank * 64, rowc);
            }
          } else {
            tma2_3d(sm.v[s], &tm_tv, l_vfull, (int)rank * 64, geo.kvh, geo.b * p.r_max + tile * kTileN);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc_s = make_idesc2(false);
      constexpr uint32_t idesc_o = make_idesc2(true);
      const uint32_t q_base = smem_u32(sm.q[0]);
      auto issue_s = [&](int t, int s) {
        const uint32_t qa = q_base + t * kTileBytes;
        const uint32_t ka = smem_u32(sm.k[s]);
#pragma unroll
        for (int k = 0; k < kHeadDim / 16; ++k) {
          mma2_ss(tmem + t * 128, sw128_desc(qa + (k >> 2) * kChunkBytes + (k & 3) * 32, 16, 1024),
                  sw128_desc(ka + (k >> 2) * kKChunk + (k & 3) * 32, 16, 1024), idesc_s, k > 0);
        }
      };
      auto issue_pv = [&](int t, int s, bool acc) {
        const uint32_t va = smem_u32(sm.v[s]);
#pragma unroll
        for (int k = 0; k < kTileN / 16; ++k) {
          mma2_ts(tmem + 256 + t * 128, tmem + t * 128 + k * 8, sw128_desc(va + k * 2048, kHalfBytes, 1024), idesc_o,
                  (acc || k > 0) ? 1u : 0u);
        }
      };
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, worker);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        mbar_wait(&sm.q_full, g_q & 1);
        mbar_wait(&sm.k_full[g_tile % kStages2], (g_tile / kStages2) & 1);
        tc_fence_after();
        for (int t = 0; t < NT; ++t) {
          issue_s(t, g_tile % kStages2);
          tc_commit2(&sm.s_full[t]);
        }
        tc_commit2(&sm.k_empty[g_tile % kStages2]);
        for (int it = 0; it < geo.n_tiles; ++it) {
          const uint32_t gt = g_tile + it;
          const int s = gt % kStages2;
          TRACE(12, gt);
          mbar_wait(&sm.v_full[s], (gt / kStages2) & 1);
          TRACE(13, gt);
          tc_fence_after();
          for (int t = 0; t < NT; ++t) {
            TRACE(0 + t * 3, gt);
            mbar_wait_cluster(&sm.p_full[t], gt & 1);
            TRACE(1 + t * 3, gt);
            if (it == 0) mbar_wait_cluster(&sm.o_free[t], (g_q & 1) ^ 1);
            tc_fence_after();
            issue_pv(t, s, it > 0);
            tc_commit2(&sm.o_done[t]);
            if (it + 1 < geo.n_tiles) {
              const int s2 = (gt + 1) % kStages2;
              if (t == 0) {
                mbar_wait(&sm.k_full[s2], ((gt + 1) / kStages2) & 1);
                tc_fence_after();
              }
              issue_s(t, s2);
              tc_commit2(&sm.s_full[t]);
              if (t == NT - 1) tc_commit2(&sm.k_empty[s2]);
            }
            TRACE(2 + t * 3, gt);
          }
          tc_commit2(&sm.v_empty[s]);
        }
        tc_commit2(&sm.q_empty);
        g_tile += geo.n_tiles;
        ++g_q;
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax (both CTAs, own 128 rows per tile) ==========
    // 8 warps per query tile: lane group (warp % 4) x column half (0/1)
    const int t = (warp - 4) >> 3;
    const int ww = (warp - 4) & 7;
    const int lg = ww & 3, half = ww >> 2;
    const int i = (lg << 5) + lane;
    const int bar_id = 1 + t * 4 + lg;
    const uint32_t lane_off = (uint32_t)(lg * 32) << 16;
    const uint32_t t_s = tmem + lane_off + t * 128;
    const uint32_t t_o = tmem + lane_off + 256 + t * 128;
    const int local = t * 2 * kTileM + (int)rank * kTileM + i;  // row within the unit
    uint32_t g_tile = 0;
    ItemIter iter(sp, worker);
    Item item;
    while (iter.next(sp, item)) {
      const ItemGeo geo = item_geo(sp, item, g);
      if (!geo.active) {
        if (half == 0) inactive_row(sp, item, geo, g, local);
        continue;
      }
      const int rho = geo.row0 + local;
      const bool row_ok = rho < geo.rows_total;
      const int node = min(rho / g, max(geo.n_nodes - 1, 0));
      const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
      float m = -INFINITY, l = 0.f;
      for (int it = 0; it < geo.n_tiles; ++it) {
        const uint32_t gt = g_tile + it;
        const bool pref = it < geo.n_pref;
        const int key0 = pref ? (geo.pa + it) * kTileN : (geo.sa + it - geo.n_pref) * kTileN;
        const int kvalid = pref ? geo.C - key0 : geo.n_nodes - key0;
        if (rank == 0 && ww == 0 && lane == 0) TRACE(6 + t * 3, gt);
        mbar_wait(&sm.s_full[t], gt & 1);
        tc_fence_after();
        if (rank == 0 && ww == 0 && lane == 0) TRACE(7 + t * 3, gt);
        softmax_half_tile<EMU>(t_s, t_o, half, sl2, it == 0, pref, kvalid, mrow, key0, p.n_words, row_ok,
                               &sm.xch[t][gt & 1][0][0], i,
                               bar_id, m, l);
        if (rank == 0 && ww == 0 && lane == 0) TRACE(8 + t * 3, gt);
        if (rank == 0)
          mbar_arrive(&sm.p_full[t]);
        else
          mbar_arrive_leader(&sm.p_full[t]);
      }
      mbar_wait(&sm.o_done[t], (g_tile + geo.n_tiles - 1) & 1);
      tc_fence_after();
      // combine the two partial row sums (the max m is identical in both halves)
      sm.xch[t][2][half][i] = l;
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      const float l_full = l + sm.xch[t][2][half ^ 1][i];
      epilogue_half_row(sp, item, geo, g, local, half, t_o, m, l_full);
      tc_fence_before();
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // xch reuse
      if (rank == 0)
        mbar_arrive(&sm.o_free[t]);
      else
        mbar_arrive_leader(&sm.o_free[t]);
      g_tile += geo.n_tiles;
    }
  }
  tc_fence_before();
  __syncwarp();
  cluster_sync();  // the pair's MMAs, remote arrivals and TMEM reads are all done
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int launch_2cta(const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv, const CUtensorMap &mtk,
                const CUtensorMap &mtv, const Sm100Params &sp, int emu, cudaStream_t stream) {
  dim3 grid(sp.n_workers * 2);
#define SDB_LAUNCH_PAIR(NT, EMU)                                                                                 \
  do {                                                                                                           \
    const size_t smem = sizeof(Smem2<NT>) + 1024;                                                                \
    cudaFuncSetAttribute(tree_attn_tcgen05_pair_kernel<NT, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                         (int)smem);                                                                             \
    tree_attn_tcgen05_pair_kernel<NT, EMU><<<grid, 128 + NT * 256, smem, stream>>>(mq, mk, mv, mtk, mtv, sp);   \
  } while (0)
  if (sp.nt == 2) {
    if (emu == 0) SDB_LAUNCH_PAIR(2, 0); else if (emu == 2) SDB_LAUNCH_PAIR(2, 2); else SDB_LAUNCH_PAIR(2, 1);
  } else {
    if (emu == 0) SDB_LAUNCH_PAIR(1, 0); else if (emu == 2) SDB_LAUNCH_PAIR(1, 2); else SDB_LAUNCH_PAIR(1, 1);
  }
#undef SDB_LAUNCH_PAIR
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

}  // namespace sm100
}  // namespace sdb

#ifdef SDB_TRACE
extern "C" int sdb_debug_trace(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, sdb::sm100::g_trace, sizeof(sdb::sm100::g_trace)) == cudaSuccess ? 0 : -4;
}
#endif
