// Tree-verify attention on the 5th-generation tensor cores (sm_100a).
//
// One CTA = one (sequence b, KV head h, block of NT x 128 query rows, KV
// split).  Query rows of a KV head are the GQA group times the tree rows,
// ordered rho = node * g + j (q head h*g + j), so one 128-row tile is 128/g
// tree nodes x g heads -- the dense QK^T / PV contraction of SURVEY.md
// section 0.6 (R*g = 512 rows per KV head at the 70B shapes).
//
// Warp roles (NT = 2: 384 threads):
//   warp 0      TMA producer: Q once, then K/V tiles of 128 keys -- committed
//               prefix pages through the block table (2-D map over the
//               [pages*heads*slots, d] pool) followed by the fresh tree K/V
//               (3-D map over [B*R, Hkv, d]); 2-stage K and V rings.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//               S_t = Q_t K^T (SS, both K-major SW128) and O_t += P_t V
//               (TS: P from TMEM, V MN-major SW128), ping-ponging the two
//               query tiles so one tile's MMAs overlap the other's softmax.
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1: thread i
//               owns TMEM lane i (one query row): S via tcgen05.ld, scale,
//               prefix validity / ancestor-bitmask, online max with lazy
//               O rescale (only when the max grows by > 2^8), exp2, P packed
//               to bf16 and written back over S with tcgen05.st.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512) fp32 columns.
#include <cuda.h>
#include <stdlib.h>

#include <algorithm>

#include "sm100_common.cuh"

namespace sdb {
namespace sm100 {

// K / V ring depth: 3 stages with one query tile (224 KB of shared memory),
// 2 with two
#ifndef SDB_KV1_STAGES
#define SDB_KV1_STAGES 3
#endif
template <int NT>
constexpr int kvStages() {
  return NT == 1 ? SDB_KV1_STAGES : 2;
}
template <int NT>
struct alignas(1024) Smem {
  uint8_t q[NT][kTileBytes];
  uint8_t k[kvStages<NT>()][kTileBytes];
  uint8_t v[kvStages<NT>()][kTileBytes];
  uint64_t q_full, q_empty;
  uint64_t k_full[kvStages<NT>()], k_empty[kvStages<NT>()], v_full[kvStages<NT>()], v_empty[kvStages<NT>()];
  uint64_t s_full[2], p_full[2], o_done[NT], o_free[NT];  // NT = 1: two S slots of the one tile
  uint32_t tmem_base;
};

// 1-CTA kernel (M = 128 MMAs): used when a KV head has <= 128 query rows
// (small trees / small GQA groups), and as the reference implementation of
// the 2-CTA pair kernel (attn_sm100_2cta.cu).
template <int NT, int EMU>
__global__ void __launch_bounds__(128 + NT * 128, 1)
    tree_attn_tcgen05_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tk,
                             const __grid_constant__ CUtensorMap tm_tv, const __grid_constant__ Sm100Params sp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NT> &sm = *reinterpret_cast<Smem<NT> *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TreeAttnParams &p = sp.p;
  griddep_launch_dependents();  // the fix-up grid may become resident (it waits for our completion)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.hq / p.hkv;
  const float sl2 = p.scale * 1.4426950408889634f;

  if (threadIdx.x == 0) {
    sp.seg[blockIdx.x] = seg_begin(sp, blockIdx.x);
    if (blockIdx.x == 0) sp.seg[sp.n_workers] = sp.total;
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int s = 0; s < kvStages<NT>(); ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 128);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(&sm.o_done[t], 1);
      mbar_init(&sm.o_free[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ===================== TMA producer =====================
    // Whole warp walks the schedule; block-table entries of the next 32 pages
    // come from one coalesced load by the 32 lanes (shuffled to the issuing
    // lane), so no TMA issue waits for a dependent global load.
    {
      if (lane == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_tk);
        tma_prefetch(&tm_tv);
      }
      const int bs = p.block_size;
      const int seg_rows = bs < 64 ? bs : 64;  // pool TMA box rows
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, blockIdx.x);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        // the plan covers w_pref prefix tiles: a longer context (ctx_len >
        // max_ctx) would lose keys -- flag it instead (CacheError)
        if (lane == 0 && p.err && geo.C - geo.k0 > sp.w_pref * kTileN) atomicOr(p.err, SDB_ERR_CACHE);
        // Q tiles of this unit once the previous unit's S MMAs are done
        mbar_wait(&sm.q_empty, (g_q & 1) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&sm.q_full, NT * kTileBytes);
          for (int t = 0; t < NT; ++t) {
            const int node0 = geo.q0 + (geo.row0 + t * kTileM) / g;
            for (int c = 0; c < 2; ++c)
              tma_load_4d(sm.q[t] + c * kChunkBytes, &tm_q, &sm.q_full, c * 64, 0, geo.kvh,
                          geo.b * p.r_max + node0);
          }
        }
        ++g_q;
        const int n_valid_pages = (geo.C + bs - 1) / bs;
        const int32_t *bt = p.block_table + (int64_t)geo.b * p.max_blocks;
        int pc_base = -64, pc_val = 0;  // lane l holds the page of logical block pc_base + l
        auto page_of = [&](int lp) {
          if (lp < pc_base || lp >= pc_base + 32) {  // warp-uniform
            pc_base = lp & ~31;
            const int e = pc_base + lane;
            pc_val = e < n_valid_pages ? __ldg(bt + e) : p.num_blocks;  // OOB page -> zero fill
          }
          return __shfl_sync(0xffffffffu, pc_val, lp - pc_base);
        };
        for (int it = 0; it < geo.n_tiles; ++it, ++g_tile) {
          constexpr int kS = kvStages<NT>();
          const int s = g_tile % kS;
          const uint32_t ph = (g_tile / kS) & 1;
          const bool pref = it < geo.n_pref;
          const int tile = pref ? geo.pa + it : geo.sa + (it - geo.n_pref);
          for (int kv = 0; kv < 2; ++kv) {
            uint64_t *emp = kv ? &sm.v_empty[s] : &sm.k_empty[s];
            uint64_t *ful = kv ? &sm.v_full[s] : &sm.k_full[s];
            uint8_t *dst = kv ? sm.v[s] : sm.k[s];
            mbar_wait(emp, ph ^ 1);
            if (lane == 0) mbar_expect_tx(ful, kTileBytes);
            if (pref) {
              const CUtensorMap *m = kv ? &tm_v : &tm_k;
              for (int r0 = 0; r0 < kTileN; r0 += seg_rows) {
                const int key = geo.k0 + tile * kTileN + r0;
                const int page = page_of(key / bs);
                const int rowc = (page * p.hkv + geo.kvh) * bs + key % bs;
                if (lane == 0)
                  for (int c = 0; c < 2; ++c) tma_load_2d(dst + c * kChunkBytes + r0 * 128, m, ful, c * 64, rowc);
              }
            } else if (lane == 0) {
              const CUtensorMap *m = kv ? &tm_tv : &tm_tk;
              for (int c = 0; c < 2; ++c)
                tma_load_3d(dst + c * kChunkBytes, m, ful, c * 64, geo.kvh, geo.b * p.r_max + tile * kTileN);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // Whole warp walks the schedule (uniform descriptors); one elected lane
    // issues (see attn_sm100_2cta.cu: a lone issuing thread costs ~16
    // instructions per tcgen05.mma).
    {
      constexpr uint32_t idesc_s = make_idesc(false);
      constexpr uint32_t idesc_o = make_idesc(true);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint64_t q_desc = sw128_desc(smem_u32(sm.q[0]), 16, 1024);
      const uint64_t k_desc = sw128_desc(smem_u32(sm.k[0]), 16, 1024);
      const uint64_t v_desc = sw128_desc(smem_u32(sm.v[0]), kChunkBytes, 1024);
      auto issue_s = [&](int t, int st) {
        const uint64_t qd = q_desc + (uint64_t)((t * kTileBytes) >> 4);
        const uint64_t kd = k_desc + (uint64_t)((st * kTileBytes) >> 4);
#pragma unroll
        for (int k = 0; k < kHeadDim / 16; ++k) {
          const uint64_t off = (uint64_t)(((k >> 2) * kChunkBytes + (k & 3) * 32) >> 4);
          mma_ss(tm + t * 128, qd + off, kd + off, idesc_s, k > 0);
        }
      };
      auto issue_pv = [&](int t, int st, bool acc) {
        const uint64_t vd = v_desc + (uint64_t)((st * kTileBytes) >> 4);
#pragma unroll
        for (int k = 0; k < kTileN / 16; ++k)
          mma_ts(tm + 256 + t * 128, tm + t * 128 + k * 8, vd + (uint64_t)((k * 2048) >> 4), idesc_o,
                 (acc || k > 0) ? 1u : 0u);
      };
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, blockIdx.x);
      Item item;
      if (NT == 1) {
        // one query tile, two S slots (TMEM columns [0,128) and [128,256), O
        // at [256,384)): S(n + 1) runs while the softmax works on item n, and
        // S(n + 2) refills slot n % 2 right after PV(n) -- at small trees the
        // item no longer serialises S -> softmax -> PV
        constexpr int kS = kvStages<NT>();  // K / V stage gt % kS; S slot gt % 2
        auto issue_s1 = [&](uint32_t gt) {
          mbar_wait(&sm.k_full[gt % kS], (gt / kS) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t kd = k_desc + (uint64_t)(((gt % kS) * kTileBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kHeadDim / 16; ++k) {
              const uint64_t off = (uint64_t)(((k >> 2) * kChunkBytes + (k & 3) * 32) >> 4);
              mma_ss(tm + (gt & 1) * 128, q_desc + off, kd + off, idesc_s, k > 0);
            }
            tc_commit(&sm.s_full[gt & 1]);
            tc_commit(&sm.k_empty[gt % kS]);
          }
          __syncwarp();
        };
        while (iter.next(sp, item)) {
          const ItemGeo geo = item_geo(sp, item, g);
          if (!geo.active) continue;
          const int n_tiles = __shfl_sync(0xffffffffu, geo.n_tiles, 0);
          mbar_wait(&sm.q_full, g_q & 1);
          issue_s1(g_tile);
          if (n_tiles > 1) issue_s1(g_tile + 1);
          for (int it = 0; it < n_tiles; ++it) {
            const uint32_t gt = g_tile + it;
            const int sl = gt & 1, st = gt % kS;
            mbar_wait(&sm.v_full[st], (gt / kS) & 1);
            mbar_wait(&sm.p_full[sl], (gt >> 1) & 1);
            if (it == 0) mbar_wait(&sm.o_free[0], (g_q & 1) ^ 1);  // previous unit's epilogue read O
            tc_fence_after();
            if (elect_one()) {
              const uint64_t vd = v_desc + (uint64_t)((st * kTileBytes) >> 4);
#pragma unroll
              for (int k = 0; k < kTileN / 16; ++k)
                // P of keys 16k .. 16k+15 at slot columns 32 (k/2) + 8 (k%2)
                // (chunk c packed into the first half of its own 32 S columns)
                mma_ts(tm + 256, tm + sl * 128 + 32 * (k >> 1) + 8 * (k & 1), vd + (uint64_t)((k * 2048) >> 4),
                       idesc_o, (it > 0 || k > 0) ? 1u : 0u);
              if (it == n_tiles - 1) tc_commit(&sm.o_done[0]);  // the epilogue may read O
              tc_commit(&sm.v_empty[st]);
            }
            __syncwarp();
            if (it + 2 < n_tiles) issue_s1(gt + 2);
          }
          if (elect_one()) tc_commit(&sm.q_empty);  // all S MMAs of this unit read Q
          __syncwarp();
          g_tile += n_tiles;
          ++g_q;
        }
      }
      while (NT == 2 && iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        const int n_tiles = __shfl_sync(0xffffffffu, geo.n_tiles, 0);
        mbar_wait(&sm.q_full, g_q & 1);
        mbar_wait(&sm.k_full[g_tile & 1], (g_tile >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          for (int t = 0; t < NT; ++t) {
            issue_s(t, g_tile & 1);
            tc_commit(&sm.s_full[t]);
          }
          tc_commit(&sm.k_empty[g_tile & 1]);
        }
        __syncwarp();
        for (int it = 0; it < n_tiles; ++it) {
          const uint32_t gt = g_tile + it;
          const int st = gt & 1;
          mbar_wait(&sm.v_full[st], (gt >> 1) & 1);
          tc_fence_after();
          for (int t = 0; t < NT; ++t) {
            mbar_wait(&sm.p_full[t], gt & 1);
            if (it == 0) mbar_wait(&sm.o_free[t], (g_q & 1) ^ 1);  // previous unit's epilogue read O_t
            tc_fence_after();
            if (elect_one()) {
              issue_pv(t, st, it > 0);
              // O is read only by the unit's epilogue (a rescale relies on the
              // in-order pipe: S(n + 1), committed after PV(n), gates it)
              if (it == n_tiles - 1) tc_commit(&sm.o_done[t]);
            }
            __syncwarp();
            if (it + 1 < n_tiles) {
              const int s2 = (gt + 1) & 1;
              if (t == 0) {
                mbar_wait(&sm.k_full[s2], ((gt + 1) >> 1) & 1);
                tc_fence_after();
              }
              if (elect_one()) {
                issue_s(t, s2);
                tc_commit(&sm.s_full[t]);
                if (t == NT - 1) tc_commit(&sm.k_empty[s2]);
              }
              __syncwarp();
            }
          }
          if (elect_one()) tc_commit(&sm.v_empty[st]);
          __syncwarp();
        }
        if (elect_one()) tc_commit(&sm.q_empty);  // all S MMAs of this unit read Q
        __syncwarp();
        g_tile += n_tiles;
        ++g_q;
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax warpgroups =====================
    // programmatic dependent launch: the mask words come from the kernel
    // launched just before (tree_build); everything else in flight above
    // (TMEM alloc, TMA of Q/K/V, first QK^T) already overlaps its tail
    griddep_wait();
    const int t = (warp - 4) >> 2;          // query tile
    const int i = ((warp & 3) << 5) + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + t * 128;
    const uint32_t t_o = tmem + lane_off + 256 + t * 128;
    const int local = t * kTileM + i;  // row within the unit
    uint32_t g_tile = 0, g_unit = 0;
    ItemIter iter(sp, blockIdx.x);
    Item item;
    if (NT == 1) {
      // items alternate between the two S slots.  Fixed reference (as in the
      // pair kernel): the row max of the first 32 keys of the piece's first
      // tile; P = exp2(s * scale * log2e - m_ref), nothing is ever rescaled
      // (O is accumulated by PV MMAs this warp does not wait for); a row
      // whose scores climb ~89 log2 units above it is recomputed exactly by
      // its own thread after the epilogue
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) {
          inactive_row(sp, item, geo, g, local);
          continue;
        }
        const int rho = geo.row0 + local;
        const bool row_ok = rho < geo.rows_total;
        const int node = min(geo.q0 + rho / g, max(geo.n_nodes - 1, 0));
        const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
        // a warp whose 32 rows are all padding only keeps the barrier phases
        const bool pad_warp = geo.row0 + (warp & 3) * 32 >= geo.rows_total;
        float m_ref = -INFINITY, l = 0.f;
        bool bad = false;
        for (int it = 0; it < geo.n_tiles; ++it) {
          const uint32_t gt = g_tile + it;
          const int sl = gt & 1;
          const bool pref = it < geo.n_pref;
          const int key0 = pref ? geo.k0 + (geo.pa + it) * kTileN : (geo.sa + it - geo.n_pref) * kTileN;
          const int kvalid = pref ? geo.C - key0 : geo.n_nodes - key0;
          const bool full = pref && kvalid >= kTileN;
          mbar_wait(&sm.s_full[sl], (gt >> 1) & 1);
          tc_fence_after();
          const uint32_t ts = tmem + lane_off + sl * 128;
          if (!pad_warp) {
            uint32_t vm[4] = {~0u, ~0u, ~0u, ~0u};
            if (!full) {
#pragma unroll
              for (int c = 0; c < 4; ++c) vm[c] = vis_word(pref, kvalid, mrow, key0, p.n_words, row_ok, 32 * c);
            }
            uint32_t r[32], r2[32];
            if (it == 0) {
              SDB_TMEM_LD32(ts, r2);
              SDB_TMEM_WAIT_LD_REGS(r2);
              if (!full) apply_mask32(r2, vm[0]);
              m_ref = max32(r2) * sl2;
            }
            const float neg_mu = (m_ref == -INFINITY) ? 0.f : -m_ref;
            const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_mu, neg_mu);
            SDB_TMEM_LD32(ts + 0, r2);
            SDB_TMEM_WAIT_LD_REGS(r2);
            SDB_TMEM_LD32(ts + 32, r);
            if (!full) apply_mask32(r2, vm[0]);
            float rs = exp_pack32<0>(r2, sc2, nm2);
            SDB_TMEM_ST16(ts + 0, r2);
            SDB_TMEM_WAIT_LD_REGS(r);
            SDB_TMEM_LD32(ts + 64, r2);
            if (!full) apply_mask32(r, vm[1]);
            rs += exp_pack32<0>(r, sc2, nm2);
            SDB_TMEM_ST16(ts + 32, r);
            SDB_TMEM_WAIT_LD_REGS(r2);
            SDB_TMEM_LD32(ts + 96, r);
            if (!full) apply_mask32(r2, vm[2]);
            rs += exp_pack32<0>(r2, sc2, nm2);
            SDB_TMEM_ST16(ts + 64, r2);
            SDB_TMEM_WAIT_LD_REGS(r);
            if (!full) apply_mask32(r, vm[3]);
            rs += exp_pack32<0>(r, sc2, nm2);
            SDB_TMEM_ST16(ts + 96, r);
            l += rs;
            bad |= rs > kOverflowSum || (m_ref == -INFINITY && rs > 0.f);
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&sm.p_full[sl]);
        }
        mbar_wait(&sm.o_done[0], g_unit & 1);  // the unit's last PV
        ++g_unit;
        tc_fence_after();
        epilogue_row(sp, item, geo, g, local, t_o, m_ref, l);
        tc_fence_before();
        mbar_arrive(&sm.o_free[0]);  // O may now be overwritten by the next unit's first PV
        if (bad) exact_row(sp, item, geo, g, local);  // overwrite this row's stores exactly
        g_tile += geo.n_tiles;
      }
    }
    while (NT == 2 && iter.next(sp, item)) {
      const ItemGeo geo = item_geo(sp, item, g);
      if (!geo.active) {
        inactive_row(sp, item, geo, g, local);
        continue;
      }
      const int rho = geo.row0 + local;
      const bool row_ok = rho < geo.rows_total;
      const int node = min(geo.q0 + rho / g, max(geo.n_nodes - 1, 0));
      const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
      float m = -INFINITY, l = 0.f;
      for (int it = 0; it < geo.n_tiles; ++it) {
        const uint32_t gt = g_tile + it;
        const bool pref = it < geo.n_pref;
        const int key0 = pref ? geo.k0 + (geo.pa + it) * kTileN : (geo.sa + it - geo.n_pref) * kTileN;
        const int kvalid = pref ? geo.C - key0 : geo.n_nodes - key0;
        mbar_wait(&sm.s_full[t], gt & 1);
        tc_fence_after();
        softmax_tile<EMU>(t_s, t_o, sl2, it == 0, pref, kvalid, mrow, key0, p.n_words, row_ok, m, l);
        mbar_arrive(&sm.p_full[t]);
      }
      mbar_wait(&sm.o_done[t], g_unit & 1);  // the unit's last PV
      ++g_unit;
      tc_fence_after();
      epilogue_row(sp, item, geo, g, local, t_o, m, l);
      tc_fence_before();
      mbar_arrive(&sm.o_free[t]);  // O_t may now be overwritten by the next unit's first PV
      g_tile += geo.n_tiles;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Stream-K fix-up: one block row per worker boundary k (1..n_workers-1).  A
// boundary strictly inside unit u splits it; the FIRST boundary inside u
// merges all of u's pieces (same math as merge_partials,
// attention.py:108-124).  grid (n_workers - 1, rows_unit / 4), one warp per row.
__global__ void __launch_bounds__(128) tree_attn_fixup_kernel(const Sm100Params sp) {
  // launched as a programmatic dependent of the attention kernel: resident
  // early, released when every attention CTA has finished and flushed
  griddep_wait();
  const TreeAttnParams &p = sp.p;
  // blockIdx.x: a split unit from the host's list (its first interior
  // boundary k), or every boundary when the list overflowed
  const int k = sp.n_split >= 0 ? sp.split_k[blockIdx.x] : blockIdx.x + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int local = blockIdx.y * 4 + warp;
  if (local >= sp.rows_unit) return;
  const int64_t ck = seg_begin(sp, k);  // (arithmetic: the same values the main kernel wrote to sp.seg)
  const int W = sp.w_unit;
  const int unit = (int)(ck / W);
  // rows past the row block: the fused tail rows of a last-block unit only
  if (local >= sp.row_blk &&
      (unit / (p.batch * p.hkv) != sp.m_blocks - 1 || local >= sp.row_blk + sp.tail_rows))
    return;
  const int64_t ustart = (int64_t)unit * W, uend = ustart + W;
  if (ck == ustart) return;                  // boundary between units: nothing split here
  if (seg_begin(sp, k - 1) > ustart) return;  // an earlier boundary inside u merges it
  const int g = p.hq / p.hkv;
  const int bh = p.batch * p.hkv;
  const int b = (unit % bh) / p.hkv, kvh = unit % p.hkv;
  const int rho = (unit / bh) * sp.row_blk + local;
  const int n_nodes = min(p.n_rows[b], p.r_max);
  const int q0 = q_first(p, b, n_nodes);
  if (q0 * g + rho >= p.r_max * g) return;
  const int node = q0 + rho / g, hq_idx = kvh * g + rho % g;
  __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(p.out) + (((int64_t)b * p.r_max + node) * p.hq + hq_idx) * kHeadDim;
  float *lse_out = p.lse ? p.lse + ((int64_t)b * p.hq + hq_idx) * p.r_max + node : nullptr;
  if (rho >= (n_nodes - q0) * g) {
    *reinterpret_cast<uint2 *>(out + lane * 4) = make_uint2(0, 0);
    if (lse_out && lane == 0) *lse_out = -INFINITY;
    return;
  }
  // pieces: worker k-1 (its first item iff its segment starts at the unit
  // start, else its last item), then the first item of every later worker
  // whose segment starts inside u.  Everything is fetched warp-parallel:
  // the segment scan by ballot (seg is monotone), the piece LSEs one per
  // lane, the partial rows four loads in flight -- a serial walk costs one
  // dependent L2 round trip per piece (C2: 7 pieces per unit).
  const int first_slot = (k - 1) * 2 + (seg_begin(sp, k - 1) == ustart ? 0 : 1);
  int kk_end = k;
  for (int base = k;; base += 32) {
    const int kk = base + lane;
    const bool inside = kk < sp.n_workers && seg_begin(sp, kk) < uend;
    const unsigned out = ~__ballot_sync(0xffffffffu, inside);
    const int lead = out ? __ffs(out) - 1 : 32;
    kk_end = base + lead;
    if (lead < 32) break;
  }
  const int np = 1 + kk_end - k;  // piece j: slot first_slot (j = 0) or (k - 1 + j) * 2
  auto slot_of = [&](int j) { return j == 0 ? first_slot : (k - 1 + j) * 2; };
  float mx = -INFINITY;
  for (int c0 = 0; c0 < np; c0 += 32) {
    const int j = c0 + lane;
    float l = j < np ? sp.part_lse[(int64_t)slot_of(j) * sp.rows_unit + local] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l = fmaxf(l, __shfl_xor_sync(0xffffffffu, l, o));
    mx = fmaxf(mx, l);
  }
  float wsum = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c0 = 0; c0 < np; c0 += 32) {
    const int j = c0 + lane;
    const float l = j < np ? sp.part_lse[(int64_t)slot_of(j) * sp.rows_unit + local] : -INFINITY;
    const float wl = l == -INFINITY ? 0.f : __expf(l - mx);
    const int m = min(32, np - c0);
    for (int t = 0; t < m; t += 4) {
      float wt[4];
      float4 o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wt[u] = __shfl_sync(0xffffffffu, wl, (t + u) & 31);
        o[u] = (t + u < m && wt[u] != 0.f)
                   ? *reinterpret_cast<const float4 *>(
                         sp.part_out + ((int64_t)slot_of(c0 + t + u) * sp.rows_unit + local) * kHeadDim + lane * 4)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (t + u >= m || wt[u] == 0.f) continue;
        wsum += wt[u];
        acc[0] = fmaf(wt[u], o[u].x, acc[0]);
        acc[1] = fmaf(wt[u], o[u].y, acc[1]);
        acc[2] = fmaf(wt[u], o[u].z, acc[2]);
        acc[3] = fmaf(wt[u], o[u].w, acc[3]);
      }
    }
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  uint2 v;
  v.x = pack_bf16(acc[0] * inv, acc[1] * inv);
  v.y = pack_bf16(acc[2] * inv, acc[3] * inv);
  *reinterpret_cast<uint2 *>(out + lane * 4) = v;
  if (lse_out && lane == 0) *lse_out = wsum > 0.f ? mx + logf(wsum) : -INFINITY;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static bool make_map(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides,
                     const cuuint32_t *box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sm100

bool tree_attn_sm100_supported(const TreeAttnParams &p) {
  if (p.head_dim != sm100::kHeadDim) return false;
  const int g = p.hq / p.hkv;
  if (g < 1 || g > 128 || (128 % g) != 0) return false;
  if (p.block_size < 8 || p.block_size > 128 || (128 % p.block_size) != 0) return false;
  if ((reinterpret_cast<uintptr_t>(p.q) | reinterpret_cast<uintptr_t>(p.k_cache) |
       reinterpret_cast<uintptr_t>(p.v_cache) | reinterpret_cast<uintptr_t>(p.tree_k) |
       reinterpret_cast<uintptr_t>(p.tree_v)) & 15)
    return false;
  if (p.r_max > 128) return false;  // one suffix tile (<= 4 mask words)
  // local chunks must start on a key tile and a page boundary
  if (p.chunk_len > 0 && (p.chunk_len % sm100::kTileN != 0 || p.chunk_len % p.block_size != 0)) return false;
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 && sm100::encode_fn() != nullptr;
}

// Work plan: CTA pairs (cta_group::2, M = 256 MMAs) whenever a KV head has
// more than 128 query rows, else single CTAs (M = 128); units x nominal tiles
// split evenly over the persistent workers (stream-K).
static void sm100_plan(const TreeAttnParams &p, int ctas_override, sm100::Sm100Params &sp) {
  using namespace sm100;
  const int g = p.hq / p.hkv;
  const int rows = p.max_q_nodes * g;  // query rows per (sequence, KV head)
  const char *fg = getenv("SDB_ATTN_CTA_GROUP");  // testing knob: force 1-CTA or pair kernels
  const int force_group = fg ? atoi(fg) : 0;
  sp.p = p;
  sp.cta_group = (force_group == 1 || force_group == 2) ? force_group : (rows > kTileM ? 2 : 1);
  const int per_tile = kTileM * sp.cta_group;
  // pair kernel: one 256-row query tile per unit (three S slots fill TMEM)
  sp.nt = (sp.cta_group == 1 && rows > per_tile) ? 2 : 1;
  if (const char *fnt = getenv("SDB_ATTN_NT")) sp.nt = atoi(fnt) == 1 ? 1 : sp.nt;  // testing knob
  sp.rows_unit = sp.nt * per_tile;
  sp.row_blk = sp.rows_unit;
  sp.m_blocks = cdiv(rows, sp.rows_unit);
  sp.tail_rows = 0;
  // pair kernel, 1..8 rows past the last full 256-row block (R = 65: 520 rows
  // per KV head): SDB_ATTN_TAIL=1 fuses those rows into the last block's
  // units on the otherwise idle warps 2 / 3 (S^T = K Q_tail^T and O^T =
  // V^T P_tail^T, N = 16) instead of a third, 97 %-padding row block.  Exact
  // (tests/test_gpu_parity.py) but measured slower at C3 R = 65 (attention
  // 1076 vs 679 us): with every TMEM column taken by O and the three S slots,
  // a tail item's S^T / O^T must be read before the slot's next S, so each
  // item waits on four cross-CTA handshakes (~500-900 cycles each) --
  // profiles/r2_attn_power_study.md section 6.  Off by default; needs warp
  // 3 (not the fused greedy scan) and warp 2 (the V loads move to warp 0).
  const char *tail_env = getenv("SDB_ATTN_TAIL");
  const bool tail_knob = tail_env && atoi(tail_env) != 0;
  if (tail_knob && sp.cta_group == 2 && sp.nt == 1 && rows > per_tile && rows % per_tile <= 8 && !p.fa_logits &&
      g <= 8) {
    sp.tail_rows = rows % per_tile;
    if (sp.tail_rows > 0) {
      sp.m_blocks = rows / per_tile;
      sp.rows_unit = per_tile + 8;
    }
  }
  sp.units = p.batch * p.hkv * sp.m_blocks;
  // nominal prefix tiles per unit: the context, or at most one local chunk
  sp.w_pref = cdiv(max(p.chunk_len > 0 ? std::min(p.max_ctx, p.chunk_len) : p.max_ctx, 0), kTileN);
  sp.w_unit = sp.w_pref + cdiv(p.r_max, kTileN);
  sp.total = (int64_t)sp.units * sp.w_unit;
  int n = ctas_override > 0 ? ctas_override : num_sms() / sp.cta_group;
  // >= ~9 tiles per worker (small batches then leave SMs to the acceptance
  // branch running concurrently, verify.TreeVerifier.step) but never fewer
  // workers than units: a unit costs ~6 us of prologue / pipeline fill /
  // epilogue, so units must not serialise
  static int tpw = -1;
  if (tpw < 0) {
    const char *e = getenv("SDB_ATTN_TPW");  // testing knob: target tiles per worker
    tpw = e ? std::max(1, atoi(e)) : 9;
  }
  n = (int)std::max<int64_t>(
      1, std::min<int64_t>(n, ctas_override > 0 ? sp.total : std::max<int64_t>(sp.units, sp.total / tpw)));
  // worker count by a cost model in tiles per worker: whole units per
  // worker (no split, no fix-up), equal pieces of every unit (+ a merge), or
  // pieces straddling unit boundaries (+ a second prologue / epilogue), each
  // overhead ~11 tiles (calibrated on C3 per-GPU shards: G 8, 64 units: 64
  // pairs 71.6 us vs 74: 86.6; G 4, 128 units: 137.4 vs 146.6; G 1, 512
  // units: 533 vs 516; C2, 8 units: 56 workers 33.0 us vs 52: 39.8); the
  // search stays within 3/4 of the SM-limited count (CTA-pair kernel)
  static int cost_plan = -1;
  if (cost_plan < 0) {
    const char *e = getenv("SDB_ATTN_COST_PLAN");  // testing knob: 0 disables
    cost_plan = e ? atoi(e) != 0 : 1;
  }
  if (ctas_override <= 0 && n > 1 && cost_plan && sp.cta_group == 2) {
    constexpr int64_t kSplit = 11;
    auto cost = [&](int m) -> int64_t {
      if (sp.units % m == 0) return (int64_t)(sp.units / m) * sp.w_unit;
      if (m % sp.units == 0) return sp.total / m + kSplit;
      return (sp.total + m - 1) / m + 2 * kSplit;
    };
    int best = n;
    for (int m = n - 1; m * 4 >= n * 3; --m)
      if (cost(m) < cost(best)) best = m;
    n = best;
  } else if (ctas_override <= 0 && n > sp.units && (n % sp.units) * 8 <= n) {
    // single-CTA kernel: equal pieces per unit when that costs <= 1/8 of the
    // workers (its split overhead is small: whole-unit plans measured slower
    // on the draft depth steps, 276 vs 215 us)
    n -= n % sp.units;
  }
  // a multiple of the row blocks per KV head keeps those blocks in step on
  // workers n / m_blocks apart (L2 serves the second read of each K/V tile);
  // a misaligned count reads K/V twice (C3, 63 pairs: +7 %)
  if (sp.m_blocks > 1 && n > sp.m_blocks) n -= n % sp.m_blocks;
  sp.n_workers = n;
  sp.part_out = nullptr;
  sp.part_lse = nullptr;
  sp.seg = nullptr;
}

int64_t tree_attn_sm100_workspace(const TreeAttnParams &p, int ctas_override) {
  sm100::Sm100Params sp;
  sm100_plan(p, ctas_override, sp);
  return (int64_t)sp.n_workers * 2 * sp.rows_unit * (sm100::kHeadDim + 1) * (int64_t)sizeof(float) +
         (int64_t)(sp.n_workers + 1) * 8 + 256;
}

int tree_attn_sm100_group(const TreeAttnParams &p, int ctas_override) {
  sm100::Sm100Params sp;
  sm100_plan(p, ctas_override, sp);
  return sp.cta_group;
}

int tree_attn_sm100_sms(const TreeAttnParams &p, int ctas_override) {
  sm100::Sm100Params sp;
  sm100_plan(p, ctas_override, sp);
  return sp.n_workers * sp.cta_group;
}

int launch_tree_attn_sm100(const TreeAttnParams &p, int ctas_override, void *workspace, cudaStream_t stream) {
  using namespace sm100;
  const int g = p.hq / p.hkv;
  const int d = kHeadDim;
  Sm100Params sp;
  sm100_plan(p, ctas_override, sp);
  const int cg = sp.cta_group;
  CUtensorMap mq, mqt, mk, mv, mtk, mtv;
  {
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)g, (cuuint64_t)p.hkv, (cuuint64_t)p.batch * p.r_max};
    cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)g * d * 2, (cuuint64_t)p.hq * d * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)g, 1, (cuuint32_t)(kTileM / g)};
    if (!make_map(&mq, p.q, 4, dims, strides, box)) return SDB_E_UNSUPPORTED;
    // fused tail rows: 8 rows (8 / g nodes x g heads) per d-chunk
    cuuint32_t boxt[4] = {64, (cuuint32_t)g, 1, (cuuint32_t)(g <= 8 ? 8 / g : 1)};
    if (!make_map(&mqt, p.q, 4, dims, strides, boxt)) return SDB_E_UNSUPPORTED;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)p.num_blocks * p.hkv * p.block_size};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(p.block_size < 64 ? p.block_size : 64)};
    if (!make_map(&mk, p.k_cache, 2, dims, strides, box)) return SDB_E_UNSUPPORTED;
    if (!make_map(&mv, p.v_cache, 2, dims, strides, box)) return SDB_E_UNSUPPORTED;
  }
  {
    // tree K: 64-row boxes for a pair (each CTA holds half the keys of a tile),
    // 128 otherwise; tree V: always 128 rows (a pair splits V by columns)
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)p.hkv, (cuuint64_t)p.batch * p.r_max};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)p.hkv * d * 2};
    cuuint32_t boxk[3] = {64, 1, (cuuint32_t)(kTileN / cg)};
    cuuint32_t boxv[3] = {64, 1, (cuuint32_t)kTileN};
    if (!make_map(&mtk, p.tree_k, 3, dims, strides, boxk)) return SDB_E_UNSUPPORTED;
    if (!make_map(&mtv, p.tree_v, 3, dims, strides, boxv)) return SDB_E_UNSUPPORTED;
  }
  sp.part_out = reinterpret_cast<float *>(workspace);
  sp.part_lse = sp.part_out + (int64_t)sp.n_workers * 2 * sp.rows_unit * kHeadDim;
  sp.seg = reinterpret_cast<int64_t *>(sp.part_lse + (int64_t)sp.n_workers * 2 * sp.rows_unit);
  static int emu = -1;
  if (emu < 0) {
    const char *e = getenv("SDB_ATTN_EMU");
    emu = e ? atoi(e) : 1;
    emu = emu < 0 ? 0 : (emu > 2 ? 2 : emu);
  }
  if (cg == 2) {
    static int emu8 = -1;  // pair kernel: exp2 pairs of every 8 emulated on the FMA pipe
    if (emu8 < 0) {
      const char *e = getenv("SDB_ATTN_EMU8");
      // fixed-reference softmax: every exp2 on the MUFU measured fastest
      // (C3: 529 us vs 553-563 with 1 of 8 pairs emulated, 569 / 580 at 2 / 3)
      emu8 = e ? atoi(e) : 0;
      emu8 = emu8 < 0 ? 0 : (emu8 > 4 ? 4 : emu8);
    }
    int rc = launch_2cta(mq, mqt, mk, mv, mtk, mtv, sp, emu8, stream);
    if (rc != SDB_OK) return rc;
  } else {
    dim3 grid(sp.n_workers);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
#define SDB_LAUNCH_TC(NT, EMU)                                                                               \
  do {                                                                                                       \
    const size_t smem = sizeof(Smem<NT>) + 1024;                                                             \
    cudaFuncSetAttribute(tree_attn_tcgen05_kernel<NT, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cudaLaunchConfig_t cfg = {};                                                                             \
    cfg.gridDim = grid;                                                                                      \
    cfg.blockDim = dim3(128 + NT * 128);                                                                     \
    cfg.dynamicSmemBytes = smem;                                                                             \
    cfg.stream = stream;                                                                                     \
    cfg.attrs = &attr;                                                                                       \
    cfg.numAttrs = sp.p.pdl ? 1 : 0;                                                                         \
    cudaLaunchKernelEx(&cfg, tree_attn_tcgen05_kernel<NT, EMU>, mq, mk, mv, mtk, mtv, sp);                   \
  } while (0)
    if (sp.nt == 2) {
      if (emu == 0) SDB_LAUNCH_TC(2, 0); else if (emu == 2) SDB_LAUNCH_TC(2, 2); else SDB_LAUNCH_TC(2, 1);
    } else {
      if (emu == 0) SDB_LAUNCH_TC(1, 0); else if (emu == 2) SDB_LAUNCH_TC(1, 2); else SDB_LAUNCH_TC(1, 1);
    }
#undef SDB_LAUNCH_TC
    SDB_CHECK_LAUNCH();
  }
  // split units (a worker boundary strictly inside): one fix-up block row
  // each; no launch at all when every unit is whole
  sp.n_split = 0;
  for (int k = 1; k < sp.n_workers && sp.n_split >= 0; ++k) {
    const int64_t ck = seg_begin(sp, k), ustart = ck / sp.w_unit * sp.w_unit;
    if (ck == ustart || seg_begin(sp, k - 1) > ustart) continue;
    if (sp.n_split == kMaxSplit) sp.n_split = -1;
    else sp.split_k[sp.n_split++] = k;
  }
  if (sp.n_workers > 1 && sp.n_split != 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sp.n_split > 0 ? sp.n_split : sp.n_workers - 1, cdiv(sp.rows_unit, 4));
    cfg.blockDim = dim3(128);
    cfg.stream = stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tree_attn_fixup_kernel, sp);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

}  // namespace sdb
