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
  uint64_t s_full[2], p_full[2];  // per TMEM S buffer
  uint64_t o_done[NT], o_free[NT];
  uint32_t tmem_base;
  float xmax[2][4][128];  // quarter-row maxima, double-buffered by item parity
  float xsum[4][128];     // quarter-row sums (epilogue)
};

constexpr int kSoftmaxWarps = 16;  // 4 TMEM lane groups x 4 column quarters
constexpr int kPairThreads = 128 + kSoftmaxWarps * 32;

// Softmax of one item for this thread's row, columns [32 qtr, 32 qtr + 32) of
// the S buffer at t_s.  The row max is combined with the 3 other quarters of
// the row (same TMEM lane group) through shared memory under a 128-thread
// named barrier; the row sum stays partial (combined in the epilogue; every
// quarter applies the same max, so partial sums add).  P (bf16) for the
// quarter lands in packed columns [16 qtr, 16 qtr + 16) -- every quarter has
// loaded its S before the barrier.  O columns [32 qtr, +32) are rescaled in
// place when the max grows by more than 2^8: the previous PV into this O
// completed before this S was committed (in-order tensor pipe).
template <int EMU>
__device__ __forceinline__ void softmax_quarter(uint32_t t_s, uint32_t t_o, int qtr, float sl2, bool first, bool pref,
                                                int kvalid, const uint32_t *mrow, int key0, int n_words, bool row_ok,
                                                float *xmax, int row, int bar_id, float &m, float &l) {
  const bool full = pref && kvalid >= kTileN;
  uint32_t r[32];
  SDB_TMEM_LD32(t_s + 32 * qtr, r);
  uint32_t vm = 0xffffffffu;
  if (!full) {
    const int lim = kvalid - 32 * qtr;
    const uint32_t low = lim >= 32 ? 0xffffffffu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
    uint32_t bits = 0xffffffffu;
    if (!pref) {
      const int wi = (key0 >> 5) + qtr;
      bits = (wi < n_words && row_ok) ? mrow[wi] : 0u;
    }
    vm = bits & low;
  }
  tmem_wait_ld();
  if (!full) {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (!((vm >> e) & 1u)) r[e] = 0xff800000u;
  }
  float c0 = fmax3(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]));
  float c1 = fmax3(__uint_as_float(r[3]), __uint_as_float(r[4]), __uint_as_float(r[5]));
  float c2 = fmax3(__uint_as_float(r[6]), __uint_as_float(r[7]), __uint_as_float(r[8]));
  float c3 = fmax3(__uint_as_float(r[9]), __uint_as_float(r[10]), __uint_as_float(r[11]));
#pragma unroll
  for (int e = 12; e < 28; e += 8) {
    c0 = fmax3(c0, __uint_as_float(r[e + 0]), __uint_as_float(r[e + 1]));
    c1 = fmax3(c1, __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
    c2 = fmax3(c2, __uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]));
    c3 = fmax3(c3, __uint_as_float(r[e + 6]), __uint_as_float(r[e + 7]));
  }
  c0 = fmax3(c0, __uint_as_float(r[28]), __uint_as_float(r[29]));
  c1 = fmax3(c1, __uint_as_float(r[30]), __uint_as_float(r[31]));
  xmax[qtr * 128 + row] = fmax3(fmaxf(c0, c1), c2, c3);
  asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
  const float mx = fmaxf(fmaxf(xmax[row], xmax[128 + row]), fmaxf(xmax[256 + row], xmax[384 + row])) * sl2;
  float corr = 1.f;
  bool rescale = false;
  if (first) {
    m = mx;
  } else if (mx > m + kRescaleThreshold) {
    corr = ex2(m - mx);
    rescale = true;
    m = mx;
  }
  const float neg_mu = (m == -INFINITY) ? 0.f : -m;
  const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_mu, neg_mu);
  uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    float x0, x1, p0, p1;
    f2unpack(ffma2(f2pack(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), sc2, nm2), x0, x1);
    if ((e & 3) >= 4 - EMU) {
      ex2_emu2(x0, x1, p0, p1);
    } else {
      p0 = ex2(x0);
      p1 = ex2(x1);
    }
    acc2[e & 3] = fadd2(acc2[e & 3], f2pack(p0, p1));
    r[e] = pack_bf16(p0, p1);
  }
  float s0, s1, s2, s3, s4, s5, s6, s7;
  f2unpack(fadd2(acc2[0], acc2[1]), s0, s1);
  f2unpack(fadd2(acc2[2], acc2[3]), s2, s3);
  l = l * corr + ((s0 + s1) + (s2 + s3));
  (void)s4; (void)s5; (void)s6; (void)s7;
  SDB_TMEM_ST16(t_s + 16 * qtr, r);
  if (rescale) {
    uint32_t o[32];
    SDB_TMEM_LD32(t_o + 32 * qtr, o);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
    SDB_TMEM_ST32(t_o + 32 * qtr, o);
  }
  tmem_wait_st();
  tc_fence_before();
}

// Epilogue for a quarter row: O columns [32 qtr, +32) normalised by the full
// row sum; quarter 0 also writes the LSE.
__device__ __forceinline__ void epilogue_quarter(const Sm100Params &sp, const Item &item, const ItemGeo &geo, int g,
                                                 int local, int qtr, uint32_t t_o, float m, float l_full) {
  const TreeAttnParams &p = sp.p;
  const int rho = geo.row0 + local;
  const bool row_ok = rho < geo.rows_total;
  const bool in_range = rho < p.r_max * g;
  const int node_o = rho / g;
  const int hq_idx = geo.kvh * g + (rho % g);
  const float inv = l_full > 0.f ? 1.f / l_full : 0.f;
  const float lse_n = l_full > 0.f ? (m + __log2f(l_full)) * 0.6931471805599453f : -INFINITY;
  uint32_t r[32];
  SDB_TMEM_LD32(t_o + 32 * qtr, r);
  tmem_wait_ld();
  const int col0 = 32 * qtr;
  if (item.whole) {
    if (in_range) {
      __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                         (((int64_t)geo.b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim + col0;
#pragma unroll
      for (int e = 0; e < 32; e += 8) {
        uint4 v;
        if (row_ok) {
          v.x = pack_bf16(__uint_as_float(r[e + 0]) * inv, __uint_as_float(r[e + 1]) * inv);
          v.y = pack_bf16(__uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
          v.z = pack_bf16(__uint_as_float(r[e + 4]) * inv, __uint_as_float(r[e + 5]) * inv);
          v.w = pack_bf16(__uint_as_float(r[e + 6]) * inv, __uint_as_float(r[e + 7]) * inv);
        } else {
          v = make_uint4(0, 0, 0, 0);
        }
        *reinterpret_cast<uint4 *>(o + e) = v;
      }
      if (qtr == 0 && p.lse)
        p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
    }
  } else {
    float *o = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim + col0;
#pragma unroll
    for (int e = 0; e < 32; e += 4)
      *reinterpret_cast<float4 *>(o + e) = make_float4(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv,
                                                       __uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
    if (qtr == 0) sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = row_ok ? lse_n : -INFINITY;
  }
}

// Work items of a unit: (KV tile j, query tile t), n = j * NT + t, processed
// in that order by all 16 softmax warps.  TMEM: two S buffers [0,128) and
// [128,256) alternate by global item parity, O_t at [256 + 128 t, +128).  The
// MMA issuer keeps the tensor pipe one item ahead: after P(n) it issues
// PV(n) then S(n + 2) (into the buffer P(n) just vacated -- in-order pipe),
// so S(n + 1) is already computed when the softmax finishes item n and the
// softmax warps run items back to back.
template <int NT, int EMU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
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
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.s_full[b], 1);
      mbar_init(&sm.p_full[b], 2 * kSoftmaxWarps);  // one arrival per softmax warp of both CTAs
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(&sm.o_done[t], 1);
      mbar_init(&sm.o_free[t], 2 * kSoftmaxWarps);
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
    // The whole warp walks the schedule (warp-uniform control flow and
    // descriptors in uniform registers); one elected lane issues.  A single
    // divergent issuing thread made ptxas wrap every tcgen05.mma in an
    // R2UR / ELECT loop (~16 instructions per MMA), which starved the tensor
    // pipe once the softmax warps saturated the issue slots.
    if (rank == 0) {
      constexpr uint32_t idesc_s = make_idesc2(false);
      constexpr uint32_t idesc_o = make_idesc2(true);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint64_t q_desc = sw128_desc(smem_u32(sm.q[0]), 16, 1024);
      const uint64_t k_desc = sw128_desc(smem_u32(sm.k[0]), 16, 1024);
      const uint64_t v_desc = sw128_desc(smem_u32(sm.v[0]), kHalfBytes, 1024);
      uint32_t g_tile = 0, g_q = 0, g_item = 0;
      ItemIter iter(sp, worker);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        const int n_tiles = __shfl_sync(0xffffffffu, geo.n_tiles, 0);
        const int N = NT * n_tiles;
        // S(n) = Q_t K_j^T into S buffer (g_item + n) & 1 (descriptor start
        // addresses are in 16-byte units, low 14 bits: smem < 256 KB, no carry)
        auto issue_item_s = [&](int n) {
          const int j = n / NT, t = n % NT;
          const uint32_t gt = g_tile + j;
          const int st = gt % kStages2;
          if (t == 0) {
            mbar_wait(&sm.k_full[st], (gt / kStages2) & 1);
            tc_fence_after();
          }
          if (elect_one()) {
            const uint32_t d = tm + ((g_item + n) & 1) * 128;
            const uint64_t qd = q_desc + (uint64_t)((t * kTileBytes) >> 4);
            const uint64_t kd = k_desc + (uint64_t)((st * kHalfBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kHeadDim / 16; ++k)
              mma2_ss(d, qd + (uint64_t)(((k >> 2) * kChunkBytes + (k & 3) * 32) >> 4),
                      kd + (uint64_t)(((k >> 2) * kKChunk + (k & 3) * 32) >> 4), idesc_s, k > 0);
            tc_commit2(&sm.s_full[(g_item + n) & 1]);
            if (t == NT - 1) tc_commit2(&sm.k_empty[st]);
          }
          __syncwarp();
        };
        mbar_wait(&sm.q_full, g_q & 1);
        tc_fence_after();
        issue_item_s(0);
        if (N > 1) issue_item_s(1);
        for (int n = 0; n < N; ++n) {
          const int j = n / NT, t = n % NT;
          const uint32_t gt = g_tile + j;
          const int st = gt % kStages2;
          const uint32_t gi = g_item + n;
          if (t == 0) mbar_wait(&sm.v_full[st], (gt / kStages2) & 1);
          TRACE(0, gi);
          mbar_wait_cluster(&sm.p_full[gi & 1], (gi >> 1) & 1);
          TRACE(1, gi);
          if (j == 0) mbar_wait_cluster(&sm.o_free[t], (g_q & 1) ^ 1);  // previous unit's epilogue read O_t
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a = tm + (gi & 1) * 128;
            const uint64_t vd = v_desc + (uint64_t)((st * kHalfBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kTileN / 16; ++k)
              mma2_ts(tm + 256 + t * 128, a + k * 8, vd + (uint64_t)((k * 2048) >> 4), idesc_o,
                      (j > 0 || k > 0) ? 1u : 0u);
            tc_commit2(&sm.o_done[t]);
            if (t == NT - 1) tc_commit2(&sm.v_empty[st]);
          }
          __syncwarp();
          if (n + 2 < N) issue_item_s(n + 2);
          TRACE(2, gi);
        }
        if (elect_one()) tc_commit2(&sm.q_empty);
        __syncwarp();
        g_tile += n_tiles;
        g_item += N;
        ++g_q;
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax (both CTAs, all 16 warps per item) =========
    const int lg = warp & 3;            // TMEM lane group (warp % 4 by hardware rule)
    const int qtr = (warp - 4) >> 2;    // column quarter
    const int i = (lg << 5) + lane;     // row within the CTA's 128-row half of a query tile
    const int bar_id = 1 + lg;
    const uint32_t lane_off = (uint32_t)(lg * 32) << 16;
    uint32_t g_item = 0, g_o = 0;
    ItemIter iter(sp, worker);
    Item item;
    while (iter.next(sp, item)) {
      const ItemGeo geo = item_geo(sp, item, g);
      int local[NT];
      bool row_ok[NT];
      const uint32_t *mrow[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        local[t] = t * 2 * kTileM + (int)rank * kTileM + i;
        const int rho = geo.row0 + local[t];
        row_ok[t] = rho < geo.rows_total;
        const int node = min(rho / g, max(geo.n_nodes - 1, 0));
        mrow[t] = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
      }
      if (!geo.active) {
        if (qtr == 0)
#pragma unroll
          for (int t = 0; t < NT; ++t) inactive_row(sp, item, geo, g, local[t]);
        continue;
      }
      float m[NT], l[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        m[t] = -INFINITY;
        l[t] = 0.f;
      }
      for (int j = 0; j < geo.n_tiles; ++j) {
        const bool pref = j < geo.n_pref;
        const int key0 = pref ? (geo.pa + j) * kTileN : (geo.sa + j - geo.n_pref) * kTileN;
        const int kvalid = pref ? geo.C - key0 : geo.n_nodes - key0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const uint32_t gi = g_item + j * NT + t;
          if (rank == 0 && warp == 4 && lane == 0) TRACE(3, gi);
          mbar_wait(&sm.s_full[gi & 1], (gi >> 1) & 1);
          tc_fence_after();
          if (rank == 0 && warp == 4 && lane == 0) TRACE(4, gi);
          softmax_quarter<EMU>(tmem + lane_off + (gi & 1) * 128, tmem + lane_off + 256 + t * 128, qtr, sl2, j == 0,
                               pref, kvalid, mrow[t], key0, p.n_words, row_ok[t], &sm.xmax[gi & 1][0][0], i, bar_id,
                               m[t], l[t]);
          __syncwarp();
          if (lane == 0) {
            if (rank == 0)
              mbar_arrive(&sm.p_full[gi & 1]);
            else
              mbar_arrive_leader(&sm.p_full[gi & 1]);
          }
          if (rank == 0 && warp == 4 && lane == 0) TRACE(5, gi);
        }
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        mbar_wait(&sm.o_done[t], (g_o + geo.n_tiles - 1) & 1);
        tc_fence_after();
        sm.xsum[qtr][i] = l[t];
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        const float l_full = (sm.xsum[0][i] + sm.xsum[1][i]) + (sm.xsum[2][i] + sm.xsum[3][i]);
        epilogue_quarter(sp, item, geo, g, local[t], qtr, tmem + lane_off + 256 + t * 128, m[t], l_full);
        tc_fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");  // xsum reuse
        __syncwarp();
        if (lane == 0) {
          if (rank == 0)
            mbar_arrive(&sm.o_free[t]);
          else
            mbar_arrive_leader(&sm.o_free[t]);
        }
      }
      g_o += geo.n_tiles;
      g_item += NT * geo.n_tiles;
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
    tree_attn_tcgen05_pair_kernel<NT, EMU><<<grid, kPairThreads, smem, stream>>>(mq, mk, mv, mtk, mtv, sp);   \
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
