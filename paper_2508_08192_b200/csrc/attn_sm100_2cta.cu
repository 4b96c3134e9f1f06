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

// ring depths: C3 attention alone 534 us (K 6 / V 3), 520 (6 / 4), 518 (5 / 5):
// with the fixed-reference softmax the MMA issuer waited ~580 cycles per
// item for V with three stages
#ifndef SDB_STAGES_K
#define SDB_STAGES_K 5
#endif
constexpr int kStagesK = SDB_STAGES_K;  // K ring: S(n) is issued ~3 items before its PV, so K needs the deeper ring
#ifndef SDB_STAGES_V
#define SDB_STAGES_V 5
#endif
constexpr int kStagesV = SDB_STAGES_V;  // (3 suffice: V(n) is consumed by PV(n), ~3 items after its load is issued)

#ifdef SDB_TRACE
// [event][iteration] clock64 stamps of worker 0 (debug builds only)
__device__ unsigned long long g_trace[24][256];
#ifndef SDB_TRACE_WORKER
#define SDB_TRACE_WORKER 0
#endif
#define TRACE(ev, it)                                                                   \
  do {                                                                                  \
    if (worker == SDB_TRACE_WORKER && (it) < 256) g_trace[ev][it] = clock64();          \
  } while (0)
// [event][worker] globaltimer stamps of every worker
#define TRACE_G(ev)                                                                     \
  do {                                                                                  \
    unsigned long long t_;                                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
    if (worker < 256) g_trace[ev][worker] = t_;                                         \
  } while (0)
#else
#define TRACE(ev, it) \
  do {                \
  } while (0)
#define TRACE_G(ev) \
  do {              \
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
// fused tail rows: generic shared-memory data handed across the pair (P^T
// halves, unit-end statistics) -- cluster-scope release / acquire
__device__ __forceinline__ void mbar_arrive_remote_rel(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_peer_f32(float *p, uint32_t cta, float v) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\nst.shared::cluster.f32 [ra], %2;\n}" ::"r"(
          smem_u32(p)),
      "r"(cta), "f"(v)
      : "memory");
}
#define SDB_TMEM_WAIT_LD_REGS16(r)                                                                                \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                    \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),  \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),         \
                 "+r"(r[15])::"memory")

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
__host__ __device__ constexpr uint32_t make_idesc2(bool b_mn_major, bool a_mn_major = false, int n = kTileN) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

constexpr int kLgStages = kStagesK + kStagesV <= 9 ? 5 : 3;  // fused argmax: 8 KB bulk-copy ring in the SMEM left over
constexpr int kLgChunk = 2048;   // floats per chunk

struct alignas(1024) Smem2 {
  uint8_t q[kTileBytes];  // this CTA's 128 query rows
  uint8_t k[kStagesK][kHalfBytes];
  uint8_t v[kStagesV][kHalfBytes];
  // fused tail rows (R = 65): the B operands of the two N = 16 tail MMAs
  uint8_t qt[2][1024];  // Q of the 8 tail rows, [8 rows][64 d] per head-dim half (both CTAs load it)
  uint8_t pt[2][1024];  // P^T, [8 rows][64 keys] per key half: this CTA writes half `rank`, the other stays 0
  uint64_t q_full, q_empty;
  uint64_t ts_full, tp_full, to_full, tread, tstat;  // tail S^T done / P^T written / O^T partial done / read; stats
  float tref[2][8];       // tail warps: per-warp row max of the reference item
  float tl[2][8];         // ... per-warp row sums at the unit end
  uint32_t tbad[2];       // ... per-warp "row needs the exact recompute" masks
  float tx[2][2][17];     // [unit parity][cta]: reference, row sum and bad mask (bits) of each tail row
  uint64_t k_full[kStagesK], k_empty[kStagesK], v_full[kStagesV], v_empty[kStagesV];
  uint64_t s_full[3], p_full[3], o_done[3];  // per TMEM S slot (o_done: running-max mode only)
  uint64_t o_last;  // the unit's last PV done (epilogue may read O)
  uint64_t o_free;
  uint32_t tmem_base;
  float mref[3][128];  // running reference max after each item (log2 units), by slot
  float lsum[3][128];  // per-warpgroup partial row sums at the end of a unit
  float msum[3][128];  // ... and the reference max they are relative to
  uint32_t bad[128];   // fixed reference exceeded in this row of the unit (exact recompute)
  alignas(128) float lg[kLgStages][kLgChunk];  // fused greedy scan: logits chunk ring (warp 3; 16-B aligned for TMA)
  uint64_t lg_full[kLgStages];
};

static_assert(sizeof(Smem2) + 1024 <= 232448, "shared memory");

constexpr int kSoftmaxWG = 3;                       // softmax warpgroups (one per S slot)
// register split (65536 per SM, one CTA per SM): the TMA / MMA / scan
// warpgroup keeps 56 per thread, the softmax warpgroups get 152
// measured (C3, attention alone): no reallocation 525 us; 56 / 152 536 us
// (and an intermittent hang); 32 / 160 569 us (the control warps spill) --
// the 128-register budget with its few softmax spills is the fastest
#ifndef SDB_REGS_CTL
#define SDB_REGS_CTL 0
#endif
#ifndef SDB_REGS_SOFTMAX
#define SDB_REGS_SOFTMAX 152
#endif
constexpr int kRegsCtl = SDB_REGS_CTL;  // 0: no register reallocation
constexpr int kRegsSoftmax = SDB_REGS_SOFTMAX;
static_assert(kRegsCtl == 0 || kRegsCtl * 128 + kRegsSoftmax * 128 * kSoftmaxWG <= 65536, "register file");
constexpr int kPairThreads = 128 + kSoftmaxWG * 128;
constexpr int kSBase = 128;                          // TMEM: O [0,128), S slot s at 128 + 128 s
constexpr int kBarUnit = 1 + 4 * kSoftmaxWG;         // named barrier: unit end, all softmax warps
constexpr int kBarTail = kBarUnit + 1;               // named barrier: the two tail warps
#ifndef SDB_ATTN_FIXREF
#define SDB_ATTN_FIXREF 1
#endif
// Fixed reference max: after the first item of a unit piece, P = exp2(s -
// m_ref) against that item's row max, with no max pass and no max hand-off
// (P, O and the row sum are all relative to one reference, so nothing is
// ever rescaled).  fp32 / bf16 hold 2^127, so exactness only needs the scores
// to stay below m_ref + ~89 (log2 units); a row that exceeds it (a score ~60
// nats above the first 32 scores of the piece's first tile) is recomputed
// exactly.
constexpr bool kFixRef = SDB_ATTN_FIXREF != 0;

// Epilogue: O columns [16 c, 16 c + 16) of this row normalised by the row sum
// (bf16 output of a whole unit, fp32 partial of a split one); chunk 0 writes
// the LSE.  Eight 16-column chunks spread 3 / 3 / 2 over the softmax
// warpgroups (the unit-end drain is on the critical path of the next unit).
__device__ __forceinline__ void epilogue_chunk(const Sm100Params &sp, const Item &item, const ItemGeo &geo, int g,
                                               int local, int c, uint32_t t_o, float m, float l_full) {
  const TreeAttnParams &p = sp.p;
  const int rho = geo.row0 + local;
  const bool row_ok = rho < geo.rows_total;
  const bool in_range = geo.q0 * g + rho < p.r_max * g;
  const int node_o = geo.q0 + rho / g;
  const int hq_idx = geo.kvh * g + (rho % g);
  const float inv = l_full > 0.f ? 1.f / l_full : 0.f;
  const float lse_n = l_full > 0.f ? (m + __log2f(l_full)) * 0.6931471805599453f : -INFINITY;
  uint32_t r[16];
  SDB_TMEM_LD16(t_o + 16 * c, r);
  tmem_wait_ld();
  const int col0 = 16 * c;
  if (item.whole) {
    if (in_range) {
      __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                         (((int64_t)geo.b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim + col0;
#pragma unroll
      for (int e = 0; e < 16; e += 8) {
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
      if (c == 0 && p.lse)
        p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
    }
  } else {
    float *o = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim + col0;
#pragma unroll
    for (int e = 0; e < 16; e += 4)
      *reinterpret_cast<float4 *>(o + e) = make_float4(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv,
                                                       __uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
    if (c == 0) sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = row_ok ? lse_n : -INFINITY;
  }
}

// Items of a unit are its KV tiles n = 0 .. N-1 (one 256-row query tile per
// pair, 128 rows per CTA).  Item n lives in TMEM S slot gi % 3 (gi = the
// worker's running item count) and is softmaxed by warpgroup gi % 3, so the
// three warpgroups work on three consecutive items at once and each has about
// two items of tensor-pipe time to finish its own.  The online-softmax
// reference max is handed from item to item along a chain of named barriers
// (only the max: it is known after the first pass over S); each warpgroup
// keeps its partial row sum relative to the last reference it saw, and the
// partial sums are combined at the end of the unit.  The MMA issuer runs
// PV(n) and then S(n + 3) into the slot P(n) just vacated (in-order pipe).
template <int EMU8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    tree_attn_tcgen05_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_qt,
                                  const __grid_constant__ CUtensorMap tm_k,
                                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tk,
                                  const __grid_constant__ CUtensorMap tm_tv, const __grid_constant__ Sm100Params sp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem2 &sm = *reinterpret_cast<Smem2 *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TreeAttnParams &p = sp.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.hq / p.hkv;
  const float sl2 = p.scale * 1.4426950408889634f;
  const uint32_t rank = cta_rank();
  const int worker = blockIdx.x >> 1;
  griddep_launch_dependents();  // the fix-up grid may become resident (it waits for our completion)
  if (threadIdx.x == 0 && rank == 0) TRACE(8, 0);
  if (threadIdx.x == 0 && rank == 0) TRACE_G(13);

  if (threadIdx.x == 0) {
    if (rank == 0) {
      sp.seg[worker] = seg_begin(sp, worker);
      if (worker == 0) sp.seg[sp.n_workers] = sp.total;
    }
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int s = 0; s < kStagesK; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kStagesV; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.p_full[s], 2 * 4);  // the 4 warps of the slot's warpgroup in both CTAs
      mbar_init(&sm.o_done[s], 1);
    }
    mbar_init(&sm.o_last, 1);
    mbar_init(&sm.o_free, 2 * 4 * kSoftmaxWG);
    mbar_init(&sm.ts_full, 1);
    mbar_init(&sm.tp_full, 2 * 2);  // tail warps 2 / 3 of both CTAs
    mbar_init(&sm.to_full, 1);
    mbar_init(&sm.tread, 2 * 2);
    mbar_init(&sm.tstat, 1);        // the peer's tail warp 2
    for (int s = 0; s < kLgStages; ++s) mbar_init(&sm.lg_full[s], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 128) sm.bad[threadIdx.x] = 0u;
  if (sp.tail_rows > 0 && threadIdx.x < 256) {
    // the other CTA's key half of this CTA's P^T rows is zero for good
    reinterpret_cast<uint32_t *>(sm.pt[rank ^ 1u])[threadIdx.x] = 0u;
    fence_proxy_async_smem();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (threadIdx.x == 0 && rank == 0) TRACE(9, 0);
  // (each role's code must be dominated by its setmaxnreg: ptxas allocates
  // a region reached from both budgets with the smaller one)
  if (warp < 4) {
  if (kRegsCtl) regs_dec<kRegsCtl ? kRegsCtl : 128>();
  const bool tail_mode = sp.tail_rows > 0;  // fused tail rows: warps 2 / 3 run them, warp 0 loads K and V
  if (warp == 0 || (warp == 2 && !tail_mode)) {
    // ============ TMA producers (both CTAs): warp 0 Q + K ring, warp 2 V ring ============
    // Each CTA loads its own half of every tile; completion bytes land on the
    // leader's barriers.  Separate K and V producers so a K load never waits
    // behind a V slot (and vice versa).  The whole warp walks the schedule:
    // the block-table entries of the next 32 pages are fetched by the 32 lanes
    // in one coalesced load and handed to the issuing lane by shuffles, so a
    // tile's TMA issue never waits for a dependent global load (with one
    // block-table load per page on the issuing lane, the V producer's two
    // serial loads per tile took longer than the tile's tensor work).
    {
      const bool kprod = warp == 0;
      const bool vprod = warp == 2 || tail_mode;
      if (lane == 0) {
        if (kprod) {
          tma_prefetch(&tm_q);
          tma_prefetch(&tm_k);
          tma_prefetch(&tm_tk);
          if (tail_mode) tma_prefetch(&tm_qt);
        }
        if (vprod) {
          tma_prefetch(&tm_v);
          tma_prefetch(&tm_tv);
        }
      }
      const int bs = p.block_size;
      const int seg_rows = bs < 64 ? bs : 64;
      const uint32_t l_qfull = leader_addr(&sm.q_full);
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, worker);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        // the plan covers w_pref prefix tiles: a longer context (ctx_len >
        // max_ctx) would lose keys -- flag it instead (CacheError)
        if (kprod && lane == 0 && rank == 0 && p.err && geo.C - geo.k0 > sp.w_pref * kTileN)
          atomicOr(p.err, SDB_ERR_CACHE);
        if (kprod) {
          mbar_wait(&sm.q_empty, (g_q & 1) ^ 1);
          if (lane == 0) {
            const bool tail_unit = tail_mode && item.unit / (p.batch * p.hkv) == sp.m_blocks - 1;
            if (rank == 0) mbar_expect_tx(&sm.q_full, 2 * kTileBytes + (tail_unit ? 2 * 2048 : 0));
            const int node0 = geo.q0 + (geo.row0 + (int)rank * kTileM) / g;
            for (int c = 0; c < 2; ++c)
              tma2_4d(sm.q + c * kChunkBytes, &tm_q, l_qfull, c * 64, 0, geo.kvh, geo.b * p.r_max + node0);
            if (tail_unit) {
              const int node_t = geo.q0 + (geo.row0 + sp.row_blk) / g;
              for (int c = 0; c < 2; ++c)
                tma2_4d(sm.qt[c], &tm_qt, l_qfull, c * 64, 0, geo.kvh, geo.b * p.r_max + node_t);
            }
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
          const bool pref = it < geo.n_pref;
          const int tile = pref ? geo.pa + it : geo.sa + (it - geo.n_pref);
          if (kprod) {
            // K half: keys [tile*128 + rank*64, +64), all 128 head-dim columns
            const int s = g_tile % kStagesK;
            mbar_wait(&sm.k_empty[s], ((g_tile / kStagesK) & 1) ^ 1);
            if (rank == 0 && lane == 0) TRACE(17, g_tile);
            const uint32_t l_kfull = leader_addr(&sm.k_full[s]);
            if (lane == 0 && rank == 0) mbar_expect_tx(&sm.k_full[s], 2 * kHalfBytes);
            if (pref) {
              for (int r0 = 0; r0 < 64; r0 += seg_rows) {
                const int key = geo.k0 + tile * kTileN + (int)rank * 64 + r0;
                const int page = page_of(key / bs);
                const int rowc = (page * p.hkv + geo.kvh) * bs + key % bs;
                if (lane == 0)
                  for (int c = 0; c < 2; ++c) tma2_2d(sm.k[s] + c * kKChunk + r0 * 128, &tm_k, l_kfull, c * 64, rowc);
              }
            } else if (lane == 0) {
              for (int c = 0; c < 2; ++c)
                tma2_3d(sm.k[s] + c * kKChunk, &tm_tk, l_kfull, c * 64, geo.kvh,
                        geo.b * p.r_max + tile * kTileN + (int)rank * 64);
            }
          }
          if (vprod) {
            // V half: all 128 keys, head-dim columns [rank*64, +64)
            const int s = g_tile % kStagesV;
            mbar_wait(&sm.v_empty[s], ((g_tile / kStagesV) & 1) ^ 1);
            if (rank == 0 && lane == 0) TRACE(16, g_tile);
            const uint32_t l_vfull = leader_addr(&sm.v_full[s]);
            if (lane == 0 && rank == 0) mbar_expect_tx(&sm.v_full[s], 2 * kHalfBytes);
            if (pref) {
              for (int r0 = 0; r0 < kTileN; r0 += seg_rows) {
                const int key = geo.k0 + tile * kTileN + r0;
                const int page = page_of(key / bs);
                const int rowc = (page * p.hkv + geo.kvh) * bs + key % bs;
                if (lane == 0) tma2_2d(sm.v[s] + r0 * 128, &tm_v, l_vfull, (int)rank * 64, rowc);
              }
            } else if (lane == 0) {
              tma2_3d(sm.v[s], &tm_tv, l_vfull, (int)rank * 64, geo.kvh, geo.b * p.r_max + tile * kTileN);
            }
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
      constexpr uint32_t idesc_ts = make_idesc2(false, false, 16);  // tail S^T: K (keys x d) . Q_t^T
      constexpr uint32_t idesc_tp = make_idesc2(false, true, 16);   // tail O^T: V^T (d x keys, MN-major) . P_t^T
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint64_t q_desc = sw128_desc(smem_u32(sm.q), 16, 1024);
      const uint64_t k_desc = sw128_desc(smem_u32(sm.k[0]), 16, 1024);
      const uint64_t v_desc = sw128_desc(smem_u32(sm.v[0]), kHalfBytes, 1024);
      uint32_t g_tile = 0, g_q = 0, g_item = 0, tgp = 0, tgr = 0;
      ItemIter iter(sp, worker);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        const int N = __shfl_sync(0xffffffffu, geo.n_tiles, 0);
        const bool tail_unit = tail_mode && item.unit / (p.batch * p.hkv) == sp.m_blocks - 1;
        // S(n) = Q K_n^T into slot (g_item + n) % 3 (descriptor start
        // addresses are in 16-byte units, low 14 bits: smem < 256 KB, no carry)
        auto issue_s = [&](int n) {
          const uint32_t gt = g_tile + n;
          const int st = gt % kStagesK;
          const int slot = (g_item + n) % 3;
          mbar_wait(&sm.k_full[st], (gt / kStagesK) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t kd = k_desc + (uint64_t)((st * kHalfBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kHeadDim / 16; ++k)
              mma2_ss(tm + kSBase + slot * 128, q_desc + (uint64_t)(((k >> 2) * kChunkBytes + (k & 3) * 32) >> 4),
                      kd + (uint64_t)(((k >> 2) * kKChunk + (k & 3) * 32) >> 4), idesc_s, k > 0);
            tc_commit2(&sm.s_full[slot]);
            if (!tail_unit) {  // (tail units: K(n) and Q_t are read again by the tail S^T(n))
              tc_commit2(&sm.k_empty[st]);
              // the unit's last S: Q is free once it completes, so the next
              // unit's Q load overlaps this unit's last three items
              if (n == N - 1) tc_commit2(&sm.q_empty);
            }
          }
          __syncwarp();
        };
        // fused tail rows: the O^T partial of item m (V(m) x P^T(m) of both
        // CTAs) into columns [48, 64) of TMEM slot dst (lanes 64..127: this
        // CTA's 64 head-dim columns; D columns 0..7 from CTA 0's keys, 8..15
        // from CTA 1's).  The A operands start one 1 KB V row group / one
        // 8 KB K chunk early so the live rows land on lanes 64..127 (the
        // lanes warps 2 / 3 may access); the rows before are don't-care reads
        // of this CTA's own shared memory.
        auto tail_pv = [&](int m, int dst) {
          const int vst = (int)((g_tile + m) % kStagesV);
          mbar_wait_acq_cluster(&sm.tp_full, tgp & 1);
          TRACE(21, g_item + m + 1);
          ++tgp;
          tc_fence_after();
          if (elect_one()) {
            const uint32_t vb = smem_u32(sm.v[vst]) - 1024;
            const uint32_t pb = smem_u32(sm.pt[0]);
#pragma unroll
            for (int k = 0; k < kTileN / 16; ++k)
              mma2_ss(tm + kSBase + dst * 128 + 48, sw128_desc(vb + k * 2048, 1024, 1024),
                      sw128_desc(pb + (k >> 2) * 1024 + (k & 3) * 32, 16, 1024), idesc_tp, k > 0 ? 1u : 0u);
            tc_commit2(&sm.to_full);
            tc_commit2(&sm.v_empty[vst]);
          }
          __syncwarp();
        };
        mbar_wait(&sm.q_full, g_q & 1);
        tc_fence_after();
        for (int n = 0; n < 3 && n < N; ++n) issue_s(n);
        for (int n = 0; n < N; ++n) {
          const uint32_t gt = g_tile + n;
          const int st = gt % kStagesV;
          const uint32_t gi = g_item + n;
          const int slot = gi % 3;
          TRACE(18, gi);
          mbar_wait(&sm.v_full[st], (gt / kStagesV) & 1);
          TRACE(0, gi);
          mbar_wait_cluster(&sm.p_full[slot], (gi / 3) & 1);
          TRACE(1, gi);
          if (n == 0) mbar_wait_cluster(&sm.o_free, (g_q & 1) ^ 1);  // previous unit's epilogue read O
          tc_fence_after();
          if (tail_unit) {
            // fused tail rows: the O^T partial of item n - 1 (its P^T was
            // written during the previous item) and S^T of item n go ahead of
            // PV(n), into columns [48, 64) / [16, 32) of this slot -- free
            // since P(n) is packed into [32c, 32c + 16) -- so warps 2 / 3 have
            // read both while PV(n) runs, and S(n + 3) reclaims the slot
            // without a tensor-pipe bubble
            if (n > 0) tail_pv(n - 1, slot);
            const int kst = gt % kStagesK;
            if (elect_one()) {
              const uint32_t kb = smem_u32(sm.k[kst]) - kKChunk;
              const uint32_t qb = smem_u32(sm.qt[0]);
#pragma unroll
              for (int k = 0; k < kHeadDim / 16; ++k)
                mma2_ss(tm + kSBase + slot * 128 + 16, sw128_desc(kb + (k >> 2) * kKChunk + (k & 3) * 32, 16, 1024),
                        sw128_desc(qb + (k >> 2) * 1024 + (k & 3) * 32, 16, 1024), idesc_ts, k > 0 ? 1u : 0u);
              tc_commit2(&sm.ts_full);
              tc_commit2(&sm.k_empty[kst]);
              if (n == N - 1) tc_commit2(&sm.q_empty);
            }
            __syncwarp();
          }
          if (elect_one()) {
            // P of keys 16k .. 16k+15 at slot columns 32 (k/2) + 8 (k%2)
            const uint32_t a = tm + kSBase + slot * 128;
            const uint64_t vd = v_desc + (uint64_t)((st * kHalfBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kTileN / 16; ++k)
              mma2_ts(tm, a + 32 * (k >> 1) + 8 * (k & 1), vd + (uint64_t)((k * 2048) >> 4), idesc_o,
                      (n > 0 || k > 0) ? 1u : 0u);
            // O progress is only waited on by a rescale (running-max mode)
            // and by the unit's epilogue (its last PV)
            if (!kFixRef) tc_commit2(&sm.o_done[slot]);
            if (n == N - 1) tc_commit2(&sm.o_last);
            if (!tail_unit) tc_commit2(&sm.v_empty[st]);  // (tail units: V(n) is read again by the O^T partial)
          }
          __syncwarp();
          if (tail_unit) {
            mbar_wait_cluster(&sm.tread, tgr & 1);  // warps 2 / 3 of both CTAs read the slot's tail columns
            TRACE(22, gi);
            ++tgr;
            tc_fence_after();
          }
          if (n + 3 < N) issue_s(n + 3);
          TRACE(2, gi);
        }
        if (tail_unit) {
          // the last item's O^T partial, into the slot the next unit's S(0) takes
          tail_pv(N - 1, (int)((g_item + N) % 3));
          mbar_wait_cluster(&sm.tread, tgr & 1);
          ++tgr;
          tc_fence_after();
        }
        g_tile += N;
        g_item += N;
        ++g_q;
      }
    }
  } else if (tail_mode) {
    // ============ fused tail rows (warps 2 / 3 of both CTAs) ============
    // The 1..8 query rows past the last full 256-row block (R = 65: node 64's
    // g heads) ride along in that block's units: per item the MMA issuer
    // adds S^T = K_n Q_t^T and the O^T partial V_n^T P_t^T (N = 16, ~1/16 of
    // the item's tensor work), and these two warps -- TMEM lanes 64..127,
    // i.e. this CTA's 64 keys of S^T, then its 64 head-dim columns of O^T --
    // do the softmax (one key per thread, 8 exps), write P^T into this CTA's
    // key half of the B operand, and accumulate the partials in registers.
    // Each CTA keeps its own fixed reference for its key half (the P^T halves
    // land in separate D columns), so the two halves meet only at the unit
    // end: (reference, row sum, overflow flags) are exchanged over DSMEM and
    // each CTA stores its 64 output columns.  Rows whose scores exceed the
    // reference by ~89 log2 units take exact_row, as in the main path.
    griddep_wait();  // the mask words come from the kernel launched just before
    const int tw = warp - 2;
    const int ti = tw * 32 + lane;
    const uint32_t t_lane = (uint32_t)(64 + tw * 32) << 16;
    const uint32_t peer = rank ^ 1u;
    uint32_t g_item = 0, tgs = 0, tgo = 0, tu = 0;
    ItemIter iter(sp, worker);
    Item item;
    while (iter.next(sp, item)) {
      const ItemGeo geo = item_geo(sp, item, g);
      const bool tail_unit = item.unit / (p.batch * p.hkv) == sp.m_blocks - 1;
      if (!geo.active) {
        if (tail_unit && rank == 0 && tw == 0 && lane < sp.tail_rows) inactive_row(sp, item, geo, g, sp.row_blk + lane);
        continue;
      }
      const int N = geo.n_tiles;
      if (!tail_unit) {
        g_item += N;
        continue;
      }
      const int rho0 = geo.row0 + sp.row_blk;  // first tail row
      float mref[8], l[8], oacc[16];
      uint32_t badm = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        mref[j] = -INFINITY;
        l[j] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) oacc[e] = 0.f;
      auto read_partial = [&](int slot_p) {
        // the O^T partial of the previous item: accumulate (columns 0..7:
        // CTA 0's keys against CTA 0's reference, 8..15: CTA 1's)
        uint32_t r[16];
        mbar_wait(&sm.to_full, tgo & 1);
        ++tgo;
        tc_fence_after();
        SDB_TMEM_LD16(tmem + t_lane + kSBase + slot_p * 128 + 48, r);
        SDB_TMEM_WAIT_LD_REGS16(r);
#pragma unroll
        for (int e = 0; e < 16; ++e) oacc[e] += __uint_as_float(r[e]);
      };
      auto arrive_read = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0)
            mbar_arrive(&sm.tread);
          else
            mbar_arrive_leader(&sm.tread);
        }
      };
      for (int n = 0; n < N; ++n) {
        const int slot = (int)((g_item + n) % 3);
        const bool pref = n < geo.n_pref;
        const int key0 = pref ? geo.k0 + (geo.pa + n) * kTileN : (geo.sa + n - geo.n_pref) * kTileN;
        const int key = key0 + (int)rank * 64 + ti;
        if (n > 0) read_partial(slot);  // (item n - 1's partial went into item n's slot)
        uint32_t r[16];
        mbar_wait(&sm.ts_full, tgs & 1);
        if (rank == 0 && ti == 0) TRACE(23, g_item + n);
        ++tgs;
        tc_fence_after();
        SDB_TMEM_LD16(tmem + t_lane + kSBase + slot * 128 + 16, r);
        SDB_TMEM_WAIT_LD_REGS16(r);
        arrive_read();  // the slot may take S(n + 3)
        float sv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          bool vis;
          if (pref) {
            vis = key < geo.C;
          } else {
            const int node = min(geo.q0 + (rho0 + j) / g, max(geo.n_nodes - 1, 0));
            const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
            vis = key < geo.n_nodes && ((__ldg(mrow + (key >> 5)) >> (key & 31)) & 1u);
          }
          sv[j] = vis ? __uint_as_float(r[j]) * sl2 : -INFINITY;
        }
        if (n == 0) {
          // reference: the row max over this CTA's 64 keys of the piece's first tile
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float m = sv[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) sm.tref[tw][j] = m;
          }
          asm volatile("bar.sync %0, 64;" ::"r"(kBarTail) : "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j) mref[j] = fmaxf(sm.tref[0][j], sm.tref[1][j]);
        }
        // P^T row j, key ti of this CTA's half (128-byte swizzle: 16-byte
        // chunk ^ row); the previous P^T was consumed (its partial was read)
        uint8_t *ptb = sm.pt[rank];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float pj = sv[j] == -INFINITY ? 0.f : ex2(sv[j] - (mref[j] == -INFINITY ? 0.f : mref[j]));
          l[j] += pj;
          if (pj > kOverflowSum || (mref[j] == -INFINITY && pj > 0.f)) badm |= 1u << j;
          *reinterpret_cast<__nv_bfloat16 *>(ptb + j * 128 + ((((ti * 2) >> 4) ^ j) << 4) + ((ti * 2) & 15)) =
              __float2bfloat16(pj);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote_rel(&sm.tp_full, 0);
      }
      read_partial((int)((g_item + N) % 3));  // the last item's partial
      arrive_read();
      g_item += N;
      // ---- unit end: this CTA's row sums; (reference, sum, flags) to the peer; store ----
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v = l[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sm.tl[tw][j] = v;
      }
      badm = __reduce_or_sync(0xffffffffu, badm);
      if (lane == 0) sm.tbad[tw] = badm;
      asm volatile("bar.sync %0, 64;" ::"r"(kBarTail) : "memory");
      const int px = (int)(tu & 1);
      if (tw == 0 && lane == 0) {
        float *mine = sm.tx[px][rank];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float lj = sm.tl[0][j] + sm.tl[1][j];
          mine[j] = mref[j];
          mine[8 + j] = lj;
          st_peer_f32(&mine[j], peer, mref[j]);
          st_peer_f32(&mine[8 + j], peer, lj);
        }
        const float bm = __uint_as_float(sm.tbad[0] | sm.tbad[1]);
        mine[16] = bm;
        st_peer_f32(&mine[16], peer, bm);
        mbar_arrive_remote_rel(&sm.tstat, peer);
      }
      asm volatile("bar.sync %0, 64;" ::"r"(kBarTail) : "memory");
      mbar_wait_acq_cluster(&sm.tstat, tu & 1);
      ++tu;
      const uint32_t bad_all = __float_as_uint(sm.tx[px][0][16]) | __float_as_uint(sm.tx[px][1][16]);
      const int col = (int)rank * 64 + ti;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= sp.tail_rows || ((bad_all >> j) & 1u)) continue;  // (flagged rows: exact_row below)
        const float m0 = sm.tx[px][0][j], m1 = sm.tx[px][1][j];
        const float l0 = sm.tx[px][0][8 + j], l1 = sm.tx[px][1][8 + j];
        const float mx = fmaxf(m0, m1);
        const float f0 = m0 == -INFINITY ? 0.f : ex2(m0 - mx), f1 = m1 == -INFINITY ? 0.f : ex2(m1 - mx);
        const float lt = l0 * f0 + l1 * f1;
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        const float o = (oacc[j] * f0 + oacc[8 + j] * f1) * inv;
        const float lse_n = lt > 0.f ? (mx + __log2f(lt)) * 0.6931471805599453f : -INFINITY;
        const int rho = rho0 + j;
        const bool row_ok = rho < geo.rows_total;
        if (item.whole) {
          if (geo.q0 * g + rho < p.r_max * g) {
            const int node_o = geo.q0 + rho / g, hq_idx = geo.kvh * g + rho % g;
            reinterpret_cast<__nv_bfloat16 *>(p.out)[(((int64_t)geo.b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim +
                                                     col] = __float2bfloat16(row_ok ? o : 0.f);
            if (rank == 0 && ti == 0 && p.lse)
              p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
          }
        } else {
          const int64_t prow = (int64_t)item.slot * sp.rows_unit + sp.row_blk + j;
          sp.part_out[prow * kHeadDim + col] = row_ok ? o : 0.f;
          if (rank == 0 && ti == 0) sp.part_lse[prow] = row_ok ? lse_n : -INFINITY;
        }
      }
      if (bad_all && rank == 0 && tw == 0 && lane < sp.tail_rows && ((bad_all >> lane) & 1u))
        exact_row(sp, item, geo, g, sp.row_blk + lane);
    }
  } else if (warp == 3) {
    // ============ fused greedy-acceptance scan (otherwise idle warp) ============
    // Packed argmax keys (orderable max, lowest index on ties; argmax_keys_kernel
    // semantics, numcore.py:51-55) of logits rows r = cta, cta + grid, ...:
    // the TMA engine streams each row through a 3 x 8 KB shared ring while
    // the tensor pipe runs the attention, so the HBM-bound acceptance scan
    // uses the attention's spare memory bandwidth instead of its own launch.
#ifdef SDB_TRACE
    // trace builds: watch the tensor pipe of worker 0 (completion of S(n) via
    // s_full, of PV(n) via v_empty) from this otherwise idle warp; completion
    // order inside the first unit: S0 S1 S2 PV0 S3 PV1 S4 ...
    if (!p.fa_logits && worker == SDB_TRACE_WORKER && rank == 0 && lane == 0) {
      // (bounded by the worker's first active unit piece)
      ItemIter wit(sp, worker);
      Item wi;
      int wn = 0;
      while (wit.next(sp, wi)) {
        const ItemGeo wg_ = item_geo(sp, wi, g);
        if (wg_.active) {
          wn = wg_.n_tiles;
          break;
        }
      }
      const int lim = min(60, wn);
      for (int gi = 0; gi < 3 && gi < lim; ++gi) {
        mbar_wait(&sm.s_full[gi % 3], (gi / 3) & 1);
        TRACE(19, gi);
      }
      for (int n = 0; n + 3 < lim; ++n) {
        mbar_wait(&sm.v_empty[n % kStagesV], (n / kStagesV) & 1);
        TRACE(20, n);
        mbar_wait(&sm.s_full[(n + 3) % 3], ((n + 3) / 3) & 1);
        TRACE(19, n + 3);
      }
    }
#endif
    if (p.fa_logits) {
      griddep_wait();  // logits may come from the kernel launched just before
      const int nrows = p.batch * p.r_max;
      const int cta = blockIdx.x, ncta = gridDim.x;
      const int nchunk = (p.fa_vocab + kLgChunk - 1) / kLgChunk;
      // this CTA's rows cta, cta + ncta, ... (n_rows gated), streamed as one
      // continuous chunk sequence so the ring never drains at row boundaries
      auto valid_from = [&](int row) {
        for (; row < nrows; row += ncta) {
          const int b = row / p.r_max, r = row % p.r_max;
          if (r < min(p.n_rows[b], p.r_max)) return row;
        }
        return nrows;
      };
      int prow = valid_from(cta), pchunk = 0;  // producer cursor (lane 0)
      uint32_t pg = 0;
      auto issue_next = [&]() {
        if (prow >= nrows) return;
        const int st = pg % kLgStages;
        const int n = min(kLgChunk, p.fa_vocab - pchunk * kLgChunk);
        mbar_expect_tx(&sm.lg_full[st], (uint32_t)n * 4u);
        bulk_g2s(sm.lg[st], p.fa_logits + (int64_t)prow * p.fa_row_stride + (int64_t)pchunk * kLgChunk,
                 (uint32_t)n * 4u, &sm.lg_full[st]);
        ++pg;
        if (++pchunk == nchunk) {
          pchunk = 0;
          prow = valid_from(prow + ncta);
        }
      };
      if (lane == 0)
        for (int c = 0; c < kLgStages; ++c) issue_next();
      uint32_t g = 0;  // consumer chunk count (ring slot / parity)
      for (int row = valid_from(cta); row < nrows; row = valid_from(row + ncta)) {
        // hot loop: 3 instructions per 16 bytes (LDS.128 + two 3-input
        // max.NaN); the lane remembers only the chunk where its max first
        // appeared, and the element index is recovered once per row
        float bv = -INFINITY;
        int bc = 0;  // (an all -inf row still resolves to its first index)
        bool nan = false;
        for (int c = 0; c < nchunk; ++c, ++g) {
          const int st = g % kLgStages;
          mbar_wait(&sm.lg_full[st], (g / kLgStages) & 1);
          const int n4 = min(kLgChunk, p.fa_vocab - c * kLgChunk) >> 2;
          const float4 *v4 = reinterpret_cast<const float4 *>(sm.lg[st]);
          float cm = -INFINITY;
#pragma unroll 4
          for (int i = lane; i < n4; i += 32) {
            const float4 v = v4[i];
            cm = max_nan3(cm, max_nan3(v.x, v.y, v.z), v.w);
          }
          nan |= cm != cm;
          if (cm > bv) {  // strict: the earliest chunk wins ties
            bv = cm;
            bc = c;
          }
          __syncwarp();
          if (lane == 0) {
            fence_proxy_async_smem();  // the slot's generic reads precede the async-proxy refill
            issue_next();
          }
        }
        // row max, then the lowest index holding it (numpy argmax tie rule)
        float m = bv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        int idx = 0x7fffffff;
        if (bv == m) {
          const float *ch = p.fa_logits + (int64_t)row * p.fa_row_stride + (int64_t)bc * kLgChunk;
          const int n4 = min(kLgChunk, p.fa_vocab - bc * kLgChunk) >> 2;
          for (int i = lane; i < n4 && idx == 0x7fffffff; i += 32) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(ch) + i);
            const int e = v.x == m ? 0 : (v.y == m ? 1 : (v.z == m ? 2 : (v.w == m ? 3 : -1)));
            if (e >= 0) idx = bc * kLgChunk + 4 * i + e;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) idx = min(idx, __shfl_xor_sync(0xffffffffu, idx, o));
        const bool any_nan = __any_sync(0xffffffffu, nan);
        if (lane == 0) {
          p.fa_keys[row] = idx != 0x7fffffff ? argmax_key(m, (uint32_t)(p.fa_vocab_offset + idx)) : LLONG_MIN;
          if (any_nan && p.fa_err) atomicOr(p.fa_err, SDB_ERR_NAN);
        }
      }
    }
  }
  if (kRegsCtl) regs_inc<128>();  // back to the launch budget for the common tail (waits for the softmax warpgroups)
  } else {
    if (kRegsCtl) regs_inc<kRegsCtl ? kRegsSoftmax : 128>();
    // programmatic dependent launch: the mask words come from the kernel
    // launched just before (tree_build); everything else in flight above
    // (TMEM alloc, TMA of Q/K/V, first QK^T) already overlaps its tail
    griddep_wait();
    // ===================== softmax: 3 warpgroups, one row per thread ===========
    const int wg = (warp - 4) >> 2;
    const int lg = warp & 3;         // TMEM lane group (warp % 4 by hardware rule)
    const int i = (lg << 5) + lane;  // row within the CTA's 128 rows == TMEM lane
    const uint32_t lane_off = (uint32_t)(lg * 32) << 16;
    const int local = (int)rank * kTileM + i;  // row within the 256-row unit
    const int bar_in = 1 + wg * 4 + lg;                          // max handoff into this warpgroup
    const int bar_out = 1 + ((wg + 1) % kSoftmaxWG) * 4 + lg;   // ... and out of it
    const bool tr = rank == 0 && lg == 0 && lane == 0;
    uint32_t g_item = 0, g_unit = 0;
    ItemIter iter(sp, worker);
    Item item;
    while (iter.next(sp, item)) {
      const ItemGeo geo = item_geo(sp, item, g);
      if (!geo.active) {
        if (wg == 0) inactive_row(sp, item, geo, g, local);
        continue;
      }
      const int rho = geo.row0 + local;
      const bool row_ok = rho < geo.rows_total;
      const int node = min(geo.q0 + rho / g, max(geo.n_nodes - 1, 0));
      const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
      const int N = geo.n_tiles;
      float m_w = -INFINITY, l_w = 0.f, m_fix = -INFINITY;
      bool seen = false, bad = false;
      for (int n = (int)((wg + 3 - g_item % 3) % 3); n < N; n += 3) {
        const uint32_t gi = g_item + n;
        const int slot = wg;
        const bool pref = n < geo.n_pref;
        const int key0 = pref ? geo.k0 + (geo.pa + n) * kTileN : (geo.sa + n - geo.n_pref) * kTileN;
        const int kvalid = pref ? geo.C - key0 : geo.n_nodes - key0;
        const bool full = pref && kvalid >= kTileN;
        if (tr) TRACE(3, gi);
        mbar_wait(&sm.s_full[slot], (gi / 3) & 1);
        tc_fence_after();
        if (tr) TRACE(4, gi);
        const uint32_t t_s = tmem + lane_off + kSBase + slot * 128;
        // a warp whose 32 rows are all padding (the short last row block of
        // R = 65: 520 rows per KV head) skips the softmax: its P rows only
        // feed O rows that are never stored.  It still waits for S (one phase
        // per item) and arrives on p_full, and its chain partners (same lane
        // group, other warpgroups) skip the hand-off alike.
        const bool pad_warp = geo.row0 + (int)rank * kTileM + lg * 32 >= geo.rows_total;
        if (!pad_warp) {
        uint32_t vm[4] = {~0u, ~0u, ~0u, ~0u};
        if (!full) {
#pragma unroll
          for (int c = 0; c < 4; ++c) vm[c] = vis_word(pref, kvalid, mrow, key0, p.n_words, row_ok, 32 * c);
        }
        if (kFixRef && n > 0) {
          // fixed reference: no max pass; the first item of this warpgroup
          // in the unit takes the reference from the chain
          if (n <= 2) {
            asm volatile("bar.sync %0, 64;" ::"r"(bar_in) : "memory");
            m_fix = sm.mref[(gi + 2) % 3][i];
            if (n == 1 && N > 2) {
              sm.mref[slot][i] = m_fix;
              asm volatile("bar.arrive %0, 64;" ::"r"(bar_out) : "memory");
            }
          }
          if (tr) TRACE(6, gi);
          if (tr) TRACE(7, gi);
        } else {
          // pass 1: row max over four 32-column chunks, each load overlapped
          // with the max of the previous chunk
          uint32_t r[32], r2[32];
          SDB_TMEM_LD32(t_s + 0, r2);
          SDB_TMEM_WAIT_LD_REGS(r2);
          if (!kFixRef) SDB_TMEM_LD32(t_s + 32, r);
          if (!full) apply_mask32(r2, vm[0]);
          float mx = max32(r2);
          if (kFixRef) {
            // fixed reference: the row max of the first 32 keys of the
            // piece's first tile is enough (anything above it by less than
            // ~89 log2 units stays exact), so the hand-off leaves right away
            mx *= sl2;
          } else {
          SDB_TMEM_WAIT_LD_REGS(r);
          SDB_TMEM_LD32(t_s + 64, r2);
          if (!full) apply_mask32(r, vm[1]);
          mx = fmaxf(mx, max32(r));
          SDB_TMEM_WAIT_LD_REGS(r2);
          SDB_TMEM_LD32(t_s + 96, r);
          if (!full) apply_mask32(r2, vm[2]);
          mx = fmaxf(mx, max32(r2));
          SDB_TMEM_WAIT_LD_REGS(r);
          if (!full) apply_mask32(r, vm[3]);
          mx = fmaxf(mx, max32(r));
          mx *= sl2;
          }
          // reference max chain (lazy: moves only when the max grows by > 2^8);
          // with the fixed reference only the unit's first item gets here and
          // hands its max to the second
          float m_prev = -INFINITY;
          if (!kFixRef && n > 0) {
            asm volatile("bar.sync %0, 64;" ::"r"(bar_in) : "memory");
            m_prev = sm.mref[(gi + 2) % 3][i];
          }
          if (tr) TRACE(6, gi);
          if (tr) TRACE(7, gi);
          const float m_ref = (n == 0 || mx > m_prev + kRescaleThreshold) ? mx : m_prev;
          m_fix = m_ref;
          if (n + 1 < N) {  // hand-offs pair up within the unit
            sm.mref[slot][i] = m_ref;
            asm volatile("bar.arrive %0, 64;" ::"r"(bar_out) : "memory");
          }
          const bool resc = !kFixRef && n > 0 && m_ref != m_prev;
          if (!kFixRef && __any_sync(0xffffffffu, resc)) {
            // O holds items < n relative to m_prev: wait for PV(n - 1), rescale in place
            const float corr = resc ? ex2(m_prev - m_ref) : 1.f;
            mbar_wait(&sm.o_done[(gi + 2) % 3], ((gi - 1) / 3) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              SDB_TMEM_LD32(tmem + lane_off + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
              SDB_TMEM_ST32(tmem + lane_off + c * 32, o);
            }
          }
        }
        if (!seen) {
          m_w = m_fix;
          seen = true;
        } else if (m_fix != m_w) {
          l_w *= ex2(m_w - m_fix);
          m_w = m_fix;
        }
        {
          // exp pass: P of chunk c (keys 32c .. 32c+31) packed into columns
          // [32c, 32c + 16) of the slot -- inside the chunk's own, already
          // loaded S columns; each load overlapped with the previous
          // chunk's exps.  The row max of the item is tracked on the side:
          // with the fixed reference, a score ~89 log2 units above m_ref
          // (or a visible key in a row whose reference is -inf) flags the
          // row for the exact recompute.
          const float neg_mu = (m_fix == -INFINITY) ? 0.f : -m_fix;
          const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_mu, neg_mu);
          uint32_t r[32], r2[32];
          SDB_TMEM_LD32(t_s + 0, r2);
          SDB_TMEM_WAIT_LD_REGS(r2);
          SDB_TMEM_LD32(t_s + 32, r);
          if (!full) apply_mask32(r2, vm[0]);
          float rs = exp_pack32<EMU8>(r2, sc2, nm2);
          SDB_TMEM_ST16(t_s + 0, r2);
          SDB_TMEM_WAIT_LD_REGS(r);
          SDB_TMEM_LD32(t_s + 64, r2);
          if (!full) apply_mask32(r, vm[1]);
          rs += exp_pack32<EMU8>(r, sc2, nm2);
          SDB_TMEM_ST16(t_s + 32, r);
          SDB_TMEM_WAIT_LD_REGS(r2);
          SDB_TMEM_LD32(t_s + 96, r);
          if (!full) apply_mask32(r2, vm[2]);
          rs += exp_pack32<EMU8>(r2, sc2, nm2);
          SDB_TMEM_ST16(t_s + 64, r2);
          SDB_TMEM_WAIT_LD_REGS(r);
          if (!full) apply_mask32(r, vm[3]);
          rs += exp_pack32<EMU8>(r, sc2, nm2);
          SDB_TMEM_ST16(t_s + 96, r);
          l_w += rs;
          // a score ~89 log2 units above the reference shows in the item's sum
          // (an exp2 that overflowed is +inf; 128 terms cannot reach 2^96
          // otherwise unless one of them is within 7 of the limit), and a
          // visible key in a row whose reference is -inf gives a positive sum
          if (kFixRef) bad |= rs > kOverflowSum || (m_fix == -INFINITY && rs > 0.f);
        }
        }  // !pad_warp
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0)
            mbar_arrive(&sm.p_full[slot]);
          else
            mbar_arrive_leader(&sm.p_full[slot]);
        }
        if (tr) TRACE(5, gi);
      }
      // ---- unit end: combine the partial row sums, normalise, store ----
      sm.lsum[wg][i] = l_w;
      sm.msum[wg][i] = seen ? m_w : -INFINITY;
      if (bad) sm.bad[i] = 1u;
      // unit-end barrier of the softmax warps, OR-reducing "a row needs the exact recompute"
      uint32_t any_bad;
      asm volatile(
          "{\n.reg .pred pi, po;\nsetp.ne.u32 pi, %1, 0;\nbar.red.or.pred po, %2, %3, pi;\n"
          "selp.u32 %0, 1, 0, po;\n}"
          : "=r"(any_bad)
          : "r"(bad ? 1u : 0u), "r"(kBarUnit), "r"(kSoftmaxWG * 128)
          : "memory");
      // the final reference is the largest one any warpgroup used (the
      // running max only grows; with the fixed reference they are all equal)
      float m_fin = -INFINITY;
#pragma unroll
      for (int w = 0; w < kSoftmaxWG; ++w) m_fin = fmaxf(m_fin, sm.msum[w][i]);
      float l_full = 0.f;
#pragma unroll
      for (int w = 0; w < kSoftmaxWG; ++w) {
        const float mw = sm.msum[w][i];
        if (mw != -INFINITY) l_full += sm.lsum[w][i] * ex2(mw - m_fin);
      }
      bool row_bad = false;
      if (any_bad && wg == 0) {
        row_bad = sm.bad[i] != 0u;
        sm.bad[i] = 0u;
      }
      bad = false;
      asm volatile("bar.sync %0, %1;" ::"r"(kBarUnit), "r"(kSoftmaxWG * 128) : "memory");
      mbar_wait(&sm.o_last, g_unit & 1);
      ++g_unit;
      tc_fence_after();
      for (int c = wg; c < 8; c += kSoftmaxWG)
        epilogue_chunk(sp, item, geo, g, local, c, tmem + lane_off, m_fin, l_full);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(&sm.o_free);
        else
          mbar_arrive_leader(&sm.o_free);
      }
      if (any_bad) {
        // every warpgroup's epilogue stores are done; overwrite the flagged rows exactly
        asm volatile("bar.sync %0, %1;" ::"r"(kBarUnit), "r"(kSoftmaxWG * 128) : "memory");
        if (row_bad) exact_row(sp, item, geo, g, local);
      }
      if (tr && wg == 0) TRACE(10, g_item);
      g_item += N;
    }
    if (kRegsCtl) regs_dec<128>();
  }
  if (threadIdx.x == 0 && rank == 0) TRACE(11, 0);
  tc_fence_before();
  __syncwarp();
  cluster_sync();  // the pair's MMAs, remote arrivals and TMEM reads are all done
  if (threadIdx.x == 0 && rank == 0) TRACE(12, 0);
  if (threadIdx.x == 0 && rank == 0) TRACE_G(14);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int launch_2cta(const CUtensorMap &mq, const CUtensorMap &mqt, const CUtensorMap &mk, const CUtensorMap &mv,
                const CUtensorMap &mtk, const CUtensorMap &mtv, const Sm100Params &sp, int emu, cudaStream_t stream) {
  dim3 grid(sp.n_workers * 2);
  const size_t smem = sizeof(Smem2) + 1024;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = sp.p.pdl ? 1 : 0;
#define SDB_LAUNCH_PAIR(EMU8)                                                                                      \
  do {                                                                                                             \
    cudaFuncSetAttribute(tree_attn_tcgen05_pair_kernel<EMU8>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                         (int)smem);                                                                               \
    cudaLaunchKernelEx(&cfg, tree_attn_tcgen05_pair_kernel<EMU8>, mq, mqt, mk, mv, mtk, mtv, sp);                      \
  } while (0)
  // emu: pairs of every 8 whose exp2 runs on the FMA pipe
  switch (emu) {
    case 0: SDB_LAUNCH_PAIR(0); break;
    case 2: SDB_LAUNCH_PAIR(2); break;
    case 3: SDB_LAUNCH_PAIR(3); break;
    case 4: SDB_LAUNCH_PAIR(4); break;
    default: SDB_LAUNCH_PAIR(1); break;
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
