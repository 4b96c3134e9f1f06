// Shared device helpers of the sm_100a tree-verify attention kernels
// (1-CTA attn_sm100.cu and 2-CTA attn_sm100_2cta.cu): mbarrier / TMA /
// tcgen05 wrappers, packed-fp32 math, the stream-K work decomposition and the
// per-tile softmax.
#pragma once

#include <cuda.h>

#include "attn_internal.cuh"

namespace sdb {
namespace sm100 {

constexpr int kTileN = 128;     // keys per KV tile
constexpr int kTileM = 128;     // query rows per tile
constexpr int kHeadDim = 128;   // d
constexpr int kChunkBytes = kTileM * 128;  // 128 rows x 64 bf16 (one SW128 column chunk)
constexpr int kTileBytes = 2 * kChunkBytes;  // 128 x 128 bf16
constexpr float kRescaleThreshold = 8.0f;   // log2 units (factor 256)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// One lane of a converged warp (elect.sync): the issuing lane for tcgen05.mma.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, %1;\n@px mov.s32 %0, 1;\n}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ---- tcgen05 --------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#define SDB_TMEM_LD32(taddr, r)                                                                                    \
  asm volatile(                                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                               \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),         \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
      : "r"(taddr))

#define SDB_TMEM_LD16(taddr, r)                                                                                    \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),         \
                 "=r"(r[15])                                                                                      \
               : "r"(taddr))

#define SDB_TMEM_ST32(taddr, r)                                                                                    \
  asm volatile(                                                                                                    \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                                \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),          \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),  \
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), \
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))

#define SDB_TMEM_ST16(taddr, r)                                                                                    \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16};" ::"r"(taddr),                                                                               \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), \
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))

// tcgen05.wait::ld that also "redefines" the 32 destination registers of
// the loads it waits for, so the compiler cannot hoist their uses above it
// (the loads complete asynchronously; a plain wait carries no register
// dependence).  Used when a load is overlapped with compute on other data.
#define SDB_TMEM_WAIT_LD_REGS(r)                                                                                  \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                    \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),  \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),         \
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),       \
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),       \
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory")

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// 1-D bulk copy global -> this CTA's shared memory (TMA engine), completion
// bytes on an mbarrier of this CTA
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 3-input max propagating NaN (sm_100 FMNMX3)
__device__ __forceinline__ float max_nan3(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// wait for the upstream kernel's completion + memory flush (no-op when the
// kernel was launched without the programmatic-serialization attribute)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Warp-specialised register budgets (whole warpgroup, warp-uniform): the
// producer / MMA warpgroup hands registers to the softmax warpgroups.
template <int N>
__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
// let the downstream PDL kernel start launching (its CTAs run their
// prologue until their own griddep_wait)
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- packed fp32x2 math (FFMA2 / FADD2) and 3-input max (FMNMX3), sm_100 ----
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fadd2_rm(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// exp2 of two values on the FMA pipe (offloads the MUFU): 2^x = 2^n * p(f),
// n = round(x), f = x - n in [-1/2, 1/2], p a cubic fit of 2^f (max relative
// error 7.7e-5, far below the bf16 rounding of P).  x is clamped at -126 so
// the exponent add stays in range (2^-126 underflows to ~0 in P anyway).
// 10 instructions per pair: 2 FMNMX, 3 FADD2, 3 FFMA2, 2 IMAD.
__device__ __forceinline__ void ex2_emu2(float x, float y, float &ox, float &oy) {
  constexpr float kRound = 12582912.0f;  // 2^23 + 2^22: x + kRound rounds x to an integer
  const uint64_t xy = f2pack(fmaxf(x, -126.f), fmaxf(y, -126.f));
  const uint64_t rr = fadd2(xy, f2pack(kRound, kRound));  // n in the low mantissa bits
  const uint64_t f = fsub2(xy, fadd2(rr, f2pack(-kRound, -kRound)));
  uint64_t pp = ffma2(f2pack(0.05508868f, 0.05508868f), f, f2pack(0.24260405f, 0.24260405f));
  pp = ffma2(pp, f, f2pack(0.69327624f, 0.69327624f));
  pp = ffma2(pp, f, f2pack(0.99992894f, 0.99992894f));
  float px, py, rx, ry;
  f2unpack(pp, px, py);
  f2unpack(rr, rx, ry);
  ox = __uint_as_float(__float_as_uint(px) + (__float_as_uint(rx) << 23));
  oy = __uint_as_float(__float_as_uint(py) + (__float_as_uint(ry) << 23));
}

// Shared-memory matrix descriptor (SM100 UMMA, version 1, 128-byte swizzle).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, bf16 x bf16 -> fp32, M = 128, N = 128.
__host__ __device__ constexpr uint32_t make_idesc(bool b_mn_major) {
  return (1u << 4)                      // D format f32
         | (1u << 7)                    // A bf16
         | (1u << 10)                   // B bf16
         | ((b_mn_major ? 1u : 0u) << 16)  // B major
         | ((uint32_t)(kTileN >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);
}

constexpr int kMaxSplit = 192;  // split units listed for the fix-up grid

struct Sm100Params {
  TreeAttnParams p;
  int cta_group;   // 1: one CTA per unit (M = 128 MMAs); 2: CTA pair (M = 256, cta_group::2)
  int nt;          // query tiles per CTA (ping-pong depth)
  int m_blocks;    // row blocks (rows_unit query rows) per (b, kvh)
  int units;       // m_blocks * batch * hkv
  int w_pref;      // nominal prefix tiles per unit: ceil(max_ctx / 128)
  int w_unit;      // nominal tiles per unit: w_pref + ceil(r_max / 128)
  int n_workers;   // stream-K workers (CTAs, or CTA pairs)
  int rows_unit;   // partial-output rows per unit: row_blk (+ 8 fused tail rows)
  int row_blk;     // query rows per row block: nt * 128 * cta_group
  int tail_rows;   // pair kernel: live rows (1..8) past the last full row block, fused into its units (0: none)
  int64_t total;   // units * w_unit
  float *part_out; // [n_workers * 2][rows_unit][128] partial outputs of split units
  float *part_lse; // [n_workers * 2][rows_unit]
  int64_t *seg;    // [n_workers + 1] segment starts, written by the main kernel for the fix-up
  int n_split;     // split units to merge (-1: more than kMaxSplit, the fix-up scans every boundary)
  int split_k[kMaxSplit];  // per split unit: its first interior worker boundary k
};

__host__ __device__ __forceinline__ int64_t seg_begin(const Sm100Params &sp, int k) {
  return sp.total * k / sp.n_workers;
}

// One contiguous piece of a unit's nominal tile range owned by a worker.
struct Item {
  int unit, t0, t1, slot;
  bool whole;
};

// Items of worker k: walk [seg_begin(k), seg_begin(k+1)).
struct ItemIter {
  int64_t cur, end;
  int idx, k;
  __device__ ItemIter(const Sm100Params &sp, int k_) : idx(0), k(k_) {
    cur = seg_begin(sp, k_);
    end = seg_begin(sp, k_ + 1);
  }
  __device__ bool next(const Sm100Params &sp, Item &it) {
    if (cur >= end) return false;
    it.unit = (int)(cur / sp.w_unit);
    it.t0 = (int)(cur % sp.w_unit);
    it.t1 = (int)min((int64_t)sp.w_unit, it.t0 + (end - cur));
    it.whole = it.t0 == 0 && it.t1 == sp.w_unit;
    cur += it.t1 - it.t0;
    it.slot = k * 2 + (idx == 0 ? 0 : 1);
    ++idx;
    return true;
  }
};

// Per-item geometry: which (b, kvh, rows) and which actual KV tiles.
struct ItemGeo {
  int b, kvh, row0, n_nodes, rows_total, C;
  int q0;  // first query node; query row rho is node q0 + rho / g
  int k0;  // first prefix key (iRoPE local chunk start; 0 without chunking)
  int pa, n_pref, sa, n_suf, n_tiles;
  bool active;
};

__device__ __forceinline__ ItemGeo item_geo(const Sm100Params &sp, const Item &it, int g) {
  const TreeAttnParams &p = sp.p;
  ItemGeo o;
  // unit = mblk * (B * Hkv) + b * Hkv + kvh: the row blocks of one KV head run
  // on workers ~n_workers / m_blocks apart at the same time, so its K/V stream
  // is read from HBM once and served from L2 to the other row blocks.
  const int bh = p.batch * p.hkv;
  o.b = (it.unit % bh) / p.hkv;
  o.kvh = it.unit % p.hkv;
  o.row0 = (it.unit / bh) * sp.row_blk;
  o.n_nodes = min(p.n_rows[o.b], p.r_max);
  o.q0 = q_first(p, o.b, o.n_nodes);
  o.rows_total = (o.n_nodes - o.q0) * g;
  o.C = p.ctx_len[o.b];
  o.k0 = prefix_start(p, o.C);
  const int pb = (o.C - o.k0 + kTileN - 1) / kTileN;
  const int sb = (o.n_nodes + kTileN - 1) / kTileN;
  o.pa = min(it.t0, pb);
  const int pe = min(min(it.t1, sp.w_pref), pb);
  o.n_pref = max(0, pe - o.pa);
  o.sa = min(max(it.t0 - sp.w_pref, 0), sb);
  const int se = min(max(it.t1 - sp.w_pref, 0), sb);
  o.n_suf = max(0, se - o.sa);
  o.n_tiles = o.n_pref + o.n_suf;
  o.active = o.n_tiles > 0 && o.row0 < o.rows_total;
  return o;
}

// ---------------------------------------------------------------------------
// Softmax of one S tile row held by this thread (TMEM lane), P written back
// over S.  Updates the running reference max m (log2 units) and sum l.
// On return P is stored (tcgen05.wait::st done) and tcgen05.fence::before
// issued; the caller signals the MMA issuer.
// ---------------------------------------------------------------------------
template <int EMU>
__device__ __forceinline__ void softmax_tile(uint32_t t_s, uint32_t t_o, float sl2, bool first, bool pref,
                                             int kvalid, const uint32_t *mrow, int key0, int n_words, bool row_ok,
                                             float &m, float &l) {
  const bool full = pref && kvalid >= kTileN;
  // visibility bits of the 128 columns: prefix -> keys < ctx; suffix ->
  // ancestor-or-self bits of this row's node (tree_build mask words)
  uint32_t vm[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int lim = kvalid - 32 * w;
    const uint32_t low = lim >= 32 ? 0xffffffffu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
    uint32_t bits = 0xffffffffu;
    if (!pref) {
      const int wi = (key0 >> 5) + w;
      bits = (wi < n_words && row_ok) ? mrow[wi] : 0u;
    }
    vm[w] = bits & low;
  }
  uint32_t r[128];
  SDB_TMEM_LD32(t_s + 0, (r + 0));
  SDB_TMEM_LD32(t_s + 32, (r + 32));
  SDB_TMEM_LD32(t_s + 64, (r + 64));
  SDB_TMEM_LD32(t_s + 96, (r + 96));
  tmem_wait_ld();
  if (!full) {
#pragma unroll
    for (int e = 0; e < 128; ++e)
      if (!((vm[e >> 5] >> (e & 31)) & 1u)) r[e] = 0xff800000u;
  }
  // row max on raw scores (scale > 0): 4 chains of 3-input max
  float c0 = fmaxf(__uint_as_float(r[0]), __uint_as_float(r[1]));
  float c1 = fmaxf(__uint_as_float(r[2]), __uint_as_float(r[3]));
  float c2 = fmaxf(__uint_as_float(r[4]), __uint_as_float(r[5]));
  float c3 = fmaxf(__uint_as_float(r[6]), __uint_as_float(r[7]));
#pragma unroll
  for (int e = 8; e < 128; e += 8) {
    c0 = fmax3(c0, __uint_as_float(r[e + 0]), __uint_as_float(r[e + 1]));
    c1 = fmax3(c1, __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
    c2 = fmax3(c2, __uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]));
    c3 = fmax3(c3, __uint_as_float(r[e + 6]), __uint_as_float(r[e + 7]));
  }
  const float mx = fmax3(fmaxf(c0, c1), c2, c3) * sl2;
  // lazy rescale: move the reference max only when it grows by > 2^8; the
  // O / l correction is applied after P is written (frees the S registers)
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
  // P = exp2(s * scale_log2 - m) (FFMA2); EMU of every 4 pairs on the FMA
  // pipe; row sum on FADD2; packed bf16 in place into r[0..63]
  const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_mu, neg_mu);
  uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int e = 0; e < 64; ++e) {
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
  f2unpack(acc2[0], s0, s1);
  f2unpack(acc2[1], s2, s3);
  f2unpack(acc2[2], s4, s5);
  f2unpack(acc2[3], s6, s7);
  l = l * corr + (((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)));
  SDB_TMEM_ST32(t_s + 0, (r + 0));
  SDB_TMEM_ST32(t_s + 32, (r + 32));
  if (rescale) {
    // the previous PV has completed: this tile's S was committed after it
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      SDB_TMEM_LD32(t_o + c * 32, o);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
      SDB_TMEM_ST32(t_o + c * 32, o);
    }
  }
  tmem_wait_st();
  tc_fence_before();
}

// Half-row variant: two warps share a TMEM lane group, each owning 64 of the
// 128 columns of a row (more softmax warps per SMSP to hide latency).  The
// partner's partial row max is exchanged through shared memory under a
// 64-thread named barrier; the row sum stays partial (combined in the
// epilogue).  P for columns [64h, 64h+64) lands in packed columns
// [32h, 32h+32) -- both halves have loaded their S before the exchange.
template <int EMU>
__device__ __forceinline__ void softmax_half_tile(uint32_t t_s, uint32_t t_o, int half, float sl2, bool first,
                                                  bool pref, int kvalid, const uint32_t *mrow, int key0, int n_words,
                                                  bool row_ok, float *xch, int xch_row, int bar_id, float &m,
                                                  float &l) {
  const bool full = pref && kvalid >= kTileN;
  uint32_t vm[2];
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const int lim = kvalid - 32 * (2 * half + w);
    const uint32_t low = lim >= 32 ? 0xffffffffu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
    uint32_t bits = 0xffffffffu;
    if (!pref) {
      const int wi = (key0 >> 5) + 2 * half + w;
      bits = (wi < n_words && row_ok) ? mrow[wi] : 0u;
    }
    vm[w] = bits & low;
  }
  uint32_t r[64];
  SDB_TMEM_LD32(t_s + 64 * half, (r + 0));
  SDB_TMEM_LD32(t_s + 64 * half + 32, (r + 32));
  tmem_wait_ld();
  if (!full) {
#pragma unroll
    for (int e = 0; e < 64; ++e)
      if (!((vm[e >> 5] >> (e & 31)) & 1u)) r[e] = 0xff800000u;
  }
  float c0 = fmaxf(__uint_as_float(r[0]), __uint_as_float(r[1]));
  float c1 = fmaxf(__uint_as_float(r[2]), __uint_as_float(r[3]));
  float c2 = fmaxf(__uint_as_float(r[4]), __uint_as_float(r[5]));
  float c3 = fmaxf(__uint_as_float(r[6]), __uint_as_float(r[7]));
#pragma unroll
  for (int e = 8; e < 64; e += 8) {
    c0 = fmax3(c0, __uint_as_float(r[e + 0]), __uint_as_float(r[e + 1]));
    c1 = fmax3(c1, __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
    c2 = fmax3(c2, __uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]));
    c3 = fmax3(c3, __uint_as_float(r[e + 6]), __uint_as_float(r[e + 7]));
  }
  const float mh = fmax3(fmaxf(c0, c1), c2, c3);
  xch[half * 128 + xch_row] = mh;
  asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
  const float mx = fmaxf(mh, xch[(half ^ 1) * 128 + xch_row]) * sl2;
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
  for (int e = 0; e < 32; ++e) {
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
  f2unpack(acc2[0], s0, s1);
  f2unpack(acc2[1], s2, s3);
  f2unpack(acc2[2], s4, s5);
  f2unpack(acc2[3], s6, s7);
  l = l * corr + (((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)));
  SDB_TMEM_ST32(t_s + 32 * half, (r + 0));
  if (rescale) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      SDB_TMEM_LD32(t_o + 64 * half + c * 32, o);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
      SDB_TMEM_ST32(t_o + 64 * half + c * 32, o);
    }
  }
  tmem_wait_st();
  tc_fence_before();
}

// Epilogue for a half row: this thread's 64 O columns, with the row sum
// combined from both halves (l_full).
__device__ __forceinline__ void epilogue_half_row(const Sm100Params &sp, const Item &item, const ItemGeo &geo, int g,
                                                  int local, int half, uint32_t t_o, float m, float l_full) {
  const TreeAttnParams &p = sp.p;
  const int rho = geo.row0 + local;
  const bool row_ok = rho < geo.rows_total;
  const bool in_range = geo.q0 * g + rho < p.r_max * g;
  const int node_o = geo.q0 + rho / g;
  const int hq_idx = geo.kvh * g + (rho % g);
  const float inv = l_full > 0.f ? 1.f / l_full : 0.f;
  const float lse_n = l_full > 0.f ? (m + __log2f(l_full)) * 0.6931471805599453f : -INFINITY;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    SDB_TMEM_LD32(t_o + 64 * half + c * 32, r);
    tmem_wait_ld();
    const int col0 = 64 * half + c * 32;
    if (item.whole) {
      if (!in_range) continue;
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
    } else {
      float *o = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim + col0;
#pragma unroll
      for (int e = 0; e < 32; e += 4)
        *reinterpret_cast<float4 *>(o + e) =
            make_float4(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv,
                        __uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
    }
  }
  if (half == 0) {
    if (item.whole) {
      if (in_range && p.lse)
        p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
    } else {
      sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = row_ok ? lse_n : -INFINITY;
    }
  }
}

// ---- fixed-reference softmax pieces (pair kernel; 1-CTA kernel with one query tile) ----
constexpr float kOverflowSum = 0x1p96f;  // an item's row sum above this flags the row (2^89 x 128 terms)

// 32 S values of one row (fp32 bits in r[0..31]) -> P = exp2(s * sl2 - m),
// packed bf16 into r[0..15]; returns the sum of the 32 probabilities.
// EMU8 of every 8 pairs run a cubic exp2 on the FMA pipe (offloads MUFU).
template <int EMU8>
__device__ __forceinline__ float exp_pack32(uint32_t *r, uint64_t sc2, uint64_t nm2) {
  uint64_t acc2[2] = {0ull, 0ull};
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    float x0, x1, p0, p1;
    f2unpack(ffma2(f2pack(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), sc2, nm2), x0, x1);
    if ((e & 7) < EMU8) {
      ex2_emu2(x0, x1, p0, p1);
    } else {
      p0 = ex2(x0);
      p1 = ex2(x1);
    }
    acc2[e & 1] = fadd2(acc2[e & 1], f2pack(p0, p1));
    r[e] = pack_bf16(p0, p1);
  }
  float s0, s1;
  f2unpack(fadd2(acc2[0], acc2[1]), s0, s1);
  return s0 + s1;
}

// Visibility bits of the 32 columns [c0, c0 + 32) of a key tile for this
// row: prefix tiles -> keys < ctx; the suffix (tree) tile -> ancestor-or-self.
__device__ __forceinline__ uint32_t vis_word(bool pref, int kvalid, const uint32_t *mrow, int key0, int n_words,
                                             bool row_ok, int c0) {
  const int lim = kvalid - c0;
  const uint32_t low = lim >= 32 ? 0xffffffffu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
  uint32_t bits = 0xffffffffu;
  if (!pref) {
    const int wi = (key0 + c0) >> 5;
    bits = (wi < n_words && row_ok) ? mrow[wi] : 0u;
  }
  return bits & low;
}
__device__ __forceinline__ void apply_mask32(uint32_t *r, uint32_t w) {
#pragma unroll
  for (int e = 0; e < 32; ++e)
    if (!((w >> e) & 1u)) r[e] = 0xff800000u;
}
__device__ __forceinline__ float max32(const uint32_t *r) {
  float c0 = fmax3(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]));
  float c1 = fmax3(__uint_as_float(r[3]), __uint_as_float(r[4]), __uint_as_float(r[5]));
#pragma unroll
  for (int e = 6; e < 30; e += 4) {
    c0 = fmax3(c0, __uint_as_float(r[e + 0]), __uint_as_float(r[e + 1]));
    c1 = fmax3(c1, __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
  }
  return fmax3(c0, c1, fmaxf(__uint_as_float(r[30]), __uint_as_float(r[31])));
}

// Normalise this thread's O row (TMEM) and store it: final bf16 output +
// LSE for a whole unit, fp32 partial for a split one.
__device__ __forceinline__ void epilogue_row(const Sm100Params &sp, const Item &item, const ItemGeo &geo, int g,
                                             int local, uint32_t t_o, float m, float l) {
  const TreeAttnParams &p = sp.p;
  const int rho = geo.row0 + local;
  const bool row_ok = rho < geo.rows_total;
  const bool in_range = geo.q0 * g + rho < p.r_max * g;
  const int node_o = geo.q0 + rho / g;
  const int hq_idx = geo.kvh * g + (rho % g);
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const float lse_n = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    SDB_TMEM_LD32(t_o + c * 32, r);
    tmem_wait_ld();
    if (item.whole) {
      if (!in_range) continue;
      __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                         (((int64_t)geo.b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim + c * 32;
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
    } else {
      float *o = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim + c * 32;
#pragma unroll
      for (int e = 0; e < 32; e += 4)
        *reinterpret_cast<float4 *>(o + e) =
            make_float4(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv,
                        __uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
    }
  }
  if (item.whole) {
    if (in_range && p.lse)
      p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
  } else {
    sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = row_ok ? lse_n : -INFINITY;
  }
}

// Zeros / -inf for a row of an inactive item (padding rows of a whole unit, or
// every row of an empty split piece).
__device__ __forceinline__ void inactive_row(const Sm100Params &sp, const Item &item, const ItemGeo &geo, int g,
                                             int local) {
  const TreeAttnParams &p = sp.p;
  const int rho = geo.row0 + local;
  if (!item.whole) {
    float *o = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim;
    for (int c = 0; c < kHeadDim; c += 4) *reinterpret_cast<float4 *>(o + c) = make_float4(0, 0, 0, 0);
    sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = -INFINITY;
  } else if (geo.q0 * g + rho < p.r_max * g) {
    const int node_o = geo.q0 + rho / g, hq_idx = geo.kvh * g + (rho % g);
    __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                       (((int64_t)geo.b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim;
    for (int c = 0; c < kHeadDim; c += 8) *reinterpret_cast<uint4 *>(o + c) = make_uint4(0, 0, 0, 0);
    if (p.lse) p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = -INFINITY;
  }
}

// Exact fallback for one query row of an item, on the CUDA cores: two fp32
// passes (max, then exp-sum and P.V) over exactly the keys the item covers
// (its prefix tiles through the block table, its tree tiles under the
// ancestor mask), writing what the epilogue writes (bf16 out + LSE of a whole
// unit, the fp32 partial of a split one).  Runs only when the fixed-reference
// softmax saw a score far above its reference (kOverflowLog2) -- never for
// attention scores within ~60 nats of the piece's first tile.
static __device__ __noinline__ void exact_row(const Sm100Params &sp, const Item &item, const ItemGeo &geo, int g,
                                       int local) {
  const TreeAttnParams &p = sp.p;
  const int rho = geo.row0 + local;
  if (rho >= geo.rows_total || geo.q0 * g + rho >= p.r_max * g) return;  // padding rows keep the epilogue's zeros
  const int node = geo.q0 + rho / g;
  const int hq_idx = geo.kvh * g + (rho % g);
  const __nv_bfloat16 *q = reinterpret_cast<const __nv_bfloat16 *>(p.q) +
                           (((int64_t)geo.b * p.r_max + node) * p.hq + hq_idx) * kHeadDim;
  const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
  const int32_t *bt = p.block_table + (int64_t)geo.b * p.max_blocks;
  const int kp0 = geo.k0 + geo.pa * kTileN, kp1 = min(geo.k0 + (geo.pa + geo.n_pref) * kTileN, geo.C);
  const int ks0 = geo.sa * kTileN, ks1 = min((geo.sa + geo.n_suf) * kTileN, geo.n_nodes);
  auto key_row = [&](int j, bool pref, bool v) -> const __nv_bfloat16 * {
    if (pref) {
      const int page = bt[j / p.block_size];
      const int64_t off = (((int64_t)page * p.hkv + geo.kvh) * p.block_size + j % p.block_size) * kHeadDim;
      return reinterpret_cast<const __nv_bfloat16 *>(v ? p.v_cache : p.k_cache) + off;
    }
    return reinterpret_cast<const __nv_bfloat16 *>(v ? p.tree_v : p.tree_k) +
           (((int64_t)geo.b * p.r_max + j) * p.hkv + geo.kvh) * kHeadDim;
  };
  auto score = [&](const __nv_bfloat16 *k) {
    float s = 0.f;
#pragma unroll 8
    for (int e = 0; e < kHeadDim; ++e) s += __bfloat162float(q[e]) * __bfloat162float(k[e]);
    return s * p.scale;
  };
  auto visible = [&](int j) { return j < geo.n_nodes && ((mrow[j >> 5] >> (j & 31)) & 1u); };
  float m = -INFINITY;
  for (int j = kp0; j < kp1; ++j) m = fmaxf(m, score(key_row(j, true, false)));
  for (int j = ks0; j < ks1; ++j)
    if (visible(j)) m = fmaxf(m, score(key_row(j, false, false)));
  // P.V in four 32-column chunks (scores recomputed per chunk: a small
  // register footprint for a path that essentially never runs)
  float l = 0.f;
  for (int c = 0; c < kHeadDim / 32; ++c) {
    float o[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) o[e] = 0.f;
    float lc = 0.f;
    auto accum = [&](int j, bool pref) {
      const float w = __expf(score(key_row(j, pref, false)) - m);
      const __nv_bfloat16 *v = key_row(j, pref, true) + 32 * c;
      lc += w;
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] += w * __bfloat162float(v[e]);
    };
    if (m != -INFINITY) {
      for (int j = kp0; j < kp1; ++j) accum(j, true);
      for (int j = ks0; j < ks1; ++j)
        if (visible(j)) accum(j, false);
    }
    if (c == 0) l = lc;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (item.whole) {
      __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                           (((int64_t)geo.b * p.r_max + node) * p.hq + hq_idx) * kHeadDim + 32 * c;
#pragma unroll
      for (int e = 0; e < 32; ++e) out[e] = __float2bfloat16(o[e] * inv);
    } else {
      float *out = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim + 32 * c;
#pragma unroll
      for (int e = 0; e < 32; ++e) out[e] = o[e] * inv;
    }
  }
  const float lse_n = l > 0.f ? m + __logf(l) : -INFINITY;
  if (item.whole) {
    if (p.lse) p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node] = lse_n;
  } else {
    sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = lse_n;
  }
}

int launch_2cta(const CUtensorMap &mq, const CUtensorMap &mqt, const CUtensorMap &mk, const CUtensorMap &mv, const CUtensorMap &mtk,
                const CUtensorMap &mtv, const Sm100Params &sp, int emu, cudaStream_t stream);

}  // namespace sm100
}  // namespace sdb
