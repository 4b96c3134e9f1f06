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

// exp2 of two values on the FMA pipe (offloads the MUFU): 2^x = 2^floor(x) *
// p(frac(x)), p a cubic fit of 2^f on [0, 1) with p(0) = 1 (max relative
// error 8.6e-5, far below the bf16 rounding of P).
__device__ __forceinline__ void ex2_emu2(float x, float y, float &ox, float &oy) {
  constexpr float kRound = 12582912.0f;  // 2^23 + 2^22
  const uint64_t xy = f2pack(fmaxf(x, -127.f), fmaxf(y, -127.f));
  const uint64_t rr = fadd2_rm(xy, f2pack(kRound, kRound));  // floor(x) in the low mantissa bits
  const uint64_t fl = fadd2(rr, f2pack(-kRound, -kRound));
  float fx, fy;
  {
    float a, b, c, d;
    f2unpack(xy, a, b);
    f2unpack(fl, c, d);
    fx = a - c;
    fy = b - d;
  }
  const uint64_t f = f2pack(fx, fy);
  uint64_t pp = f2pack(0.07706617563962936f, 0.07706617563962936f);
  pp = ffma2(pp, f, f2pack(0.22764593362808228f, 0.22764593362808228f));
  pp = ffma2(pp, f, f2pack(0.6951165795326233f, 0.6951165795326233f));
  pp = ffma2(pp, f, f2pack(1.0f, 1.0f));
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

struct Sm100Params {
  TreeAttnParams p;
  int m_blocks;    // row blocks (NT x 128 query rows) per (b, kvh)
  int units;       // batch * hkv * m_blocks
  int w_pref;      // nominal prefix tiles per unit: ceil(max_ctx / 128)
  int w_unit;      // nominal tiles per unit: w_pref + ceil(r_max / 128)
  int n_ctas;      // persistent CTAs (stream-K partition of units * w_unit tiles)
  int rows_unit;   // NT * 128
  int64_t total;   // units * w_unit
  float *part_out; // [n_ctas * 2][rows_unit][128] partial outputs of split units
  float *part_lse; // [n_ctas * 2][rows_unit]
  int64_t *seg;    // [n_ctas + 1] segment starts, written by the main kernel for the fix-up
};

__host__ __device__ __forceinline__ int64_t seg_begin(const Sm100Params &sp, int k) {
  return sp.total * k / sp.n_ctas;
}

// One contiguous piece of a unit's nominal tile range owned by a CTA.
struct Item {
  int unit, t0, t1, slot;
  bool whole;
};

// i-th item of CTA k (items walk the CTA's [seg_begin(k), seg_begin(k+1)) range).
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
  int pa, n_pref, sa, n_suf, n_tiles;
  bool active;
};

__device__ __forceinline__ ItemGeo item_geo(const Sm100Params &sp, const Item &it, int g) {
  const TreeAttnParams &p = sp.p;
  ItemGeo o;
  // unit = mblk * (B * Hkv) + b * Hkv + kvh: the row blocks of one KV head run
  // on CTAs ~n_ctas / m_blocks apart at the same time, so its K/V stream is
  // read from HBM once and served from L2 to the other row blocks.
  const int bh = p.batch * p.hkv;
  o.b = (it.unit % bh) / p.hkv;
  o.kvh = it.unit % p.hkv;
  o.row0 = (it.unit / bh) * sp.rows_unit;
  o.n_nodes = min(p.n_rows[o.b], p.r_max);
  o.rows_total = o.n_nodes * g;
  o.C = p.ctx_len[o.b];
  const int pb = (o.C + kTileN - 1) / kTileN;
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

template <int NT>
struct alignas(1024) Smem {
  uint8_t q[NT][kTileBytes];
  uint8_t k[2][kTileBytes];
  uint8_t v[2][kTileBytes];
  uint64_t q_full, q_empty;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[NT], p_full[NT], o_done[NT], o_free[NT];
  uint32_t tmem_base;
};

template <int NT, int EMU>
__global__ void __launch_bounds__(128 + NT * 128, 1)
    tree_attn_tcgen05_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tk,
                             const __grid_constant__ CUtensorMap tm_tv, const Sm100Params sp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NT> &sm = *reinterpret_cast<Smem<NT> *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TreeAttnParams &p = sp.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.hq / p.hkv;
  const float sl2 = p.scale * 1.4426950408889634f;

  if (threadIdx.x == 0) {
    sp.seg[blockIdx.x] = seg_begin(sp, blockIdx.x);
    if (blockIdx.x == 0) sp.seg[sp.n_ctas] = sp.total;
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 128);
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
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      tma_prefetch(&tm_tk);
      tma_prefetch(&tm_tv);
      const int bs = p.block_size;
      const int pages_per_tile = kTileN / bs;
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, blockIdx.x);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        // Q tiles of this unit once the previous unit's S MMAs are done
        mbar_wait(&sm.q_empty, (g_q & 1) ^ 1);
        mbar_expect_tx(&sm.q_full, NT * kTileBytes);
        for (int t = 0; t < NT; ++t) {
          const int node0 = (geo.row0 + t * kTileM) / g;
          for (int c = 0; c < 2; ++c)
            tma_load_4d(sm.q[t] + c * kChunkBytes, &tm_q, &sm.q_full, c * 64, 0, geo.kvh,
                        geo.b * p.r_max + node0);
        }
        ++g_q;
        const int n_valid_pages = (geo.C + bs - 1) / bs;
        const int32_t *bt = p.block_table + (int64_t)geo.b * p.max_blocks;
        for (int it = 0; it < geo.n_tiles; ++it, ++g_tile) {
          const int s = g_tile & 1;
          const uint32_t ph = (g_tile >> 1) & 1;
          const bool pref = it < geo.n_pref;
          const int tile = pref ? geo.pa + it : geo.sa + (it - geo.n_pref);
          for (int kv = 0; kv < 2; ++kv) {
            uint64_t *emp = kv ? &sm.v_empty[s] : &sm.k_empty[s];
            uint64_t *ful = kv ? &sm.v_full[s] : &sm.k_full[s];
            uint8_t *dst = kv ? sm.v[s] : sm.k[s];
            mbar_wait(emp, ph ^ 1);
            mbar_expect_tx(ful, kTileBytes);
            if (pref) {
              const CUtensorMap *m = kv ? &tm_v : &tm_k;
              for (int pg = 0; pg < pages_per_tile; ++pg) {
                const int lp = tile * pages_per_tile + pg;
                const int page = lp < n_valid_pages ? bt[lp] : p.num_blocks;  // OOB page -> zero fill
                const int rowc = (page * p.hkv + geo.kvh) * bs;
                for (int c = 0; c < 2; ++c) tma_load_2d(dst + c * kChunkBytes + pg * bs * 128, m, ful, c * 64, rowc);
              }
            } else {
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
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc(false);
      constexpr uint32_t idesc_o = make_idesc(true);
      const uint32_t q_base = smem_u32(sm.q[0]);
      auto issue_s = [&](int t, int s) {
        const uint32_t qa = q_base + t * kTileBytes;
        const uint32_t ka = smem_u32(sm.k[s]);
#pragma unroll
        for (int k = 0; k < kHeadDim / 16; ++k) {
          const uint32_t off = (k >> 2) * kChunkBytes + (k & 3) * 32;
          mma_ss(tmem + t * 128, sw128_desc(qa + off, 16, 1024), sw128_desc(ka + off, 16, 1024), idesc_s, k > 0);
        }
      };
      auto issue_pv = [&](int t, int s, bool acc) {
        const uint32_t va = smem_u32(sm.v[s]);
#pragma unroll
        for (int k = 0; k < kTileN / 16; ++k) {
          mma_ts(tmem + 256 + t * 128, tmem + t * 128 + k * 8, sw128_desc(va + k * 2048, kChunkBytes, 1024),
                 idesc_o, (acc || k > 0) ? 1u : 0u);
        }
      };
      uint32_t g_tile = 0, g_q = 0;
      ItemIter iter(sp, blockIdx.x);
      Item item;
      while (iter.next(sp, item)) {
        const ItemGeo geo = item_geo(sp, item, g);
        if (!geo.active) continue;
        mbar_wait(&sm.q_full, g_q & 1);
        mbar_wait(&sm.k_full[g_tile & 1], (g_tile >> 1) & 1);
        tc_fence_after();
        for (int t = 0; t < NT; ++t) {
          issue_s(t, g_tile & 1);
          tc_commit(&sm.s_full[t]);
        }
        tc_commit(&sm.k_empty[g_tile & 1]);
        for (int it = 0; it < geo.n_tiles; ++it) {
          const uint32_t gt = g_tile + it;
          const int s = gt & 1;
          mbar_wait(&sm.v_full[s], (gt >> 1) & 1);
          tc_fence_after();
          for (int t = 0; t < NT; ++t) {
            mbar_wait(&sm.p_full[t], gt & 1);
            if (it == 0) mbar_wait(&sm.o_free[t], (g_q & 1) ^ 1);  // previous unit's epilogue read O_t
            tc_fence_after();
            issue_pv(t, s, it > 0);
            tc_commit(&sm.o_done[t]);
            if (it + 1 < geo.n_tiles) {
              const int s2 = (gt + 1) & 1;
              if (t == 0) {
                mbar_wait(&sm.k_full[s2], ((gt + 1) >> 1) & 1);
                tc_fence_after();
              }
              issue_s(t, s2);
              tc_commit(&sm.s_full[t]);
              if (t == NT - 1) tc_commit(&sm.k_empty[s2]);
            }
          }
          tc_commit(&sm.v_empty[s]);
        }
        tc_commit(&sm.q_empty);  // all S MMAs of this unit read Q
        g_tile += geo.n_tiles;
        ++g_q;
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax warpgroups =====================
    const int t = (warp - 4) >> 2;          // query tile
    const int i = ((warp & 3) << 5) + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + t * 128;
    const uint32_t t_o = tmem + lane_off + 256 + t * 128;
    const int local = t * kTileM + i;  // row within the unit
    uint32_t g_tile = 0;
    ItemIter iter(sp, blockIdx.x);
    Item item;
    while (iter.next(sp, item)) {
      const ItemGeo geo = item_geo(sp, item, g);
      const int rho = geo.row0 + local;
      const bool row_ok = rho < geo.rows_total;
      const bool in_range = rho < p.r_max * g;
      const int node_o = rho / g;
      const int hq_idx = geo.kvh * g + (rho % g);
      if (!geo.active) {
        // padding rows / an empty split piece: zeros and -inf
        if (!item.whole) {
          float *o = sp.part_out + ((int64_t)item.slot * sp.rows_unit + local) * kHeadDim;
          for (int c = 0; c < kHeadDim; c += 4) *reinterpret_cast<float4 *>(o + c) = make_float4(0, 0, 0, 0);
          sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = -INFINITY;
        } else if (in_range) {
          __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                             (((int64_t)geo.b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim;
          for (int c = 0; c < kHeadDim; c += 8) *reinterpret_cast<uint4 *>(o + c) = make_uint4(0, 0, 0, 0);
          if (p.lse) p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = -INFINITY;
        }
        continue;
      }
      const int node = min(rho / g, max(geo.n_nodes - 1, 0));
      const uint32_t *mrow = p.mask_words + ((int64_t)geo.b * p.r_max + node) * p.n_words;
      float m = -INFINITY, l = 0.f;
      for (int it = 0; it < geo.n_tiles; ++it) {
        const uint32_t gt = g_tile + it;
        const bool pref = it < geo.n_pref;
        const int key0 = pref ? (geo.pa + it) * kTileN : (geo.sa + it - geo.n_pref) * kTileN;
        const int kvalid = pref ? geo.C - key0 : geo.n_nodes - key0;
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
            bits = (wi < p.n_words && row_ok) ? mrow[wi] : 0u;
          }
          vm[w] = bits & low;
        }
        mbar_wait(&sm.s_full[t], gt & 1);
        tc_fence_after();
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
        if (it == 0) {
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
          // PV(it-1) has completed: s_full(it) was committed after it
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
        mbar_arrive(&sm.p_full[t]);
      }
      // epilogue: wait for the last PV, normalise, store (final or partial)
      mbar_wait(&sm.o_done[t], (g_tile + geo.n_tiles - 1) & 1);
      tc_fence_after();
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
      // O_t may now be overwritten by the next unit's first PV
      tc_fence_before();
      mbar_arrive(&sm.o_free[t]);
      if (item.whole) {
        if (in_range && p.lse)
          p.lse[((int64_t)geo.b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
      } else {
        sp.part_lse[(int64_t)item.slot * sp.rows_unit + local] = row_ok ? lse_n : -INFINITY;
      }
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

// Stream-K fix-up: one block row per CTA boundary k (1..n_ctas-1).  A
// boundary strictly inside unit u splits it; the FIRST boundary inside u
// merges all of u's pieces (same math as merge_partials,
// attention.py:108-124).  grid (n_ctas - 1, rows_unit / 4), one warp per row.
__global__ void __launch_bounds__(128) tree_attn_fixup_kernel(const Sm100Params sp) {
  const TreeAttnParams &p = sp.p;
  const int k = blockIdx.x + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int local = blockIdx.y * 4 + warp;
  if (local >= sp.rows_unit) return;
  const int64_t ck = sp.seg[k];
  const int W = sp.w_unit;
  const int unit = (int)(ck / W);
  const int64_t ustart = (int64_t)unit * W, uend = ustart + W;
  if (ck == ustart) return;              // boundary between units: nothing split here
  if (sp.seg[k - 1] > ustart) return;    // an earlier boundary inside u merges it
  const int g = p.hq / p.hkv;
  const int bh = p.batch * p.hkv;
  const int b = (unit % bh) / p.hkv, kvh = unit % p.hkv;
  const int rho = (unit / bh) * sp.rows_unit + local;
  if (rho >= p.r_max * g) return;
  const int n_nodes = min(p.n_rows[b], p.r_max);
  const int node = rho / g, hq_idx = kvh * g + rho % g;
  __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(p.out) + (((int64_t)b * p.r_max + node) * p.hq + hq_idx) * kHeadDim;
  float *lse_out = p.lse ? p.lse + ((int64_t)b * p.hq + hq_idx) * p.r_max + node : nullptr;
  if (rho >= n_nodes * g) {
    *reinterpret_cast<uint2 *>(out + lane * 4) = make_uint2(0, 0);
    if (lse_out && lane == 0) *lse_out = -INFINITY;
    return;
  }
  // pieces: CTA k-1 (its first item iff its segment starts at the unit start,
  // else its last item), then the first item of every later CTA starting in u
  const int first_slot = (k - 1) * 2 + (sp.seg[k - 1] == ustart ? 0 : 1);
  int kk_end = k;
  while (kk_end < sp.n_ctas && sp.seg[kk_end] < uend) ++kk_end;  // CTAs k..kk_end-1 start inside u
  float mx = sp.part_lse[(int64_t)first_slot * sp.rows_unit + local];
  for (int kk = k; kk < kk_end; ++kk) mx = fmaxf(mx, sp.part_lse[(int64_t)(kk * 2) * sp.rows_unit + local]);
  float wsum = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int kk = k - 1; kk < kk_end; ++kk) {
    const int sl = kk == k - 1 ? first_slot : kk * 2;
    const float l = sp.part_lse[(int64_t)sl * sp.rows_unit + local];
    if (l == -INFINITY) continue;
    const float w = __expf(l - mx);
    wsum += w;
    const float4 o =
        *reinterpret_cast<const float4 *>(sp.part_out + ((int64_t)sl * sp.rows_unit + local) * kHeadDim + lane * 4);
    acc[0] = fmaf(w, o.x, acc[0]);
    acc[1] = fmaf(w, o.y, acc[1]);
    acc[2] = fmaf(w, o.z, acc[2]);
    acc[3] = fmaf(w, o.w, acc[3]);
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
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 && sm100::encode_fn() != nullptr;
}

// Stream-K plan: units x nominal tiles split evenly over the persistent CTAs.
static void sm100_plan(const TreeAttnParams &p, int ctas_override, sm100::Sm100Params &sp) {
  using namespace sm100;
  const int g = p.hq / p.hkv;
  const int rows = p.r_max * g;
  const int nt = rows > kTileM ? 2 : 1;
  sp.p = p;
  sp.rows_unit = nt * kTileM;
  sp.m_blocks = cdiv(rows, sp.rows_unit);
  sp.units = p.batch * p.hkv * sp.m_blocks;
  sp.w_pref = cdiv(max(p.max_ctx, 0), kTileN);
  sp.w_unit = sp.w_pref + cdiv(p.r_max, kTileN);
  sp.total = (int64_t)sp.units * sp.w_unit;
  int n = ctas_override > 0 ? ctas_override : num_sms();
  // at least ~2 tiles per CTA
  n = (int)std::max<int64_t>(1, std::min<int64_t>(n, ctas_override > 0 ? sp.total : sp.total / 2));
  sp.n_ctas = n;
  sp.part_out = nullptr;
  sp.part_lse = nullptr;
  sp.seg = nullptr;
}

int64_t tree_attn_sm100_workspace(const TreeAttnParams &p, int ctas_override) {
  sm100::Sm100Params sp;
  sm100_plan(p, ctas_override, sp);
  return (int64_t)sp.n_ctas * 2 * sp.rows_unit * (sm100::kHeadDim + 1) * (int64_t)sizeof(float) +
         (int64_t)(sp.n_ctas + 1) * 8 + 256;
}

int launch_tree_attn_sm100(const TreeAttnParams &p, int ctas_override, void *workspace, cudaStream_t stream) {
  using namespace sm100;
  const int g = p.hq / p.hkv;
  const int d = kHeadDim;
  CUtensorMap mq, mk, mv, mtk, mtv;
  {
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)g, (cuuint64_t)p.hkv, (cuuint64_t)p.batch * p.r_max};
    cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)g * d * 2, (cuuint64_t)p.hq * d * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)g, 1, (cuuint32_t)(kTileM / g)};
    if (!make_map(&mq, p.q, 4, dims, strides, box)) return SDB_E_UNSUPPORTED;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)p.num_blocks * p.hkv * p.block_size};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)p.block_size};
    if (!make_map(&mk, p.k_cache, 2, dims, strides, box)) return SDB_E_UNSUPPORTED;
    if (!make_map(&mv, p.v_cache, 2, dims, strides, box)) return SDB_E_UNSUPPORTED;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)p.hkv, (cuuint64_t)p.batch * p.r_max};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)p.hkv * d * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kTileN};
    if (!make_map(&mtk, p.tree_k, 3, dims, strides, box)) return SDB_E_UNSUPPORTED;
    if (!make_map(&mtv, p.tree_v, 3, dims, strides, box)) return SDB_E_UNSUPPORTED;
  }
  Sm100Params sp;
  sm100_plan(p, ctas_override, sp);
  sp.part_out = reinterpret_cast<float *>(workspace);
  sp.part_lse = sp.part_out + (int64_t)sp.n_ctas * 2 * sp.rows_unit * kHeadDim;
  sp.seg = reinterpret_cast<int64_t *>(sp.part_lse + (int64_t)sp.n_ctas * 2 * sp.rows_unit);
  static int emu = -1;
  if (emu < 0) {
    const char *e = getenv("SDB_ATTN_EMU");
    emu = e ? atoi(e) : 1;
    emu = emu < 0 ? 0 : (emu > 2 ? 2 : emu);
  }
  dim3 grid(sp.n_ctas);
#define SDB_LAUNCH_TC(NT, EMU)                                                                               \
  do {                                                                                                       \
    const size_t smem = sizeof(Smem<NT>) + 1024;                                                             \
    cudaFuncSetAttribute(tree_attn_tcgen05_kernel<NT, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    tree_attn_tcgen05_kernel<NT, EMU><<<grid, 128 + NT * 128, smem, stream>>>(mq, mk, mv, mtk, mtv, sp);   \
  } while (0)
  if (sp.rows_unit == 2 * kTileM) {
    if (emu == 0) SDB_LAUNCH_TC(2, 0); else if (emu == 2) SDB_LAUNCH_TC(2, 2); else SDB_LAUNCH_TC(2, 1);
  } else {
    if (emu == 0) SDB_LAUNCH_TC(1, 0); else if (emu == 2) SDB_LAUNCH_TC(1, 2); else SDB_LAUNCH_TC(1, 1);
  }
#undef SDB_LAUNCH_TC
  SDB_CHECK_LAUNCH();
  if (sp.n_ctas > 1) {
    dim3 fgrid(sp.n_ctas - 1, cdiv(sp.rows_unit, 4));
    tree_attn_fixup_kernel<<<fgrid, 128, 0, stream>>>(sp);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

}  // namespace sdb
