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
  int m_blocks;  // CTA row blocks per (b, kvh)
};

template <int NT>
struct alignas(1024) Smem {
  uint8_t q[NT][kTileBytes];
  uint8_t k[2][kTileBytes];
  uint8_t v[2][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[NT], p_full[NT], o_done[NT];
  uint32_t tmem_base;
};

template <int NT>
__global__ void __launch_bounds__(128 + NT * 128, 1)
    tree_attn_tcgen05_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tk,
                             const __grid_constant__ CUtensorMap tm_tv, const Sm100Params sp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NT> &sm = *reinterpret_cast<Smem<NT> *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TreeAttnParams &p = sp.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, mblk = blockIdx.y;
  const int b = blockIdx.z / p.hkv, kvh = blockIdx.z % p.hkv;
  const int g = p.hq / p.hkv;
  const int n_nodes = min(p.n_rows[b], p.r_max);
  const int rows_total = n_nodes * g;
  const int row0 = mblk * NT * kTileM;
  const int C = p.ctx_len[b];
  const int n_pref_tiles = (C + kTileN - 1) / kTileN;
  const int n_suf_tiles = (n_nodes + kTileN - 1) / kTileN;
  const int tiles_per = (n_pref_tiles + p.num_splits - 1) / p.num_splits;
  const int t_begin = min(split * tiles_per, n_pref_tiles);
  const int t_end_pref = min(t_begin + tiles_per, n_pref_tiles);
  const bool last_split = split == p.num_splits - 1;
  const int n_tiles = (t_end_pref - t_begin) + (last_split ? n_suf_tiles : 0);
  const float sl2 = p.scale * 1.4426950408889634f;

  // Whole CTA is padding, or this split has no keys: write zeros / -inf.
  if (row0 >= rows_total || n_tiles == 0) {
    if (threadIdx.x >= 128) {
      const int i = threadIdx.x - 128;  // 0 .. NT*128-1
      const int rho = row0 + i;
      const bool in_range = rho < p.r_max * g;
      if (in_range && (p.num_splits > 1 || rho >= rows_total)) {
        const int node = rho / g, hq_idx = kvh * g + rho % g;
        if (p.num_splits == 1) {
          __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) + (((int64_t)b * p.r_max + node) * p.hq + hq_idx) * kHeadDim;
          for (int c = 0; c < kHeadDim; c += 8) *reinterpret_cast<uint4 *>(o + c) = make_uint4(0, 0, 0, 0);
          if (p.lse) p.lse[((int64_t)b * p.hq + hq_idx) * p.r_max + node] = -INFINITY;
        } else {
          const int64_t total = (int64_t)p.batch * p.r_max * p.hq;
          const int64_t wid = ((int64_t)b * p.r_max + node) * p.hq + hq_idx;
          float *o = p.ws_out + (split * total + wid) * kHeadDim;
          for (int c = 0; c < kHeadDim; c += 4) *reinterpret_cast<float4 *>(o + c) = make_float4(0, 0, 0, 0);
          p.ws_lse[(int64_t)split * total + ((int64_t)b * p.hq + hq_idx) * p.r_max + node] = -INFINITY;
        }
      }
    }
    return;
  }

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
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
      // Q: NT tiles x 2 column chunks; box = {64, g, 1, 128/g} over
      // [B*R, Hkv, g, d] -> rows (node, j) of this KV head.
      mbar_expect_tx(&sm.q_full, NT * kTileBytes);
      const int nodes_per_tile = kTileM / g;
      for (int t = 0; t < NT; ++t) {
        const int node0 = (row0 + t * kTileM) / g;
        for (int c = 0; c < 2; ++c)
          tma_load_4d(sm.q[t] + c * kChunkBytes, &tm_q, &sm.q_full, c * 64, 0, kvh, b * p.r_max + node0);
      }
      (void)nodes_per_tile;
      const int bs = p.block_size;
      const int pages_per_tile = kTileN / bs;
      const int n_valid_pages = (C + bs - 1) / bs;
      const int32_t *bt = p.block_table + (int64_t)b * p.max_blocks;
      for (int it = 0; it < n_tiles; ++it) {
        const int s = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        const bool pref = it < (t_end_pref - t_begin);
        const int tile = t_begin + it;
        // K
        mbar_wait(&sm.k_empty[s], ph ^ 1);
        mbar_expect_tx(&sm.k_full[s], kTileBytes);
        if (pref) {
          for (int pg = 0; pg < pages_per_tile; ++pg) {
            const int lp = tile * pages_per_tile + pg;
            const int page = lp < n_valid_pages ? bt[lp] : p.num_blocks;  // OOB page -> zero fill
            const int rowc = (page * p.hkv + kvh) * bs;
            for (int c = 0; c < 2; ++c) tma_load_2d(sm.k[s] + c * kChunkBytes + pg * bs * 128, &tm_k, &sm.k_full[s], c * 64, rowc);
          }
        } else {
          const int st = it - (t_end_pref - t_begin);
          for (int c = 0; c < 2; ++c)
            tma_load_3d(sm.k[s] + c * kChunkBytes, &tm_tk, &sm.k_full[s], c * 64, kvh, b * p.r_max + st * kTileN);
        }
        // V
        mbar_wait(&sm.v_empty[s], ph ^ 1);
        mbar_expect_tx(&sm.v_full[s], kTileBytes);
        if (pref) {
          for (int pg = 0; pg < pages_per_tile; ++pg) {
            const int lp = tile * pages_per_tile + pg;
            const int page = lp < n_valid_pages ? bt[lp] : p.num_blocks;
            const int rowc = (page * p.hkv + kvh) * bs;
            for (int c = 0; c < 2; ++c) tma_load_2d(sm.v[s] + c * kChunkBytes + pg * bs * 128, &tm_v, &sm.v_full[s], c * 64, rowc);
          }
        } else {
          const int st = it - (t_end_pref - t_begin);
          for (int c = 0; c < 2; ++c)
            tma_load_3d(sm.v[s] + c * kChunkBytes, &tm_tv, &sm.v_full[s], c * 64, kvh, b * p.r_max + st * kTileN);
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
      mbar_wait(&sm.q_full, 0);
      mbar_wait(&sm.k_full[0], 0);
      tc_fence_after();
      for (int t = 0; t < NT; ++t) {
        issue_s(t, 0);
        tc_commit(&sm.s_full[t]);
      }
      tc_commit(&sm.k_empty[0]);
      for (int it = 0; it < n_tiles; ++it) {
        const int s = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        mbar_wait(&sm.v_full[s], ph);
        tc_fence_after();
        for (int t = 0; t < NT; ++t) {
          mbar_wait(&sm.p_full[t], it & 1);
          tc_fence_after();
          issue_pv(t, s, it > 0);
          tc_commit(&sm.o_done[t]);
          if (it + 1 < n_tiles) {
            const int s2 = (it + 1) & 1;
            if (t == 0) {
              mbar_wait(&sm.k_full[s2], ((it + 1) >> 1) & 1);
              tc_fence_after();
            }
            issue_s(t, s2);
            tc_commit(&sm.s_full[t]);
            if (t == NT - 1) tc_commit(&sm.k_empty[s2]);
          }
        }
        tc_commit(&sm.v_empty[s]);
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax warpgroups =====================
    const int t = (warp - 4) >> 2;          // query tile
    const int i = ((warp & 3) << 5) + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + t * 128;
    const uint32_t t_o = tmem + lane_off + 256 + t * 128;
    const int rho = row0 + t * kTileM + i;
    const bool row_ok = rho < rows_total;
    const int node = min(rho / g, max(n_nodes - 1, 0));
    const uint32_t *mrow = p.mask_words + ((int64_t)b * p.r_max + node) * p.n_words;
    float m = -INFINITY, l = 0.f;
    const int n_pref_it = t_end_pref - t_begin;
    for (int it = 0; it < n_tiles; ++it) {
      const bool pref = it < n_pref_it;
      const int key0 = pref ? (t_begin + it) * kTileN : (it - n_pref_it) * kTileN;  // prefix key / suffix row
      const int kvalid = pref ? C - key0 : n_nodes - key0;                         // keys valid in this tile
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
      mbar_wait(&sm.s_full[t], it & 1);
      tc_fence_after();
      // the whole S row (128 fp32) in registers: one TMEM pass
      uint32_t r[128];
      SDB_TMEM_LD32(t_s + 0, (r + 0));
      SDB_TMEM_LD32(t_s + 32, (r + 32));
      SDB_TMEM_LD32(t_s + 64, (r + 64));
      SDB_TMEM_LD32(t_s + 96, (r + 96));
      tmem_wait_ld();
      if (!full) {
        // invisible keys -> -inf (prefix tail beyond ctx, or not an ancestor)
#pragma unroll
        for (int e = 0; e < 128; ++e)
          if (!((vm[e >> 5] >> (e & 31)) & 1u)) r[e] = 0xff800000u;
      }
      // row max with 8 independent chains, on raw scores (scale > 0)
      float mx8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = __uint_as_float(r[k]);
#pragma unroll
      for (int e = 8; e < 128; e += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mx8[k] = fmaxf(mx8[k], __uint_as_float(r[e + k]));
      }
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
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
      // P = exp2(s * scale_log2 - m), packed bf16 in place into r[0..63]
      float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 128; e += 2) {
        const float p0 = ex2(fmaf(__uint_as_float(r[e]), sl2, neg_mu));
        const float p1 = ex2(fmaf(__uint_as_float(r[e + 1]), sl2, neg_mu));
        l8[(e >> 1) & 7] += p0 + p1;
        r[e >> 1] = pack_bf16(p0, p1);
      }
      l = l * corr + (((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7])));
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
    // epilogue: wait for the last PV, normalise, store
    mbar_wait(&sm.o_done[t], (n_tiles - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const float lse_n = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
    const int hq_idx = kvh * g + (rho % g);
    const int node_o = rho / g;
    const bool in_range = rho < p.r_max * g;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      SDB_TMEM_LD32(t_o + c * 32, r);
      tmem_wait_ld();
      if (!in_range) continue;
      if (p.num_splits == 1) {
        __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(p.out) +
                           (((int64_t)b * p.r_max + node_o) * p.hq + hq_idx) * kHeadDim + c * 32;
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
      } else if (row_ok) {
        const int64_t total = (int64_t)p.batch * p.r_max * p.hq;
        const int64_t wid = ((int64_t)b * p.r_max + node_o) * p.hq + hq_idx;
        float *o = p.ws_out + (split * total + wid) * kHeadDim + c * 32;
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4 *>(o + e) =
              make_float4(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv,
                          __uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
      }
    }
    if (in_range) {
      if (p.num_splits == 1) {
        if (p.lse) p.lse[((int64_t)b * p.hq + hq_idx) * p.r_max + node_o] = row_ok ? lse_n : -INFINITY;
      } else if (row_ok) {
        const int64_t total = (int64_t)p.batch * p.r_max * p.hq;
        p.ws_lse[(int64_t)split * total + ((int64_t)b * p.hq + hq_idx) * p.r_max + node_o] = lse_n;
      }
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
  if (p.n_words > 4) return false;  // suffix tile bit rows: <= 128 tree rows per tile word window
  if (p.r_max > 128) return false;
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 && sm100::encode_fn() != nullptr;
}

int launch_tree_attn_sm100(const TreeAttnParams &p, cudaStream_t stream) {
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
  const int rows = p.r_max * g;
  const int nt = rows > kTileM ? 2 : 1;
  Sm100Params sp;
  sp.p = p;
  sp.m_blocks = cdiv(rows, nt * kTileM);
  dim3 grid(p.num_splits, sp.m_blocks, p.batch * p.hkv);
  if (nt == 2) {
    const size_t smem = sizeof(Smem<2>) + 1024;
    cudaFuncSetAttribute(tree_attn_tcgen05_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tree_attn_tcgen05_kernel<2><<<grid, 384, smem, stream>>>(mq, mk, mv, mtk, mtv, sp);
  } else {
    const size_t smem = sizeof(Smem<1>) + 1024;
    cudaFuncSetAttribute(tree_attn_tcgen05_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tree_attn_tcgen05_kernel<1><<<grid, 256, smem, stream>>>(mq, mk, mv, mtk, mtv, sp);
  }
  SDB_CHECK_LAUNCH();
  if (p.num_splits > 1) return launch_tree_attn_combine_bf16(p, stream);
  return SDB_OK;
}

}  // namespace sdb
