// tcgen05.mma throughput on one SM / one SM pair, with the descriptors of the
// attention kernels: S = Q K^T (SS, K-major SW128) and O += P V (TS, P in
// TMEM, V MN-major SW128), cta_group::1 (M = 128) and ::2 (M = 256).
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2508_08192_b200/csrc -I../../include
//        mma_bench.cu -o mma_bench -lcuda && ./mma_bench
#include "sm100_common.cuh"
#include <cstdio>

using namespace sdb::sm100;

constexpr int NITER = 512;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_mn(int M, int N, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// MODE 0: SS (S = QK^T) only; 1: TS (PV) only; 2: alternate SS + TS (one attention tile)
template <int CG, int N, int MODE, int LOAD>
__global__ void __launch_bounds__(256, 1) kbench(long long *cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *A = base;           // 32 KB: 128 rows x 128 (2 SW128 chunks)
  uint8_t *B = base + 32768;   // 64 KB
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 97u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    // two bf16 in [-2, 2): sign | exponent 126..127 | random mantissa
    const uint32_t lo = ((h & 1u) << 15) | ((126u + ((h >> 1) & 1u)) << 7) | ((h >> 2) & 0x7fu);
    const uint32_t hi = (((h >> 9) & 1u) << 15) | ((126u + ((h >> 10) & 1u)) << 7) | ((h >> 11) & 0x7fu);
    reinterpret_cast<uint32_t *>(base)[i] = (LOAD & 4) ? (lo | (hi << 16)) : 0x3c003c00u;
  }
  if (threadIdx.x == 0) {
    done = 0;
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const bool leader = CG == 1 || cta_rank() == 0;
  if ((LOAD & 4) && warp < 4) {
    uint32_t r[32];
    for (int e = 0; e < 32; ++e) r[e] = reinterpret_cast<uint32_t *>(base)[(threadIdx.x * 32 + e) & 8191];
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    for (int c = 0; c < 4; ++c) SDB_TMEM_ST32(tmem + lane_off + 384 + c * 32, r);
    tmem_wait_st();
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && leader) {
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    constexpr int M = 128 * CG;
    constexpr uint32_t id_ss = idesc_mn(M, N, false), id_ts = idesc_mn(M, N, true);
    // K-major B: N rows per CTA (cg2: N/2 rows each) -> chunk stride
    constexpr uint32_t bchunk = (N / CG) * 128;
    long long t0 = clock64();
    for (int it = 0; it < NITER; ++it) {
      if (MODE == 0 || MODE == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = sw128_desc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sw128_desc(b + (k >> 2) * bchunk + (k & 3) * 32, 16, 1024);
          if (CG == 2) mma2(tmem, ad, bd, id_ss, k > 0); else mma_ss(tmem, ad, bd, id_ss, k > 0);
        }
      }
      if ((LOAD & 8) && MODE == 2) tc_commit(&bar2);
      if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // V MN-major: 16 keys x N/CG cols per K step (N/CG <= 64 -> one SW128 chunk row block of 2 KB)
          const uint64_t bd = sw128_desc(b + k * 2048, (N / CG) * 256, 1024);
          if (CG == 2) mma2_ts(tmem + 256, tmem + 384 + k * 8, bd, id_ts, k > 0);
          else mma_ts(tmem + 256, tmem + 384 + k * 8, bd, id_ts, k > 0);
        }
      }
    }
    if (CG == 2) commit2(&bar); else tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    done = 1;
  }
  if ((LOAD & 3) && warp >= 4) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t r[32];
    int n = 0;
    while (!done) {
      SDB_TMEM_LD32(tmem + lane_off + 384, r);
      SDB_TMEM_LD32(tmem + lane_off + 416, (r));
      tmem_wait_ld();
      if ((LOAD & 3) == 2) { SDB_TMEM_ST32(tmem + lane_off + 448, r); tmem_wait_st(); }
      ++n;
    }
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0 && warp == 4) printf("   load loops %d (r %u)\n", n, r[3]);
  }
  if (CG == 2 && !leader && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    done = 1;
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int CG, int N, int MODE, int LOAD = 0>
void run(const char *name, int ctas) {
  long long *cyc;
  cudaMalloc(&cyc, 296 * 8);
  cudaMemset(cyc, 0, 296 * 8);
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(kbench<CG, N, MODE, LOAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, kbench<CG, N, MODE, LOAD>, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, cyc, ctas * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  int n = 0;
  for (int i = 0; i < ctas; ++i)
    if (h[i]) { c += h[i]; ++n; }
  c /= n;
  const double gemms = (MODE == 2 ? 2.0 : 1.0) * NITER;
  const double flop_per_sm = gemms * 2.0 * 128 * N * 128;  // per SM: 128 rows of M, N cols, K = 128
  printf("%-28s ctas %3d: %8.0f cyc, %6.0f flop/clk/SM, %5.1f clk per M128xN%dxK16 (%s)\n", name, ctas, c,
         flop_per_sm / c, c / (gemms * 8), N, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<2, 128, 2, 4>("cg2 SS+TS N128 random", 148);
  run<2, 128, 2, 8>("cg2 SS+TS N128 commits", 148);
  run<2, 128, 2, 12>("cg2 SS+TS N128 random+commits", 148);
  run<1, 128, 2, 4>("cg1 SS+TS N128 random", 148);
  run<2, 128, 0, 4>("cg2 SS N128 random", 148);
  run<2, 128, 1, 4>("cg2 TS N128 random", 148);
  run<2, 256, 0, 4>("cg2 SS N256 random", 148);
  run<2, 128, 2, 1>("cg2 SS+TS N128 +LDTM", 148);
  run<2, 128, 2, 2>("cg2 SS+TS N128 +LDTM/STTM", 148);
  run<1, 128, 2, 1>("cg1 SS+TS N128 +LDTM", 148);
  run<1, 128, 2, 2>("cg1 SS+TS N128 +LDTM/STTM", 148);
  for (int ctas : {148}) {
    run<1, 128, 0>("cg1 SS N128", ctas);
    run<1, 256, 0>("cg1 SS N256", ctas);
    run<1, 128, 1>("cg1 TS N128", ctas);
    run<1, 128, 2>("cg1 SS+TS N128", ctas);
    run<2, 128, 0>("cg2 SS N128", ctas);
    run<2, 256, 0>("cg2 SS N256", ctas);
    run<2, 128, 1>("cg2 TS N128", ctas);
    run<2, 128, 2>("cg2 SS+TS N128", ctas);
  }
  return 0;
}
