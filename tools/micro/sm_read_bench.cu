// Per-SM HBM read bandwidth of a streaming reduction on K SMs (the rest
// idle): (a) LDG.128, 1024 threads x U loads in flight; (b) 1-D TMA bulk
// copies (cp.async.bulk) into shared memory, each warp owning S stages of
// C bytes (its own producer and consumer: no cross-warp sync).  Decides
// whether a bulk-copy scan can beat the ~92 GB/s per SM the LDG scans reach
// (the C3 greedy scan on the reserved SMs, the C5 validation scan).
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o sm_read_bench sm_read_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U>
__global__ void __launch_bounds__(1024, 1) ldg_kernel(const float4 *__restrict__ buf, size_t n4, float *out) {
  float acc = -INFINITY;
  const size_t step = (size_t)gridDim.x * 1024 * U;
  for (size_t i0 = (size_t)blockIdx.x * 1024 * U; i0 < n4; i0 += step) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = i0 + (size_t)u * 1024 + threadIdx.x;
      v[u] = i < n4 ? __ldcs(buf + i) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = max_nan(acc, max_nan(max_nan(v[u].x, v[u].y), max_nan(v[u].z, v[u].w)));
  }
  if (acc == 12345.f) out[0] = acc;
}

// W warps per CTA, S stages of C bytes per warp
template <int W, int S, int C>
__global__ void __launch_bounds__(W * 32, 1) tma_kernel(const char *__restrict__ buf, size_t bytes, float *out) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[W * S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t n_chunks = bytes / C;
  const size_t per_round = (size_t)gridDim.x * W * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp * S + s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int s, size_t chunk) {
    uint64_t *b = &bar[warp * S + s];
    char *dst = smem + (size_t)(warp * S + s) * C;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(C) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(buf + chunk * C), "r"(C), "r"(smem_u32(b))
                 : "memory");
  };
  const size_t base = (size_t)blockIdx.x * W * S + (size_t)warp * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s)
      if (base + s < n_chunks) issue(s, base + s);
  float acc = -INFINITY;
  uint32_t phase = 0;
  for (size_t r0 = 0;; r0 += per_round, phase ^= 1) {
    bool any = false;
    for (int s = 0; s < S; ++s) {
      const size_t chunk = r0 + base + s;
      if (chunk >= n_chunks) break;
      any = true;
      uint64_t *b = &bar[warp * S + s];
      asm volatile(
          "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
              smem_u32(b)),
          "r"(phase)
          : "memory");
      const float4 *src = reinterpret_cast<const float4 *>(smem + (size_t)(warp * S + s) * C);
#pragma unroll 8
      for (int i = lane; i < C / 16; i += 32) {
        const float4 v = src[i];
        acc = max_nan(acc, max_nan(max_nan(v.x, v.y), max_nan(v.z, v.w)));
      }
      __syncwarp();
      if (lane == 0 && chunk + per_round < n_chunks) issue(s, chunk + per_round);
    }
    if (!any) break;
  }
  if (acc == 12345.f) out[0] = acc;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  const size_t bytes = (size_t)2 << 30;
  char *buf;
  float *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(buf, 0, bytes);
  const size_t n4 = bytes / 16;
  auto report = [&](const char *name, int k, float ms) {
    const double gbs = bytes / (ms * 1e-3) / 1e9;
    printf("%-28s K=%3d  %8.1f us  %7.1f GB/s  %6.1f GB/s/SM\n", name, k, ms * 1e3, gbs, gbs / k);
  };
  constexpr int kTmaSmemA = 8 * 2 * 12288;  // 8 warps x 2 stages x 12 KB = 192 KB
  constexpr int kTmaSmemB = 16 * 1 * 12288;  // 16 warps x 1 stage x 12 KB = 192 KB
  constexpr int kTmaSmemC = 4 * 4 * 12288;   // 4 warps x 4 stages x 12 KB = 192 KB
  cudaFuncSetAttribute(tma_kernel<8, 2, 12288>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemA);
  cudaFuncSetAttribute(tma_kernel<16, 1, 12288>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemB);
  cudaFuncSetAttribute(tma_kernel<4, 4, 12288>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemC);
  for (int k : {20, 56, 148}) {
    report("ldg U4", k, time_it([&] { ldg_kernel<4><<<k, 1024>>>((const float4 *)buf, n4, out); }));
    report("ldg U8", k, time_it([&] { ldg_kernel<8><<<k, 1024>>>((const float4 *)buf, n4, out); }));
    report("ldg U12", k, time_it([&] { ldg_kernel<12><<<k, 1024>>>((const float4 *)buf, n4, out); }));
    report("tma 8w x 2st x 12KB", k,
           time_it([&] { tma_kernel<8, 2, 12288><<<k, 8 * 32, kTmaSmemA>>>(buf, bytes, out); }));
    report("tma 16w x 1st x 12KB", k,
           time_it([&] { tma_kernel<16, 1, 12288><<<k, 16 * 32, kTmaSmemB>>>(buf, bytes, out); }));
    report("tma 4w x 4st x 12KB", k,
           time_it([&] { tma_kernel<4, 4, 12288><<<k, 4 * 32, kTmaSmemC>>>(buf, bytes, out); }));
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
