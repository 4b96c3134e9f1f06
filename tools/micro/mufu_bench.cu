// Throughput of the exp2 paths on one SM (results per clock per SM):
// MUFU.EX2 f32, ex2.approx.f16x2, ex2.approx.ftz.bf16x2, FFMA2.
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_bench.cu -o mufu && ./mufu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>

constexpr int ITERS = 4096;

__global__ void k_f32(float *out, long long *cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_f16x2(float *out, long long *cyc) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    __half2 h = __floats2half2_rn(-0.001f * threadIdx.x, -0.002f * i);
    a[i] = *reinterpret_cast<uint32_t *>(&h);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __low2float(*reinterpret_cast<__half2 *>(&a[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_bf16x2(float *out, long long *cyc) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(-0.001f * threadIdx.x, -0.002f * i);
    a[i] = *reinterpret_cast<uint32_t *>(&h);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __low2float(*reinterpret_cast<__nv_bfloat162 *>(&a[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma2(float *out, long long *cyc) {
  uint64_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = (uint64_t)__float_as_uint(0.001f * i) | ((uint64_t)__float_as_uint(0.5f) << 32);
  const uint64_t b = (uint64_t)__float_as_uint(0.999f) | ((uint64_t)__float_as_uint(0.999f) << 32);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[i]) : "l"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __uint_as_float((uint32_t)a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// mixed: f16x2 conversion path per 2 elements: cvt f32x2->f16x2, ex2 f16x2, unpack to f32 x2
__global__ void k_f16path(float *out, long long *cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  float acc = 0.f;
  uint32_t pk = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      uint32_t h;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i + 1]), "f"(a[i]));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
      float lo, hi;
      asm volatile("{.reg .f16 l, h;\nmov.b32 {l, h}, %2;\ncvt.f32.f16 %0, l;\ncvt.f32.f16 %1, h;}" : "=f"(lo), "=f"(hi) : "r"(h));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(hi), "f"(lo));
      acc += lo + hi;
      a[i] += 1e-7f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + pk;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// F2FP: cvt.rn.bf16x2.f32 alone (8 independent chains)
__global__ void k_cvt(float *out, long long *cyc) {
  float a[8];
  uint32_t pk = 0;
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
      pk ^= r;
      a[i] = __uint_as_float(__float_as_uint(a[i]) ^ (r & 1u));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a[0] + pk;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// the softmax mix per element pair: FFMA2 scale, 2 x MUFU.EX2, F2FP pack, FADD2 sum
__global__ void k_mix(float *out, long long *cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint64_t acc = 0;
  uint32_t pk = 0;
  const uint64_t sc = (uint64_t)__float_as_uint(0.125f) | ((uint64_t)__float_as_uint(0.125f) << 32);
  const uint64_t nm = (uint64_t)__float_as_uint(-1.f) | ((uint64_t)__float_as_uint(-1.f) << 32);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      uint64_t x;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[2 * e]), "f"(a[2 * e + 1]));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(sc), "l"(nm));
      float x0, x1, p0, p1;
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(x0));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(x1));
      uint32_t r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(p1), "f"(p0));
      pk ^= r;
      uint64_t pp;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(pp) : "f"(p0), "f"(p1));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pp));
      a[2 * e] = p0;
      a[2 * e + 1] = p1;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((uint32_t)acc) + pk;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// same mix without the F2FP pack
__global__ void k_mix_nocvt(float *out, long long *cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint64_t acc = 0;
  const uint64_t sc = (uint64_t)__float_as_uint(0.125f) | ((uint64_t)__float_as_uint(0.125f) << 32);
  const uint64_t nm = (uint64_t)__float_as_uint(-1.f) | ((uint64_t)__float_as_uint(-1.f) << 32);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      uint64_t x;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[2 * e]), "f"(a[2 * e + 1]));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(sc), "l"(nm));
      float x0, x1, p0, p1;
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(x0));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(x1));
      uint64_t pp;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(pp) : "f"(p0), "f"(p1));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pp));
      a[2 * e] = p0;
      a[2 * e + 1] = p1;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((uint32_t)acc);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the softmax mix with a packed bf16x2 exp2: FFMA2 scale, F2FP pack of x,
// one MUFU.EX2 bf16x2, unpack (shift / and) and FADD2 sum in fp32
__global__ void k_mix_bf16(float *out, long long *cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint64_t acc = 0;
  uint32_t pk = 0;
  const uint64_t sc = (uint64_t)__float_as_uint(0.125f) | ((uint64_t)__float_as_uint(0.125f) << 32);
  const uint64_t nm = (uint64_t)__float_as_uint(-1.f) | ((uint64_t)__float_as_uint(-1.f) << 32);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      uint64_t x;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[2 * e]), "f"(a[2 * e + 1]));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(sc), "l"(nm));
      float x0, x1;
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
      uint32_t h;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h));
      pk ^= h;
      const float p0 = __uint_as_float(h << 16), p1 = __uint_as_float(h & 0xffff0000u);
      uint64_t pp;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(pp) : "f"(p0), "f"(p1));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pp));
      a[2 * e] += 1e-7f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((uint32_t)acc) + pk;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char *name, K kern, double results_per_thread_iter, int threads) {
  float *out;
  long long *cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  kern<<<148, threads>>>(out, cyc);
  kern<<<148, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  double res = results_per_thread_iter * ITERS * threads;
  printf("%-10s threads %4d: %.2f results/clk/SM  (%.0f cycles)\n", name, threads, res / c, c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run("ex2.f32", k_f32, 8, t);
    run("ex2.f16x2", k_f16x2, 16, t);
    run("ex2.bf16x2", k_bf16x2, 16, t);
    run("ffma2", k_ffma2, 16, t);
    run("f16path", k_f16path, 16, t);
    run("cvt.bf16x2", k_cvt, 8, t);
    run("mix", k_mix, 8, t);
    run("mix-nocvt", k_mix_nocvt, 8, t);
    run("mix-bf16", k_mix_bf16, 8, t);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
