// Device Philox4x64-10 uniforms, bit-identical to the reference's
// rank_sliced_uniforms (sampling.py:112-124): numpy's Philox BitGenerator
// keyed by (seed, step), Generator.random((padded_batch, width)) row-major.
// numpy pre-increments the 256-bit counter before each block, so matrix
// element n = row * width + i is lane n % 4 of the block with counter
// (n / 4 + 1, 0, 0, 0), and a double is (x >> 11) * 2^-53.  Pinned by the
// known-answer test in SURVEY.md section 8(c) and tests/golden/philox.npz.
//
// The engine consumes row 0 of the matrix per session (engine.py:251-254),
// with seed = sampler.seed + seq (engine.py:234-235) and step = 2*round + 2 for
// acceptance (engine.py:499); seeds and steps are per-sequence device arrays
// so one launch serves a batch of sessions at different rounds.
#include "sdb_common.cuh"

namespace sdb {

constexpr uint64_t kPhiloxM0 = 0xD2E7470EE14C6C93ull, kPhiloxM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhiloxW0 = 0x9E3779B97F4A7C15ull, kPhiloxW1 = 0xBB67AE8584CAA73Bull;

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kPhiloxM0 * c[0], hi0 = __umul64hi(kPhiloxM0, c[0]);
    const uint64_t lo1 = kPhiloxM1 * c[2], hi1 = __umul64hi(kPhiloxM1, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
}

// One thread per 4-lane block of the requested row span; out[b][i].
__global__ void philox_uniforms_kernel(const int64_t *__restrict__ seeds, const int64_t *__restrict__ steps,
                                       int64_t row, int width, double *__restrict__ out) {
  const int b = blockIdx.y;
  const uint64_t k0 = (uint64_t)seeds[b], k1 = (uint64_t)steps[b];
  const uint64_t n0 = (uint64_t)row * (uint64_t)width;  // first matrix element of the row
  const uint64_t first_blk = n0 >> 2, last_blk = (n0 + width - 1) >> 2;
  const uint64_t blk = first_blk + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (width <= 0 || blk > last_blk) return;
  uint64_t c[4] = {blk + 1, 0, 0, 0};
  philox4x64_10(c, k0, k1);
#pragma unroll
  for (int lane = 0; lane < 4; ++lane) {
    const uint64_t n = blk * 4 + lane;
    if (n >= n0 && n < n0 + (uint64_t)width)
      out[(int64_t)b * width + (int64_t)(n - n0)] = (double)(c[lane] >> 11) * (1.0 / 9007199254740992.0);
  }
}

}  // namespace sdb

extern "C" int sdb_philox_uniforms(const int64_t *seeds, const int64_t *steps, int batch, int64_t row, int width,
                                   double *out, void *stream) {
  if (!seeds || !steps || !out || batch < 0 || batch > 65535 || row < 0 || width < 0) return SDB_E_INVALID;
  if (batch == 0 || width == 0) return SDB_OK;
  const uint64_t n0 = (uint64_t)row * (uint64_t)width;
  const uint64_t nblk = ((n0 + width - 1) >> 2) - (n0 >> 2) + 1;
  const int threads = 128;
  dim3 grid((unsigned)((nblk + threads - 1) / threads), (unsigned)batch);
  sdb::philox_uniforms_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(seeds, steps, row, width, out);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
