// Drop-in, reference-precision (float64) sampling ops on the device:
//   target_dist  (sampling.py:87-102 with softmax_lse numcore.py:41-60 and
//                 top_p_mask sampling.py:52-72)
//   mss_verify   (sampling.py:149-202 with sample_from 105-109 and
//                 check_dist 43-49) on explicit distributions.
// These serve the numpy-in/numpy-out API of paper_2508_08192_b200.sampling;
// the batched perf path is accept.cu.
#include <math.h>

#include "sdb_common.cuh"

namespace sdb {

constexpr int kF64Threads = 512;

__device__ double f64_block_sum(double v, double *red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kF64Threads / 32 ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

__device__ double f64_block_max(double v, double *red) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kF64Threads / 32 ? red[lane] : -INFINITY;
    v = warp_max(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

// One CTA per row.
__global__ void __launch_bounds__(kF64Threads) target_dist_f64_kernel(const double *__restrict__ logits,
                                                                      const uint8_t *__restrict__ allowed, int vocab,
                                                                      double temperature, double top_p,
                                                                      double *__restrict__ dist,
                                                                      int32_t *__restrict__ err) {
  __shared__ double red[32];
  __shared__ int s_flag, s_arg;
  const int64_t r = blockIdx.x;
  const double *row = logits + r * vocab;
  const uint8_t *al = allowed ? allowed + r * vocab : nullptr;
  double *out = dist + r * vocab;
  if (threadIdx.x == 0) {
    s_flag = 0;
    s_arg = INT_MAX;
  }
  __syncthreads();
  auto val = [&](int i) { return (al && !al[i]) ? -INFINITY : row[i]; };
  bool nan = false, any_allowed = !al;
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) {
    double v = val(i);
    nan |= row[i] != row[i] && (!al || al[i]);
    if (al && al[i]) any_allowed = true;
    mx = fmax(mx, v);
  }
  if (__syncthreads_or(nan)) {
    if (threadIdx.x == 0) atomicOr(err, SDB_ERR_NAN);
    return;
  }
  if (!__syncthreads_or(any_allowed)) {
    if (threadIdx.x == 0) atomicOr(err, SDB_ERR_NO_ALLOWED);
    return;
  }
  mx = f64_block_max(mx, red);
  if (temperature == 0.0) {
    // exact argmax, lowest index on ties (numcore.py:51-55)
    for (int i = threadIdx.x; i < vocab; i += kF64Threads)
      if (val(i) == mx) atomicMin(&s_arg, i);
    __syncthreads();
    for (int i = threadIdx.x; i < vocab; i += kF64Threads) out[i] = i == s_arg ? 1.0 : 0.0;
    return;
  }
  // softmax(x / T) with lse (numcore.py:56-60)
  const double m = mx / temperature;
  double s = 0.0;
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) s += exp(val(i) / temperature - m);
  s = f64_block_sum(s, red);
  const double lse = m + log(s);
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) out[i] = exp(val(i) / temperature - lse);
  __syncthreads();
  if (!(top_p < 1.0)) return;
  // top_p_mask: keep the smallest (prob desc, index asc) prefix whose cumsum
  // reaches top_p - 1e-12.  The cut value theta is found by bisection on the
  // (monotone, non-negative) float64 bit patterns; ties at theta are taken in
  // index order with the reference's sequential cumsum.
  double psum = 0.0;
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) psum += out[i];
  const double total = f64_block_sum(psum, red);
  const double tau = top_p - 1e-12;
  unsigned long long lo = 0ull, hi = 0ull;  // largest theta with mass(p >= theta) >= tau
  {
    double pm = 0.0;
    for (int i = threadIdx.x; i < vocab; i += kF64Threads) pm = fmax(pm, out[i]);
    hi = (unsigned long long)__double_as_longlong(f64_block_max(pm, red));
  }
  if (total < tau) {
    lo = 0ull;  // never reaches tau: keep everything (cutoff clamped to V-1)
  } else {
    // invariant: mass(>= lo) >= tau; answer in [lo, hi]
    while (lo < hi) {
      unsigned long long mid = lo + (hi - lo + 1) / 2;
      double th = __longlong_as_double((long long)mid);
      double ms = 0.0;
      for (int i = threadIdx.x; i < vocab; i += kF64Threads)
        if (out[i] >= th) ms += out[i];
      ms = f64_block_sum(ms, red);
      if (ms >= tau)
        lo = mid;
      else
        hi = mid - 1;
    }
  }
  const double theta = __longlong_as_double((long long)lo);
  double above = 0.0;
  for (int i = threadIdx.x; i < vocab; i += kF64Threads)
    if (out[i] > theta) above += out[i];
  above = f64_block_sum(above, red);
  __shared__ int s_cut_idx;
  if (threadIdx.x == 0) {
    // ties at theta in index order, sequential cumsum as np.cumsum does
    int cut = vocab - 1;
    double c = above;
    bool done = total < tau;
    if (!done) {
      for (int i = 0; i < vocab; ++i) {
        if (out[i] == theta) {
          c += theta;
          if (c >= tau) {
            cut = i;
            break;
          }
        }
      }
    }
    s_cut_idx = done ? vocab - 1 : cut;
  }
  __syncthreads();
  const int cut_idx = s_cut_idx;
  const bool keep_all = total < tau;
  double kept_mass = 0.0;
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) {
    double p = out[i];
    bool k = keep_all || p > theta || (p == theta && i <= cut_idx);
    if (k) kept_mass += p;
  }
  kept_mass = f64_block_sum(kept_mass, red);
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) {
    double p = out[i];
    bool k = keep_all || p > theta || (p == theta && i <= cut_idx);
    out[i] = k ? p / kept_mass : 0.0;
  }
}

// Single CTA: the MSS walk with explicit float64 distributions.
__global__ void __launch_bounds__(kF64Threads) mss_verify_f64_kernel(
    const int32_t *__restrict__ parent, const int32_t *__restrict__ tokens, int n_nodes, int vocab,
    const double *__restrict__ node_dists, const double *__restrict__ target_dists,
    const double *__restrict__ uniforms, int n_uniforms, int32_t *__restrict__ out_path,
    int64_t *__restrict__ out_scalars, double *__restrict__ residual, int32_t *__restrict__ err) {
  __shared__ double red[32];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  // check_dist on every target distribution (sampling.py:167)
  for (int r = 0; r <= n_nodes; ++r) {
    const double *d = target_dists + (int64_t)r * vocab;
    double s = 0.0;
    bool neg = false;
    for (int i = threadIdx.x; i < vocab; i += kF64Threads) {
      s += d[i];
      neg |= d[i] < 0.0;
    }
    s = f64_block_sum(s, red);
    if (__syncthreads_or(neg) || fabs(s - 1.0) > 1e-9) {
      if (threadIdx.x == 0) atomicOr(err, SDB_ERR_BAD_DIST);
      return;
    }
  }
  int used = 0, cur = -1, len = 0;
  const double *p = target_dists;
  const double *anchor = p;
  while (true) {
    bool descended = false;
    for (int c = 0; c < n_nodes; ++c) {
      if (parent[c] != cur) continue;
      const int t = tokens[c];
      const double *q = node_dists + (int64_t)c * vocab;
      if (used >= n_uniforms) {
        if (threadIdx.x == 0) atomicOr(err, SDB_ERR_UNIFORMS);
        return;
      }
      const double u = uniforms[used++];
      const double qt = q[t], pt = p[t];
      const bool accept = qt <= 0.0 ? pt > 0.0 : u < fmin(1.0, pt / qt);
      if (accept) {
        if (threadIdx.x == 0) out_path[len] = c;
        ++len;
        p = target_dists + (int64_t)(1 + c) * vocab;
        anchor = p;
        cur = c;
        descended = true;
        break;
      }
      double ms = 0.0;
      for (int i = threadIdx.x; i < vocab; i += kF64Threads) {
        double v = fmax(p[i] - q[i], 0.0);
        residual[i] = v;
        ms += v;
      }
      ms = f64_block_sum(ms, red);
      if (ms <= 1e-12) {
        p = anchor;
      } else {
        for (int i = threadIdx.x; i < vocab; i += kF64Threads) residual[i] /= ms;
        __syncthreads();
        p = residual;
      }
    }
    if (!descended) break;
  }
  if (used >= n_uniforms) {
    if (threadIdx.x == 0) atomicOr(err, SDB_ERR_UNIFORMS);
    return;
  }
  const double u = uniforms[used++];
  // check_dist(p) (sample_from -> check_dist)
  double s = 0.0;
  bool neg = false;
  for (int i = threadIdx.x; i < vocab; i += kF64Threads) {
    s += p[i];
    neg |= p[i] < 0.0;
  }
  s = f64_block_sum(s, red);
  if (__syncthreads_or(neg) || fabs(s - 1.0) > 1e-9) {
    if (threadIdx.x == 0) atomicOr(err, SDB_ERR_BAD_DIST);
    return;
  }
  if (p != residual) {
    for (int i = threadIdx.x; i < vocab; i += kF64Threads) residual[i] = p[i];
    __syncthreads();
  }
  // inverse CDF: warps own contiguous segments
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kF64Threads / 32;
  const int seg = (vocab + nw - 1) / nw;
  const int s0 = warp * seg, s1 = min(vocab, s0 + seg);
  double ws = 0.0;
  for (int i = s0 + lane; i < s1; i += 32) ws += residual[i];
  ws = warp_sum(ws);
  __shared__ double segsum[32];
  __shared__ double s_prefix;
  __shared__ int s_seg, s_tok;
  if (lane == 0) segsum[warp] = ws;
  __syncthreads();
  if (threadIdx.x == 0) {
    double cum = 0.0;
    int k = 0;
    for (; k < nw - 1; ++k) {
      if (cum + segsum[k] > u) break;
      cum += segsum[k];
    }
    s_prefix = cum;
    s_seg = k;
    s_tok = -1;
  }
  __syncthreads();
  if (warp == s_seg && lane == 0) {
    // sequential within the segment, as np.cumsum + searchsorted(side='right')
    double cum = s_prefix;
    int found = -1;
    for (int i = s0; i < s1; ++i) {
      cum += residual[i];
      if (cum > u) {
        found = i;
        break;
      }
    }
    s_tok = found;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tok = s_tok < 0 ? vocab - 1 : s_tok;
    out_scalars[0] = len;
    out_scalars[1] = min(tok, vocab - 1);
    out_scalars[2] = used;
  }
}

}  // namespace sdb

extern "C" int sdb_target_dist_f64(const double *logits, const uint8_t *allowed, int64_t rows, int vocab,
                                   double temperature, double top_p, double *dist, int32_t *err, void *stream) {
  if (!logits || !dist || !err || rows < 0 || vocab < 1) return SDB_E_INVALID;
  if (temperature < 0.0 || !(top_p > 0.0) || top_p > 1.0) return SDB_E_INVALID;
  if (rows == 0) return SDB_OK;
  sdb::target_dist_f64_kernel<<<(unsigned)rows, sdb::kF64Threads, 0, sdb::as_stream(stream)>>>(
      logits, allowed, vocab, temperature, top_p, dist, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_mss_verify_f64(const int32_t *parent, const int32_t *tokens, int n_nodes, int vocab,
                                  const double *node_dists, const double *target_dists, const double *uniforms,
                                  int n_uniforms, int32_t *out_path, int64_t *out_scalars, double *residual,
                                  int32_t *err, void *stream) {
  if (n_nodes < 0 || vocab < 1 || !target_dists || !uniforms || !out_scalars || !residual || !err)
    return SDB_E_INVALID;
  if (n_nodes > 0 && (!parent || !tokens || !node_dists || !out_path)) return SDB_E_INVALID;
  sdb::mss_verify_f64_kernel<<<1, sdb::kF64Threads, 0, sdb::as_stream(stream)>>>(
      parent, tokens, n_nodes, vocab, node_dists, target_dists, uniforms, n_uniforms, out_path, out_scalars,
      residual, err);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
