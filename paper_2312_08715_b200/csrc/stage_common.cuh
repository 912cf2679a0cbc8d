// stage_common.cuh -- the per-stage reduction as a block-level device
// routine: max / argmax (first index on ties), fp64 sum exp(x - max),
// logsumexp, optional normalised probabilities, and one categorical draw
// with the device xoshiro256** stream (rng.cpp:30-44).  Reference semantics:
// score_cells normalisation (inference.cpp:315-330), sample_categorical
// (inference.cpp:345-353), logsumexp (inference.cpp:16-23), argmax
// (tracking.cpp:132-134, inference.cpp:539-545).
#pragma once

#include <cfloat>
#include <climits>
#include <cstdint>

#include "b3d_kernels.cuh"

namespace b3d200 {
namespace stage {

__device__ __forceinline__ unsigned long long rotl64(unsigned long long x, int k) {
  return (x << k) | (x >> (64 - k));
}

// rng.cpp:30-44 (state[0] = seed, state[1..4] = s)
__device__ __forceinline__ double rng_uniform(unsigned long long* st) {
  unsigned long long* s = st + 1;
  const unsigned long long result = rotl64(s[1] * 5, 7) * 9;
  const unsigned long long t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return (double)(result >> 11) * 0x1.0p-53;
}

// The reference's draw, sequentially (score_cells + sample_categorical,
// inference.cpp:315-330 and 345-353): total = sum of exp(x - max) in index
// order, then the first i whose running sum of exp(x_i - max) / total exceeds
// u (the last index if none).  Used when u lies within 8 n eps of a boundary
// of the parallel CDF, where summation order could move the pick; it then
// agrees with the reference up to exp's last-ulp differences between this
// device's libm and the host's.
__device__ __noinline__ long long sequential_pick(const double* __restrict__ x, long long n,
                                                  int stride, int col, double m, int all_zero,
                                                  double u) {
  double total = 0.0;
  if (!all_zero)
    for (long long i = 0; i < n; ++i) total += exp(x[i * stride + col] - m);
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) {
    acc += all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / total;
    if (u < acc) return i;
  }
  return n - 1;
}

__device__ __forceinline__ bool better(double x, long long i, double bx, long long bi) {
  // strict max, lowest index among equals; NaN never wins
  return x > bx || (x == bx && i < bi);
}

// One CTA of kT threads, contiguous per-thread chunks (chunk order = index
// order), values of chunks of <= kCache elements kept in registers across
// the passes.  Used by stage_reduce_kernel (1,024 threads) and at the end of
// the score kernel by its last CTA (fused stage reduction).
constexpr int kCache = 4;

template <int kT>
struct StageSmem {
  double v[kT / 32];
  long long i[kT / 32];
  unsigned int nf[kT / 32];
  double sum[kT / 32];
  double max, u;
  int allzero, chunk;
};

template <int kT>
__device__ __forceinline__ void block_stage_reduce(const double* __restrict__ x, long long n,
                                                   int stride, int col,
                                                   unsigned long long* rng_state,
                                                   KStageResult* out, double* probs,
                                                   StageSmem<kT>& sm) {
  static_assert(kT % 32 == 0 && kT <= 1024, "one block of whole warps");
  constexpr int kW = kT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    sm.chunk = INT_MAX;
    if (rng_state) sm.u = rng_uniform(rng_state);  // the stage's one uniform()
  }
  const long long chunk = (n + kT - 1) / kT;
  const long long c0 = (long long)tid * chunk, c1 = min(n, c0 + chunk);
  const bool cached = chunk <= kCache;
  double xv[kCache];
#pragma unroll
  for (int j = 0; j < kCache; ++j)
    xv[j] = (cached && c0 + j < c1) ? __ldcg(x + (c0 + j) * stride + col) : 0.0;
  auto xat = [&](long long i) -> double {
    if (cached) {
      double v = xv[0];
#pragma unroll
      for (int j = 1; j < kCache; ++j)
        if (i - c0 == j) v = xv[j];
      return v;
    }
    return __ldcg(x + i * stride + col);
  };

  // max / argmax (strict max, lowest index among equals) and non-finite count
  double bv = -DBL_MAX * 2;  // -inf
  long long bi = LLONG_MAX;
  unsigned int nf = 0;
  for (long long i = c0; i < c1; ++i) {
    const double v = xat(i);
    nf += !isfinite(v);
    if (better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
  }
  if (lane == 0) {
    sm.v[warp] = bv;
    sm.i[warp] = bi;
    sm.nf[warp] = nf;
  }
  __syncthreads();
  if (warp == 0) {
    bv = lane < kW ? sm.v[lane] : -DBL_MAX * 2;
    bi = lane < kW ? sm.i[lane] : LLONG_MAX;
    nf = lane < kW ? sm.nf[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
      nf += __shfl_xor_sync(0xffffffffu, nf, o);
    }
    if (lane == 0) {
      if (bi == LLONG_MAX) bi = 0;  // every entry NaN or -inf: index 0 (tracking.cpp:132-134)
      sm.max = bv;
      sm.allzero = !isfinite(bv);
      out->argmax = (unsigned long long)bi;
      out->max_score = bv;
      out->n_nonfinite = nf;
    }
  }
  __syncthreads();
  const double m = sm.max;
  const int all_zero = sm.allzero;

  // sum exp(x - max): chunk sums, then an inclusive block scan (warp
  // shuffles + a scan of the warp totals)
  double local = 0.0;
  for (long long i = c0; i < c1; ++i) local += all_zero ? 1.0 : exp(xat(i) - m);
  double incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sm.sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double wv = lane < kW ? sm.sum[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= o) wv += y;
    }
    if (lane < kW) sm.sum[lane] = wv;  // inclusive over warps
  }
  __syncthreads();
  incl += warp ? sm.sum[warp - 1] : 0.0;
  const double total = sm.sum[kW - 1];
  if (tid == 0) {
    out->all_zero = all_zero;
    out->total = total;
    out->logsumexp = all_zero ? m : m + log(total);
  }

  // optional normalised probabilities (CellScores)
  if (probs) {
    for (long long i = c0; i < c1; ++i)
      probs[i] = all_zero ? 1.0 / (double)n : exp(xat(i) - m) / total;
  }

  if (!rng_state) return;
  const double u = sm.u;
  // first chunk whose inclusive prefix exceeds u (in probability units); its
  // thread scans it (inference.cpp:345-353), exactly when u is not within
  // 8 n eps of a CDF boundary, else the sequential CDF is redone
  if (u < incl / total && c0 < c1) atomicMin(&sm.chunk, tid);
  __syncthreads();
  const int owner = sm.chunk == INT_MAX ? 0 : sm.chunk;
  if (tid != owner) return;
  const double eps = 8.0 * (double)n * DBL_EPSILON;
  long long pick = -1;
  double margin = 0.0;
  if (sm.chunk != INT_MAX) {
    double acc = (incl - local) / total;
    double prev = acc;
    for (long long i = c0; i < c1; ++i) {
      const double pi = all_zero ? 1.0 / (double)n : exp(xat(i) - m) / total;
      prev = acc;
      acc += pi;
      if (u < acc) {
        pick = i;
        margin = fmin(acc - u, u - prev);
        break;
      }
    }
  }
  unsigned int fallback = 0;
  if (pick < 0 || !(margin > eps)) {  // near a boundary: the reference's order
    fallback = 1;
    pick = sequential_pick(x, n, stride, col, m, all_zero, u);
  }
  out->sample = (unsigned long long)pick;
  out->sample_fallback = fallback;
  out->sample_logp =
      all_zero ? -log((double)n) : log(exp(x[pick * stride + col] - m) / total);
}

}  // namespace stage
}  // namespace b3d200
