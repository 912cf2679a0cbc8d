// stage.cu -- per-stage reduction for sm_100a: max / argmax (first index on
// ties), fp64 sum exp(x - max), logsumexp, and one categorical draw with a
// device-resident xoshiro256** stream that reproduces the reference Rng
// bit for bit (rng.cpp:30-44), plus the grid-centre update that chains
// coarse-to-fine stages without a host round trip.
//
// Reference semantics: score_cells normalisation (inference.cpp:315-330),
// sample_categorical (inference.cpp:345-353), logsumexp (inference.cpp:16-23),
// argmax (tracking.cpp:132-134, inference.cpp:539-545).
#include <cfloat>
#include <climits>
#include <cstdint>

#include "b3d_kernels.cuh"
#include "posemath.cuh"

namespace b3d200 {

namespace {

constexpr int kT = 1024;
constexpr int kW = kT / 32;

__device__ __forceinline__ unsigned long long rotl64(unsigned long long x, int k) {
  return (x << k) | (x >> (64 - k));
}

// rng.cpp:30-44 (state[0] = seed, state[1..4] = s)
__device__ double rng_uniform(unsigned long long* st) {
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

__device__ __forceinline__ bool better(double x, long long i, double bx, long long bi) {
  // strict max, lowest index among equals; NaN never wins
  return x > bx || (x == bx && i < bi);
}

}  // namespace

__global__ void __launch_bounds__(kT)
stage_reduce_kernel(const double* __restrict__ x, long long n, int stride, int col,
                    unsigned long long* rng_state, KStageResult* out, double* probs) {
  __shared__ double s_v[kW];
  __shared__ long long s_i[kW];
  __shared__ double s_sum[kW];
  __shared__ double s_max;
  __shared__ int s_allzero;
  __shared__ double s_total;
  __shared__ double s_u;
  __shared__ int s_chunk;
  __shared__ double s_excl[kT];
  __shared__ unsigned int s_nonfinite;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_chunk = INT_MAX;
    s_nonfinite = 0;
  }

  // max / argmax
  double bv = -DBL_MAX * 2;  // -inf
  long long bi = LLONG_MAX;
  unsigned int nf = 0;
  for (long long i = tid; i < n; i += kT) {
    const double v = x[i * stride + col];
    nf += !isfinite(v);
    if (better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
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
    s_v[warp] = bv;
    s_i[warp] = bi;
    atomicAdd(&s_nonfinite, nf);
  }
  __syncthreads();
  if (tid == 0) {
    double v = s_v[0];
    long long i = s_i[0];
    for (int k = 1; k < kW; ++k)
      if (better(s_v[k], s_i[k], v, i)) {
        v = s_v[k];
        i = s_i[k];
      }
    if (i == LLONG_MAX) i = 0;  // every entry NaN or -inf: index 0 (tracking.cpp:132-134)
    s_max = v;
    s_allzero = !isfinite(v);
    out->argmax = (unsigned long long)i;
    out->max_score = v;
    out->n_nonfinite = s_nonfinite;
  }
  __syncthreads();
  const double m = s_max;
  const int all_zero = s_allzero;

  // sum exp(x - max) over contiguous chunks (chunk order = index order)
  const long long chunk = (n + kT - 1) / kT;
  const long long c0 = (long long)tid * chunk, c1 = min(n, c0 + chunk);
  double local = 0.0;
  if (!all_zero) {
    for (long long i = c0; i < c1; ++i) local += exp(x[i * stride + col] - m);
  } else {
    for (long long i = c0; i < c1; ++i) local += 1.0;
  }
  // inclusive block scan of chunk sums (warp shuffle + warp totals)
  double incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double wv = s_sum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= o) wv += y;
    }
    s_sum[lane] = wv;  // inclusive over warps
  }
  __syncthreads();
  const double warp_excl = warp ? s_sum[warp - 1] : 0.0;
  incl += warp_excl;
  s_excl[tid] = incl - local;
  if (tid == kT - 1) s_total = incl;
  __syncthreads();
  const double total = s_total;
  if (tid == 0) {
    out->all_zero = all_zero;
    out->total = total;
    out->logsumexp = all_zero ? m : m + log(total);
  }

  // optional normalised probabilities (CellScores)
  if (probs) {
    for (long long i = c0; i < c1; ++i)
      probs[i] = all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / total;
  }

  if (!rng_state) return;
  if (tid == 0) s_u = rng_uniform(rng_state);
  __syncthreads();
  const double u = s_u;
  // first chunk whose inclusive prefix exceeds u (in probability units)
  const double incl_p = incl / total;
  if (u < incl_p && c0 < c1) atomicMin(&s_chunk, tid);
  __syncthreads();
  if (tid == 0) {
    const double eps = 8.0 * (double)n * DBL_EPSILON;
    long long pick = -1;
    double margin = 0.0;
    if (s_chunk != INT_MAX) {
      const int t = s_chunk;
      const long long a0 = (long long)t * chunk, a1 = min(n, a0 + chunk);
      double acc = s_excl[t] / total;
      double prev = acc;
      for (long long i = a0; i < a1; ++i) {
        const double pi = all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / total;
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
    if (pick < 0 || !(margin > eps)) {
      // sequential CDF exactly as inference.cpp:345-353
      fallback = 1;
      double acc = 0.0;
      pick = n - 1;
      for (long long i = 0; i < n; ++i) {
        acc += all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / total;
        if (u < acc) {
          pick = i;
          break;
        }
      }
    }
    out->sample = (unsigned long long)pick;
    out->sample_fallback = fallback;
    out->sample_logp =
        all_zero ? -log((double)n) : log(exp(x[pick * stride + col] - m) / total);
  }
}

// n_samples categorical draws from one stage's posterior (scores already
// reduced into `r`: max, total): the reference Rng stream supplies
// u_0..u_{k-1} in order (thread 0, rng.cpp:30-44), then every draw locates
// its index in parallel by bisection over the per-chunk prefix sums and a
// scan of one chunk (sample_categorical semantics, inference.cpp:345-353),
// falling back to the sequential CDF when u is within 8 n eps of a boundary.
__global__ void __launch_bounds__(kT)
sample_many_kernel(const double* __restrict__ x, long long n, int stride, int col,
                   const KStageResult* r, unsigned long long* rng_state, int n_samples,
                   double* u_buf, unsigned long long* out) {
  __shared__ double s_incl[kT];
  const int tid = threadIdx.x;
  const double m = r->max_score, total = r->total;
  const int all_zero = r->all_zero;
  const long long chunk = (n + kT - 1) / kT;
  const long long c0 = (long long)tid * chunk, c1 = min(n, c0 + chunk);
  double local = 0.0;
  for (long long i = c0; i < c1; ++i)
    local += all_zero ? 1.0 : exp(x[i * stride + col] - m);
  // inclusive scan of chunk sums (simple Hillis-Steele in shared memory)
  s_incl[tid] = local;
  __syncthreads();
  for (int o = 1; o < kT; o <<= 1) {
    const double y = tid >= o ? s_incl[tid - o] : 0.0;
    __syncthreads();
    s_incl[tid] += y;
    __syncthreads();
  }
  if (tid == 0)
    for (int k = 0; k < n_samples; ++k) u_buf[k] = rng_uniform(rng_state);
  __syncthreads();
  const double tot = s_incl[kT - 1];  // equals r->total up to summation order
  (void)total;
  const double eps = 8.0 * (double)n * DBL_EPSILON;
  for (int k = tid; k < n_samples; k += kT) {
    const double u = u_buf[k];
    // first chunk t with u < incl[t] / tot
    int lo = 0, hi = kT - 1;
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      if (u < s_incl[mid] / tot) hi = mid; else lo = mid + 1;
    }
    long long pick = -1;
    double margin = 0.0;
    {
      const long long a0 = (long long)lo * chunk, a1 = min(n, a0 + chunk);
      double acc = (lo ? s_incl[lo - 1] : 0.0) / tot, prev = acc;
      for (long long i = a0; i < a1; ++i) {
        const double pi = all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / tot;
        prev = acc;
        acc += pi;
        if (u < acc) {
          pick = i;
          margin = fmin(acc - u, u - prev);
          break;
        }
      }
    }
    if (pick < 0 || !(margin > eps)) {
      double acc = 0.0;
      pick = n - 1;
      for (long long i = 0; i < n; ++i) {
        acc += all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / tot;
        if (u < acc) {
          pick = i;
          break;
        }
      }
    }
    out[k] = (unsigned long long)pick;
  }
}

cudaError_t launch_sample_many(const double* x, long long n, int stride, int col,
                               const KStageResult* r, unsigned long long* rng_state,
                               int n_samples, double* u_buf, unsigned long long* out,
                               cudaStream_t st) {
  sample_many_kernel<<<1, kT, 0, st>>>(x, n, stride, col, r, rng_state, n_samples, u_buf, out);
  return cudaGetLastError();
}

// Stage chaining: the next stage's grid centre is the pose of the chosen
// hypothesis of this stage (argmax or sample), computed on the device.
__global__ void select_center_kernel(KGrid g, const KStageResult* r, int use_sample,
                                     KPose* center_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long idx = (long long)(use_sample ? r->sample : r->argmax);
  KPose p;
  pm::grid_pose(g, idx, p);
  *center_out = p;
}

cudaError_t launch_stage_reduce(const double* x, long long n, int stride, int col,
                                unsigned long long* rng_state, KStageResult* out,
                                double* probs, cudaStream_t st) {
  stage_reduce_kernel<<<1, kT, 0, st>>>(x, n, stride, col, rng_state, out, probs);
  return cudaGetLastError();
}

cudaError_t launch_select_center(const KGrid& g, const KStageResult* r, int use_sample,
                                 KPose* center_out, cudaStream_t st) {
  select_center_kernel<<<1, 32, 0, st>>>(g, r, use_sample, center_out);
  return cudaGetLastError();
}

}  // namespace b3d200
