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
#include "stage_common.cuh"

namespace b3d200 {

namespace {

constexpr int kT = 1024;
using stage::better;
using stage::rng_uniform;

}  // namespace

__global__ void __launch_bounds__(kT)
stage_reduce_kernel(const double* __restrict__ x, long long n, int stride, int col,
                    unsigned long long* rng_state, KStageResult* out, double* probs) {
  // programmatic dependent launch: this CTA may be resident before the
  // score kernel that produced x has finished (it is launched into the last
  // wave's idle SMs); wait for that grid's completion and memory here
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ stage::StageSmem<kT> sm;
  stage::block_stage_reduce<kT>(x, n, stride, col, rng_state, out, probs, sm);
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
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kT);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e =
      cudaLaunchKernelEx(&cfg, stage_reduce_kernel, x, n, stride, col, rng_state, out, probs);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_select_center(const KGrid& g, const KStageResult* r, int use_sample,
                                 KPose* center_out, cudaStream_t st) {
  select_center_kernel<<<1, 32, 0, st>>>(g, r, use_sample, center_out);
  return cudaGetLastError();
}

}  // namespace b3d200
