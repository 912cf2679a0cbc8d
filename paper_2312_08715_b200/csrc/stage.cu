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

// ------------------------------------------------------------ large batches
// One CTA reduces ~1,024 scores in a few microseconds but 1,048,576 in over a
// millisecond.  Above kGridMin scores the reduction runs over the grid:
// partial max / first argmax / non-finite count per kPart-element chunk,
// then per-chunk sums of exp(x - max), then one CTA combines the partials
// (chunk order), draws u, finds the chunk whose prefix crosses u * total and
// locates the index inside it with a block scan (the same 8 n eps boundary
// rule and sequential fallback as the single-CTA routine).  Draws for
// sample_many scan their chunk per thread, spread over several CTAs.
namespace {
constexpr long long kGridMin = 16384;
constexpr int kPart = 2048;  // elements per partial
constexpr int kPT = 256;     // threads of the partial kernels

struct Partials {
  double* max;
  long long* idx;
  unsigned int* nf;
  double* sum;
};

__host__ __device__ inline long long n_parts(long long n) { return (n + kPart - 1) / kPart; }

Partials partials_at(void* scratch, long long n) {
  const long long g = n_parts(n);
  char* b = static_cast<char*>(scratch);
  Partials p;
  p.max = reinterpret_cast<double*>(b);
  p.sum = reinterpret_cast<double*>(b + 8 * g);
  p.idx = reinterpret_cast<long long*>(b + 16 * g);
  p.nf = reinterpret_cast<unsigned int*>(b + 24 * g);
  return p;
}

template <int kThr>
__device__ __forceinline__ void block_best(double& bv, long long& bi, unsigned int& nf) {
  __shared__ double sv[kThr / 32];
  __shared__ long long si[kThr / 32];
  __shared__ unsigned int sn[kThr / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    sv[warp] = bv;
    si[warp] = bi;
    sn[warp] = nf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThr / 32; ++w) {
      if (better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
      nf += sn[w];
    }
  }
}

// fixed-order block sum (same tree for every launch): thread 0 gets it
template <int kThr>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sw[kThr / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThr / 32; ++w) t += sw[w];
  return t;
}

__global__ void __launch_bounds__(kPT)
part_max_kernel(const double* __restrict__ x, long long n, int stride, int col, Partials pt) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the scores' producer
  const long long a0 = (long long)blockIdx.x * kPart, a1 = min(n, a0 + kPart);
  double bv = -DBL_MAX * 2;
  long long bi = LLONG_MAX;
  unsigned int nf = 0;
  for (long long i = a0 + threadIdx.x; i < a1; i += kPT) {
    const double v = __ldcg(x + i * stride + col);
    nf += !isfinite(v);
    if (better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
  block_best<kPT>(bv, bi, nf);
  if (threadIdx.x == 0) {
    pt.max[blockIdx.x] = bv;
    pt.idx[blockIdx.x] = bi;
    pt.nf[blockIdx.x] = nf;
  }
}

// the global max over the partials (every CTA, a few hundred values)
__device__ __forceinline__ double global_max(const Partials& pt, long long g) {
  __shared__ double s_m;
  double m = -DBL_MAX * 2;
  for (long long c = threadIdx.x; c < g; c += blockDim.x) m = fmax(m, pt.max[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sw[32];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = sw[0];
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) t = fmax(t, sw[w]);
    s_m = t;
  }
  __syncthreads();
  return s_m;
}

// per-chunk sum of exp(x - max) (or of 1 when every score is -inf / NaN);
// `m_in` (sample_many) gives the max of an earlier reduction
__global__ void __launch_bounds__(kPT)
part_sum_kernel(const double* __restrict__ x, long long n, int stride, int col, Partials pt,
                const KStageResult* m_in) {
  const long long g = n_parts(n);
  double m;
  int all_zero;
  if (m_in) {
    m = m_in->max_score;
    all_zero = m_in->all_zero;
  } else {
    m = global_max(pt, g);
    all_zero = !isfinite(m);
  }
  const long long a0 = (long long)blockIdx.x * kPart, a1 = min(n, a0 + kPart);
  double s = 0.0;
  for (long long i = a0 + threadIdx.x; i < a1; i += kPT)
    s += all_zero ? 1.0 : exp(__ldcg(x + i * stride + col) - m);
  s = block_sum<kPT>(s);
  if (threadIdx.x == 0) pt.sum[blockIdx.x] = s;
}

// inclusive prefix of the partial sums in chunk order, by thread 0 (a few
// hundred additions), into shared memory when it fits, else recomputed
__global__ void __launch_bounds__(kT)
stage_finish_kernel(const double* __restrict__ x, long long n, int stride, int col,
                    Partials pt, unsigned long long* rng_state, KStageResult* out,
                    double* probs) {
  const long long g = n_parts(n);
  __shared__ double s_u, s_total, s_m;
  __shared__ long long s_chunk;
  __shared__ int s_allzero;
  const int tid = threadIdx.x;
  // max / first argmax / non-finite count over the partials
  double bv = -DBL_MAX * 2;
  long long bi = LLONG_MAX;
  unsigned int nf = 0;
  for (long long c = tid; c < g; c += kT) {
    if (better(pt.max[c], pt.idx[c], bv, bi)) {
      bv = pt.max[c];
      bi = pt.idx[c];
    }
    nf += pt.nf[c];
  }
  block_best<kT>(bv, bi, nf);
  if (tid == 0) {
    if (bi == LLONG_MAX) bi = 0;  // every entry NaN or -inf: index 0
    const int all_zero = !isfinite(bv);
    double total = 0.0;
    for (long long c = 0; c < g; ++c) total += pt.sum[c];
    out->argmax = (unsigned long long)bi;
    out->max_score = bv;
    out->n_nonfinite = nf;
    out->all_zero = all_zero;
    out->total = total;
    out->logsumexp = all_zero ? bv : bv + log(total);
    s_m = bv;
    s_total = total;
    s_allzero = all_zero;
    s_chunk = -1;
    if (rng_state) {
      const double u = rng_uniform(rng_state);
      s_u = u;
      double acc = 0.0;  // first chunk whose inclusive prefix exceeds u
      for (long long c = 0; c < g; ++c) {
        acc += pt.sum[c];
        if (u < acc / total) {
          s_chunk = c;
          break;
        }
      }
      if (s_chunk < 0) s_chunk = g - 1;
    }
  }
  __syncthreads();
  const double m = s_m, total = s_total;
  const int all_zero = s_allzero;
  if (probs)
    for (long long i = tid; i < n; i += kT)
      probs[i] = all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / total;
  if (!rng_state) return;
  // inside the chunk: two elements per thread, block scan of their
  // probabilities from the chunk's starting prefix
  const long long c = s_chunk, a0 = c * kPart, a1 = min(n, a0 + kPart);
  __shared__ double s_base;
  if (tid == 0) {
    double acc = 0.0;
    for (long long k = 0; k < c; ++k) acc += pt.sum[k];
    s_base = acc / total;
  }
  const long long e0 = a0 + 2 * (long long)tid, e1 = min(a1, e0 + 2);
  double p[2] = {0.0, 0.0};
  for (long long i = e0; i < e1; ++i)
    p[i - e0] = all_zero ? 1.0 / (double)n : exp(x[i * stride + col] - m) / total;
  __shared__ double s_scan[kT];
  s_scan[tid] = p[0] + p[1];
  __syncthreads();
  for (int o = 1; o < kT; o <<= 1) {
    const double y = tid >= o ? s_scan[tid - o] : 0.0;
    __syncthreads();
    s_scan[tid] += y;
    __syncthreads();
  }
  const double u = s_u;
  __shared__ int s_owner;
  if (tid == 0) s_owner = INT_MAX;
  __syncthreads();
  if (e0 < e1 && u < s_base + s_scan[tid]) atomicMin(&s_owner, tid);
  __syncthreads();
  if (tid != (s_owner == INT_MAX ? 0 : s_owner)) return;
  const double eps = 8.0 * (double)n * DBL_EPSILON;
  long long pick = -1;
  double margin = 0.0;
  if (s_owner != INT_MAX) {
    double acc = s_base + (tid ? s_scan[tid - 1] : 0.0), prev = acc;
    for (long long i = e0; i < e1; ++i) {
      prev = acc;
      acc += p[i - e0];
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
    pick = stage::sequential_pick(x, n, stride, col, m, all_zero, u);
  }
  out->sample = (unsigned long long)pick;
  out->sample_fallback = fallback;
  out->sample_logp = all_zero ? -log((double)n) : log(exp(x[pick * stride + col] - m) / total);
}

// draws for sample_many over the partial sums: the uniforms in stream order
// by one thread, then one draw per thread (bisection over the chunk prefix,
// a scan of one 2,048-element chunk), spread over ceil(k / 128) CTAs
__global__ void draw_uniforms_kernel(unsigned long long* rng_state, int k, double* u_buf) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int i = 0; i < k; ++i) u_buf[i] = rng_uniform(rng_state);
}

__global__ void __launch_bounds__(128)
draw_many_kernel(const double* __restrict__ x, long long n, int stride, int col,
                 const KStageResult* r, Partials pt, int k, const double* u_buf,
                 unsigned long long* out) {
  const long long g = n_parts(n);
  extern __shared__ double s_pre[];  // inclusive prefix of the chunk sums
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (long long c = 0; c < g; ++c) s_pre[c] = (acc += pt.sum[c]);
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const double m = r->max_score, tot = s_pre[g - 1];
  const int all_zero = r->all_zero;
  const double u = u_buf[j];
  long long lo = 0, hi = g - 1;
  while (lo < hi) {
    const long long mid = (lo + hi) / 2;
    if (u < s_pre[mid] / tot) hi = mid; else lo = mid + 1;
  }
  const double eps = 8.0 * (double)n * DBL_EPSILON;
  long long pick = -1;
  double margin = 0.0;
  {
    const long long a0 = lo * kPart, a1 = min(n, a0 + kPart);
    double acc = (lo ? s_pre[lo - 1] : 0.0) / tot, prev = acc;
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
  out[j] = (unsigned long long)pick;
}
}  // namespace

size_t stage_scratch_bytes(long long n) { return n > kGridMin ? 32ull * n_parts(n) + 64 : 0; }

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
    if (pick < 0 || !(margin > eps))  // near a boundary: the reference's order
      pick = stage::sequential_pick(x, n, stride, col, m, all_zero, u);
    out[k] = (unsigned long long)pick;
  }
}

cudaError_t launch_sample_many(const double* x, long long n, int stride, int col,
                               const KStageResult* r, unsigned long long* rng_state,
                               int n_samples, double* u_buf, unsigned long long* out,
                               cudaStream_t st, void* scratch) {
  const long long g = n_parts(n);
  if (n > kGridMin && scratch && 8ull * g <= 48 * 1024) {
    const Partials pt = partials_at(scratch, n);
    part_sum_kernel<<<(unsigned)g, kPT, 0, st>>>(x, n, stride, col, pt, r);
    draw_uniforms_kernel<<<1, 32, 0, st>>>(rng_state, n_samples, u_buf);
    draw_many_kernel<<<(n_samples + 127) / 128, 128, 8 * g, st>>>(x, n, stride, col, r, pt,
                                                                n_samples, u_buf, out);
    return cudaGetLastError();
  }
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
                                double* probs, cudaStream_t st, void* scratch) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at0[1];
  at0[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at0[0].val.programmaticStreamSerializationAllowed = 1;
  if (n > kGridMin && scratch) {
    const Partials pt = partials_at(scratch, n);
    const long long g = n_parts(n);
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(kPT);
    cfg.stream = st;
    cfg.attrs = at0;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, part_max_kernel, x, n, stride, col, pt);
    if (e != cudaSuccess) return e;
    part_sum_kernel<<<(unsigned)g, kPT, 0, st>>>(x, n, stride, col, pt, nullptr);
    stage_finish_kernel<<<1, kT, 0, st>>>(x, n, stride, col, pt, rng_state, out, probs);
    return cudaGetLastError();
  }
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
