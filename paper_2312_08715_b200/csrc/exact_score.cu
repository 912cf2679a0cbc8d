// exact_score.cu -- batched fp64 likelihood over rendered depth images, in the
// reference's own per-pixel arithmetic.  The score path for the settings the
// fused fp32 epilogue cannot reproduce within tolerance:
//   * window < 0: the untruncated full_log_likelihood (likelihood.cpp:82-104)
//     that the inference seam selects when ModelConfig::windowed is false
//     (inference.cpp:51-56; b3d_infer's `window < 0`, b3d_capi.cpp:328-330);
//   * a tiny or zero outlier probability: with floor = p/V ~ 0 every term is
//     log(coef * S) and an observed pixel whose window holds only far-away
//     rendered points has S > 0 in fp64 but S = 0 after an fp32 exp, so the
//     fused kernel would turn a finite score into -inf.
// Hypotheses are rendered first (render-mode kernel, depth to HBM), then one
// CTA per image computes |y|, every observed pixel's window (or full) sum per
// distinct sigma in the reference's order (likelihood.cpp:192-218), and the
// per-noise totals with a fixed-order block reduction.  An empty render
// scores -inf with status 1 (the windowed reference throws,
// likelihood.cpp:159-160; the full form returns -inf, inference.cpp:54).
#include <cstdint>

#include "b3d_kernels.cuh"

namespace b3d200 {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ void backproject(const KExactArgs& a, int u, int v, float z,
                                            double o[3]) {
  const double zd = z;  // likelihood.cpp:150-155 / 118-124
  o[0] = (u - a.cx) * zd / a.fx;
  o[1] = (v - a.cy) * zd / a.fy;
  o[2] = zd;
}

// Eigen squaredNorm of a 3-vector: d0^2 + (d1^2 + d2^2)
__device__ __forceinline__ double sqnorm(const double o[3], const double r[3]) {
  const double dx = o[0] - r[0], dy = o[1] - r[1], dz = o[2] - r[2];
  return __dadd_rn(__dmul_rn(dx, dx), __dadd_rn(__dmul_rn(dy, dy), __dmul_rn(dz, dz)));
}

template <typename T>
__device__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kT / 32; ++w) s += red[w];
  __syncthreads();
  if (threadIdx.x == 0) red[0] = s;
  __syncthreads();
  const T r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kT) exact_score_kernel(KExactArgs a) {
  __shared__ double s_red[kT / 32];
  __shared__ int s_redi[kT / 32];
  __shared__ int s_off[kT / 32 + 1];
  const KExactLik& L = a.lik;
  const int npx = a.W * a.H;
  double* pts = a.pts ? a.pts + (size_t)blockIdx.x * 3 * npx : nullptr;
  for (long long h = blockIdx.x; h < a.n; h += gridDim.x) {
    const float* rend = a.rend + (size_t)h * npx;
    // |y| and, for the full form, the rendered cloud in row-major order
    // (depth_to_cloud, geometry.cpp:54-70)
    int count = 0;
    for (int base = 0; base < npx; base += kT) {
      const int i = base + threadIdx.x;
      const bool valid = i < npx && rend[i] < a.far_f;
      if (pts) {
        const unsigned b = __ballot_sync(0xffffffffu, valid);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_off[warp + 1] = __popc(b);
        __syncthreads();
        if (threadIdx.x == 0) {
          s_off[0] = 0;
          for (int w = 0; w < kT / 32; ++w) s_off[w + 1] += s_off[w];
        }
        __syncthreads();
        if (valid) {
          const int k = count + s_off[warp] + __popc(b & ((1u << lane) - 1u));
          backproject(a, i % a.W, i / a.W, rend[i], pts + 3 * (size_t)k);
        }
        count += s_off[kT / 32];
        __syncthreads();
      } else {
        count += valid;
      }
    }
    if (!pts) count = block_sum<int>(count, s_redi);
    if (count == 0) {
      if (threadIdx.x < L.n_noise)
        a.scores[h * a.ld + a.col0 + threadIdx.x] = -__longlong_as_double(0x7ff0000000000000ll);
      if (threadIdx.x == 0 && a.status) a.status[h] = 1;
      continue;
    }
    __syncthreads();  // pts visible to the whole CTA
    double coef[kMaxNoise];
#pragma unroll
    for (int e = 0; e < kMaxNoise; ++e)
      coef[e] = e < L.n_noise ? L.one_minus_p[e] / (double)count * L.norm3[e] : 0.0;
    double acc[kMaxNoise];
#pragma unroll
    for (int e = 0; e < kMaxNoise; ++e) acc[e] = 0.0;
    for (int i = threadIdx.x; i < npx; i += kT) {
      const float4 ob = a.obs[i];
      if (ob.w == 0.f) continue;  // ObservationCache skips sentinel pixels
      const float oz = ob.z;
      const int u = i % a.W, v = i / a.W;
      double o[3];
      backproject(a, u, v, oz, o);
      double S[kMaxSlots];
#pragma unroll
      for (int s = 0; s < kMaxSlots; ++s) S[s] = 0.0;
      if (L.window >= 0) {
        const int w = L.window;
        const int v0 = max(0, v - w), v1 = min(a.H - 1, v + w);
        const int u0 = max(0, u - w), u1 = min(a.W - 1, u + w);
        for (int rv = v0; rv <= v1; ++rv)
          for (int ru = u0; ru <= u1; ++ru) {
            const float rz = rend[rv * a.W + ru];
            if (!(rz < a.far_f)) continue;
            double r[3];
            backproject(a, ru, rv, rz, r);
            const double d2 = sqnorm(o, r);
#pragma unroll
            for (int s = 0; s < kMaxSlots; ++s)
              if (s < L.n_slots) S[s] += exp(-d2 * L.inv2s2[s]);
          }
      } else {
        for (int j = 0; j < count; ++j) {
          const double r[3] = {pts[3 * j], pts[3 * j + 1], pts[3 * j + 2]};
          const double d2 = sqnorm(o, r);
#pragma unroll
          for (int s = 0; s < kMaxSlots; ++s)
            if (s < L.n_slots) S[s] += exp(-d2 * L.inv2s2[s]);
        }
      }
#pragma unroll
      for (int e = 0; e < kMaxNoise; ++e)
        if (e < L.n_noise) acc[e] += log(L.floor_term[e] + coef[e] * S[L.slot_of[e]]);
    }
    for (int e = 0; e < L.n_noise; ++e) {
      const double t = block_sum<double>(acc[e], s_red);
      if (threadIdx.x == 0) a.scores[h * a.ld + a.col0 + e] = L.prefactor[e] + t;
    }
    if (threadIdx.x == 0 && a.status) a.status[h] = 0;
    __syncthreads();
  }
}

__global__ void fill_column_kernel(double* s, long long n, int ld, int col, double v) {
  for (long long h = blockIdx.x * (long long)blockDim.x + threadIdx.x; h < n;
       h += (long long)gridDim.x * blockDim.x)
    s[h * ld + col] = v;
}

}  // namespace

size_t exact_score_pts_bytes(int W, int H, int ctas) { return 24ull * W * H * ctas; }

cudaError_t launch_exact_score(const KExactArgs& a, int ctas, cudaStream_t st) {
  exact_score_kernel<<<ctas, kT, 0, st>>>(a);
  return cudaGetLastError();
}

namespace {
// per-pixel merges of renders of disjoint instance groups (camera scenes of
// more than one launch's instances): the z-test's minimum; keys are
// (depth bits << 32 | draw index), so a depth tie keeps the lower index
__global__ void min_merge_f32_kernel(float* dst, const float* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    if (src[i] < dst[i]) dst[i] = src[i];
}
__global__ void min_merge_u64_kernel(unsigned long long* dst, const unsigned long long* src,
                                     size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    if (src[i] < dst[i]) dst[i] = src[i];
}
// render-many's output convention (render_score.cuh, kOut): far sentinel,
// id -1 for the background
__global__ void keys_to_depth_ids_kernel(const unsigned long long* keys, size_t n, float far_f,
                                         float* depth, int32_t* ids) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const float z = __uint_as_float((unsigned int)(k >> 32));
    depth[i] = z < far_f ? z : far_f;
    if (ids) {
      const unsigned int d = (unsigned int)(k & 0xffffffffull);
      ids[i] = d == 0xffffffffu ? -1 : (int32_t)d;
    }
  }
}
unsigned grid_for(size_t n) {
  const size_t b = (n + 255) / 256;
  return (unsigned)(b < 4096 ? (b > 0 ? b : 1) : 4096);
}
}  // namespace

cudaError_t launch_min_merge_f32(float* dst, const float* src, size_t n, cudaStream_t st) {
  min_merge_f32_kernel<<<grid_for(n), 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}
cudaError_t launch_min_merge_u64(unsigned long long* dst, const unsigned long long* src,
                                 size_t n, cudaStream_t st) {
  min_merge_u64_kernel<<<grid_for(n), 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}
cudaError_t launch_keys_to_depth_ids(const unsigned long long* keys, size_t n, float far_f,
                                     float* depth, int32_t* ids, cudaStream_t st) {
  keys_to_depth_ids_kernel<<<grid_for(n), 256, 0, st>>>(keys, n, far_f, depth, ids);
  return cudaGetLastError();
}

cudaError_t launch_fill_column(double* s, long long n, int ld, int col, double v,
                               cudaStream_t st) {
  const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  fill_column_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(s, n, ld, col, v);
  return cudaGetLastError();
}

}  // namespace b3d200
