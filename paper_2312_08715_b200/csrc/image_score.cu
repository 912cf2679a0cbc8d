// image_score.cu -- b3d_log_likelihood on the GPU: the reference's single
// image likelihood (b3d_capi.cpp:276-295) in fp64 with a deterministic,
// fixed-order reduction.  window >= 0: windowed_log_likelihood
// (likelihood.cpp:128-229); window < 0: full_log_likelihood over the two
// depth clouds (likelihood.cpp:82-104, geometry.cpp:54-70).  Not the hot
// path (one image per call); kept exact rather than fast.
#include <cstdint>

namespace b3d200 {

namespace {

constexpr int kB = 256;
constexpr int kMaxBlocks = 1024;
constexpr double kTwoPi = 6.283185307179586476925287;

struct ImgArgs {
  const float* obs;
  const float* rend;
  int W, H;
  double fx, fy, cx, cy;
  float far_f;
  double floor_term, inv_two_sigma2, one_minus_p, norm3, prefactor;
  int window;
};

__global__ void count_kernel(const float* rend, int n, float far_f, int* count) {
  int c = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    c += rend[i] < far_f;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__device__ __forceinline__ void backproject(const ImgArgs& a, int u, int v, float z,
                                            double o[3]) {
  const double zd = z;
  o[0] = (u - a.cx) * zd / a.fx;
  o[1] = (v - a.cy) * zd / a.fy;
  o[2] = zd;
}

// one log term per observed valid pixel; per-block fixed-order tree sums
__global__ void terms_kernel(ImgArgs a, const int* count, double* partial) {
  __shared__ double s[kB];
  const int n = a.W * a.H;
  const double coef = a.one_minus_p / (double)(*count) * a.norm3;
  double acc = 0.0;
  for (int i = blockIdx.x * kB + threadIdx.x; i < n; i += gridDim.x * kB) {
    const float oz = a.obs[i];
    if (!(oz < a.far_f)) continue;
    const int u = i % a.W, v = i / a.W;
    double o[3];
    backproject(a, u, v, oz, o);
    double S = 0.0;
    if (a.window >= 0) {
      const int w = a.window;
      const int v0 = max(0, v - w), v1 = min(a.H - 1, v + w);
      const int u0 = max(0, u - w), u1 = min(a.W - 1, u + w);
      for (int rv = v0; rv <= v1; ++rv)
        for (int ru = u0; ru <= u1; ++ru) {
          const float rz = a.rend[rv * a.W + ru];
          if (!(rz < a.far_f)) continue;
          double r[3];
          backproject(a, ru, rv, rz, r);
          const double dx = o[0] - r[0], dy = o[1] - r[1], dz = o[2] - r[2];
          S += exp(-(dx * dx + (dy * dy + dz * dz)) * a.inv_two_sigma2);
        }
    } else {
      for (int j = 0; j < n; ++j) {
        const float rz = a.rend[j];
        if (!(rz < a.far_f)) continue;
        double r[3];
        backproject(a, j % a.W, j / a.W, rz, r);
        const double dx = o[0] - r[0], dy = o[1] - r[1], dz = o[2] - r[2];
        S += exp(-(dx * dx + (dy * dy + dz * dz)) * a.inv_two_sigma2);
      }
    }
    acc += log(a.floor_term + coef * S);
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kB / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void final_kernel(const double* partial, int nb, double prefactor, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = prefactor;
    for (int b = 0; b < nb; ++b) t += partial[b];
    *out = t;
  }
}

}  // namespace

cudaError_t launch_image_loglik(const float* obs, const float* rend, int W, int H, double fx,
                                double fy, double cx, double cy, float far_f,
                                double p_outlier, double sigma, double sigma_max,
                                double volume, int window, int prefactor,
                                double* d_partial, double* d_out, int* d_count,
                                cudaStream_t st) {
  // asynchronous: the caller checked for an empty render on the host (the
  // reference's error) and reads d_out / d_count after its one sync;
  // d_partial holds image_loglik_partials(W * H) doubles
  const int n = W * H;
  cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  int nb = (n + kB - 1) / kB;
  if (nb > kMaxBlocks) nb = kMaxBlocks;
  count_kernel<<<nb, kB, 0, st>>>(rend, n, far_f, d_count);
  double* partial = d_partial;
  ImgArgs a;
  a.obs = obs;
  a.rend = rend;
  a.W = W;
  a.H = H;
  a.fx = fx;
  a.fy = fy;
  a.cx = cx;
  a.cy = cy;
  a.far_f = far_f;
  const double sigma2 = sigma * sigma;
  a.floor_term = p_outlier / volume;
  a.inv_two_sigma2 = 1.0 / (2.0 * sigma2);
  a.one_minus_p = 1.0 - p_outlier;
  a.norm3 = pow(kTwoPi * sigma2, -1.5);
  a.prefactor = prefactor == 0 ? log(sigma / sigma_max) : -log(sigma_max);
  a.window = window;
  terms_kernel<<<nb, kB, 0, st>>>(a, d_count, partial);
  final_kernel<<<1, 32, 0, st>>>(partial, nb, a.prefactor, d_out);
  return cudaGetLastError();
}

int image_loglik_partials(int n) {
  const int nb = (n + kB - 1) / kB;
  return nb > kMaxBlocks ? kMaxBlocks : nb;
}

}  // namespace b3d200
