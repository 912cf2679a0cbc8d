// render_score.cu -- auxiliary kernels (observation cache, base-scene terms)
// and the host-side launch helpers of the fused render/score kernel
// (render_score.cuh; score variants instantiated in rs_score_w*.cu).
#include "render_score.cuh"

#include <map>
#include <mutex>
#include <tuple>

namespace b3d200 {
B3D_RS_SCORE_KERNELS(extern, 0)
B3D_RS_SCORE_KERNELS(extern, 1)
B3D_RS_SCORE_KERNELS(extern, 2)
B3D_RS_SCORE_KERNELS(extern, 3)
B3D_RS_SCORE_KERNELS(extern, -1)
B3D_RS_CAM_KERNELS(extern)
B3D_RS_SCORE_KERNELS2(extern, 1, true)
B3D_RS_SCORE_KERNELS2(extern, 2, true)
B3D_RS_SCORE_KERNELS2(extern, 4, true)

// ---------------------------------------------------------------- base scene
// Padded depth-bit image of the base scene (halo of `pad` background pixels)
// so the S_base window sums below run the exact same tap code as the
// hypothesis kernel.
__global__ void base_pad_kernel(const unsigned long long* keys, int W, int H, int pad,
                                unsigned int* out) {
  const int PW = W + 2 * pad, PH = H + 2 * pad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < PW * PH; i += gridDim.x * blockDim.x) {
    const int v = i / PW - pad, u = i % PW - pad;
    out[i] = (u >= 0 && u < W && v >= 0 && v < H) ? (unsigned int)(keys[(size_t)v * W + u] >> 32)
                                                  : __float_as_uint(kBgDepth);
  }
}

// S_base(p, slot): the window sums of every observed pixel against the base
// image alone (likelihood.cpp:198-214 restricted to the fixed scene).
__global__ void sbase_kernel(const KParams p, const unsigned int* padded, int pad,
                             float* sbase) {
  Region rg;
  rg.u0 = 0;
  rg.v0 = 0;
  rg.u1 = p.W - 1;
  rg.v1 = p.H - 1;
  rg.ox = -pad;
  rg.oy = -pad;
  rg.rw = p.W + 2 * pad;
  rg.rh = p.H + 2 * pad;
  const size_t npx = (size_t)p.W * p.H;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (int)npx; i += gridDim.x * blockDim.x) {
    const int v = i / p.W, u = i % p.W;
    const float4 o = p.obs[i];
    float S[kMaxSlots];
#pragma unroll
    for (int sl = 0; sl < kMaxSlots; ++sl) S[sl] = 0.f;
    if (o.w != 0.f) window_sums_rt<false>(p, padded, rg, u, v, o, S);
    for (int sl = 0; sl < p.lik.n_slots; ++sl) sbase[(size_t)sl * npx + i] = S[sl];
  }
}

// G_e(l) = sum over observed pixels of log(floor_e + coef_e(|y| = e^l) * S_base)
// at the kCheb Chebyshev nodes of [lo, hi] (fp64, fixed-order reduction).
__global__ void gnode_kernel(const KParams p, const float* sbase, double lo, double hi,
                             double* G) {
  __shared__ double s_red[256];
  const int k = blockIdx.x, e = blockIdx.y;
  const double node = 0.5 * (lo + hi) + 0.5 * (hi - lo) * cos(3.14159265358979323846 * (k + 0.5) / kCheb);
  const double y = exp(node);
  const double coef = p.lik.one_minus_p[e] / y * p.lik.norm3[e];
  const double fl = p.lik.floor_term[e];
  const size_t npx = (size_t)p.W * p.H;
  const float* sb = sbase + (size_t)p.lik.slot_of[e] * npx;
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < npx; i += blockDim.x)
    if (p.obs[i].w != 0.f) acc += log(fl + coef * (double)sb[i]);
  s_red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) G[e * kCheb + k] = s_red[0];
}

cudaError_t launch_base_terms(const KParams& p, const unsigned long long* base_keys,
                              unsigned int* padded, float* sbase, double* G, cudaStream_t st) {
  const int pad = p.lik.window;
  const int n_pad = (p.W + 2 * pad) * (p.H + 2 * pad);
  base_pad_kernel<<<(n_pad + 255) / 256, 256, 0, st>>>(base_keys, p.W, p.H, pad, padded);
  const int npx = p.W * p.H;
  sbase_kernel<<<(npx + 255) / 256, 256, 0, st>>>(p, padded, pad, sbase);
  gnode_kernel<<<dim3(kCheb, p.lik.n_noise), 256, 0, st>>>(p, sbase, p.cheb_lo, p.cheb_hi, G);
  return cudaGetLastError();
}

// Observation cache (likelihood.cpp:106-126) as per-pixel fp32 points plus
// the valid count M.  count[0] = M; count[1] = a block counter that wraps
// back to 0 (atomicInc); count[2 + b] = block b's partial: the last block to
// finish sums the partials, so no memset precedes the launch.
__global__ void obs_prepare_kernel(const float* depth, int W, int H, float far_f, float fcx,
                                   float fcy, float inv_fx, float inv_fy, float4* out,
                                   int* count) {
  // a score kernel launched behind this one with programmatic serialization
  // may start now; it waits (griddepcontrol.wait) before reading the cache
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int c = 0;
  const int n = W * H;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float z = depth[i];
    const int u = i % W, v = i / W;
    if (z < far_f) {
      out[i] = make_float4(((float)u - fcx) * inv_fx * z, ((float)v - fcy) * inv_fy * z, z, 1.f);
      ++c;
    } else {
      out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  c = warp_sum_i(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    count[2 + blockIdx.x] = s_cnt;
    __threadfence();
    if (atomicInc(reinterpret_cast<unsigned int*>(count + 1), gridDim.x - 1) == gridDim.x - 1) {
      __threadfence();
      int m = 0;
      for (unsigned int b = 0; b < gridDim.x; ++b) m += __ldcg(count + 2 + b);
      count[0] = m;
    }
  }
}

// Host-side launch helpers (declared in b3d_capi.cpp).
template <bool kIds, bool kScore, bool kOut, int kWin, bool kS1, bool kCam = false>
static auto pick_vs(bool vs) {
  return vs ? render_score_kernel<kIds, kScore, kOut, true, kWin, kS1, kCam>
            : render_score_kernel<kIds, kScore, kOut, false, kWin, kS1, kCam>;
}

// Score kernels are instantiated per window radius 0..3 (else generic) and
// for one / several distinct sigmas -- one small kernel per launch keeps the
// hot instruction footprint down; render kernels once.
template <bool kIds, bool kScore, bool kOut>
static auto pick_kernel(bool vs, int window, int n_noise, bool cam = false) {
  if constexpr (kScore && !kIds) {
    const bool s1 = n_noise == 1;
    if (cam) {  // camera mode: the bench-tracking windows (1, 2, 4), else generic
      switch (window) {
        case 1: return s1 ? pick_vs<kIds, kScore, kOut, 1, true, true>(vs) : pick_vs<kIds, kScore, kOut, 1, false, true>(vs);
        case 2: return s1 ? pick_vs<kIds, kScore, kOut, 2, true, true>(vs) : pick_vs<kIds, kScore, kOut, 2, false, true>(vs);
        case 4: return s1 ? pick_vs<kIds, kScore, kOut, 4, true, true>(vs) : pick_vs<kIds, kScore, kOut, 4, false, true>(vs);
        default: return s1 ? pick_vs<kIds, kScore, kOut, -1, true, true>(vs) : pick_vs<kIds, kScore, kOut, -1, false, true>(vs);
      }
    }
    switch (window) {
      case 0: return s1 ? pick_vs<kIds, kScore, kOut, 0, true>(vs) : pick_vs<kIds, kScore, kOut, 0, false>(vs);
      case 1: return s1 ? pick_vs<kIds, kScore, kOut, 1, true>(vs) : pick_vs<kIds, kScore, kOut, 1, false>(vs);
      case 2: return s1 ? pick_vs<kIds, kScore, kOut, 2, true>(vs) : pick_vs<kIds, kScore, kOut, 2, false>(vs);
      case 3: return s1 ? pick_vs<kIds, kScore, kOut, 3, true>(vs) : pick_vs<kIds, kScore, kOut, 3, false>(vs);
      default: return s1 ? pick_vs<kIds, kScore, kOut, -1, true>(vs) : pick_vs<kIds, kScore, kOut, -1, false>(vs);
    }
  } else {
    (void)window;
    (void)n_noise;
    return cam ? pick_vs<kIds, kScore, kOut, -1, false, true>(vs)
               : pick_vs<kIds, kScore, kOut, -1, false>(vs);
  }
}

// Host-side launch bookkeeping is cached: the dynamic shared-memory limit is
// set once per (kernel, size) and occupancy / static shared memory are
// queried once -- per call these CUDA runtime queries cost tens of us, as
// much as a small batch's kernel (device ordinal is part of the key).
namespace {
std::mutex g_launch_mu;
std::map<std::tuple<const void*, int, size_t>, int> g_occupancy;  // -> blocks/SM
std::map<std::pair<const void*, int>, size_t> g_smem_limit;        // -> current limit

cudaError_t ensure_smem_limit(const void* kern, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_launch_mu);
  size_t& cur = g_smem_limit[{kern, dev}];
  if (cur >= smem) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}
}  // namespace

template <bool kIds, bool kScore, bool kOut>
cudaError_t launch_render_score(const KParams& p, int grid, size_t smem, cudaStream_t st,
                                bool pdl) {
  auto kern = pick_kernel<kIds, kScore, kOut>(p.nv <= p.vcap, p.lik.window, p.lik.n_noise,
                                              p.cams != nullptr);
  cudaError_t e = ensure_smem_limit(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  if (p.n_hyp <= 0) return cudaSuccess;
  if (pdl) {  // camera mode: the kernel waits (griddepcontrol.wait) before reading inputs
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)std::min<long long>(grid, p.n_hyp));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  kern<<<(int)std::min<long long>(grid, p.n_hyp), kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

template <bool kIds, bool kScore, bool kOut>
cudaError_t occupancy_render_score(int* blocks, size_t smem, bool vs) {
  auto kern = pick_kernel<kIds, kScore, kOut>(vs, 1, 1);  // same resources for every variant
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), dev, smem);
  {
    std::lock_guard<std::mutex> lk(g_launch_mu);
    auto it = g_occupancy.find(key);
    if (it != g_occupancy.end()) {
      *blocks = it->second;
      return cudaSuccess;
    }
  }
  cudaError_t e = ensure_smem_limit(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kern, kThreads, smem);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_launch_mu);
    g_occupancy[key] = *blocks;
  }
  return e;
}

template <bool kIds, bool kScore, bool kOut>
size_t static_smem_render_score() {
  static const size_t cached = [] {
    size_t mx = 0;
    for (int vs = 0; vs < 2; ++vs)
      for (int cam = 0; cam < 2; ++cam) {
        cudaFuncAttributes a{};
        if (cudaFuncGetAttributes(&a, pick_kernel<kIds, kScore, kOut>(vs, 1, 1, cam)) !=
            cudaSuccess)
          return (size_t)8192;
        if (a.sharedSizeBytes > mx) mx = a.sharedSizeBytes;
      }
    return mx;
  }();
  return cached;
}

#define B3D_INST(I, S, O)                                                                 \
  template cudaError_t launch_render_score<I, S, O>(const KParams&, int, size_t,         \
                                                    cudaStream_t, bool);                 \
  template cudaError_t occupancy_render_score<I, S, O>(int*, size_t, bool);              \
  template size_t static_smem_render_score<I, S, O>();
B3D_INST(false, true, false)
B3D_INST(true, false, true)
B3D_INST(false, false, true)
#undef B3D_INST

constexpr int kObsBlocks = 1184;
size_t obs_count_ints() { return 2 + kObsBlocks; }  // count buffer (zeroed once)

cudaError_t launch_obs_prepare(const float* depth, int W, int H, float far_f, float fcx,
                               float fcy, float inv_fx, float inv_fy, float4* out, int* count,
                               cudaStream_t st) {
  const int n = W * H;
  int grid = (n + 255) / 256;
  if (grid > kObsBlocks) grid = kObsBlocks;
  obs_prepare_kernel<<<grid, 256, 0, st>>>(depth, W, H, far_f, fcx, fcy, inv_fx, inv_fy, out,
                                           count);
  return cudaGetLastError();
}

int render_score_threads() { return kThreads; }

size_t render_score_staging_bytes(int nt) { return (void)nt, sizeof(WarpQ) * kWarps; }

}  // namespace b3d200
