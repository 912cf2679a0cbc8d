// track.cu -- track_camera's per-frame stage chain on the device
// (tracking.cpp:105-170, beam width 1).
//
// A frame runs refine_stages + 1 stages of a ppd^3 spherical lattice around
// the previous stage's argmax.  Every lattice coordinate a frame can visit is
// known up front per axis (stage s has ppd^(s+1) candidate values, a tree
// over the earlier picks), so the host computes them -- and the sin / cos of
// every azimuth and altitude with its own libm, exactly the values the
// reference's camera_pose_from_spherical would use -- once per frame.  The
// device then chains the stages without a host round trip:
//   cam_stage_kernel: the previous stage's argmax -- first index of the
//     strict maximum over the valid lattice points (tracking.cpp:132-134),
//     appended to the per-axis path -- then this stage's ppd^3 camera poses
//     from the tables (generative.cpp:35-59 arithmetic after the trig calls:
//     products, sqrt, divisions -- IEEE-exact, no FMA contraction, so
//     bitwise the host's);
//   the camera-mode score kernel;
//   cam_argmax_kernel: the last stage's argmax.
// The argmax kernels are launched with programmatic stream serialization, so
// they are resident when the score grid ends.
#include <cuda_runtime.h>

#include <cmath>

#include "b3d_kernels.cuh"

namespace b3d200 {
namespace {

constexpr double kHalfPiD = 1.5707963267948966;

__device__ __forceinline__ double dsq3(const double v[3]) {
  return v[0] * v[0] + (v[1] * v[1] + v[2] * v[2]);
}

__device__ __forceinline__ void dnormalize3(double v[3]) {
  const double n2 = dsq3(v);
  if (n2 > 0) {
    const double n = sqrt(n2);
    v[0] /= n;
    v[1] /= n;
    v[2] /= n;
  }
}

// Eigen Quaternion(const Matrix3&), m row-major (as b3d_capi.cpp quat_from_rot)
__device__ __forceinline__ void dquat_from_rot(const double m[9], double q[4]) {
  double t = m[0] + (m[4] + m[8]);
  if (t > 0) {
    t = sqrt(t + 1.0);
    q[0] = 0.5 * t;
    t = 0.5 / t;
    q[1] = (m[7] - m[5]) * t;
    q[2] = (m[2] - m[6]) * t;
    q[3] = (m[3] - m[1]) * t;
  } else {
    int i = 0;
    if (m[4] > m[0]) i = 1;
    if (m[8] > m[3 * i + i]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    double c[3];
    t = sqrt(m[3 * i + i] - m[3 * j + j] - m[3 * k + k] + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (m[3 * k + j] - m[3 * j + k]) * t;
    c[j] = (m[3 * j + i] + m[3 * i + j]) * t;
    c[k] = (m[3 * k + i] + m[3 * i + k]) * t;
    q[1] = c[0];
    q[2] = c[1];
    q[3] = c[2];
  }
}

// camera_pose_from_spherical (generative.cpp:35-59) given cos / sin of the
// altitude (ca, sa) and azimuth (cz, sz) from the host's libm
__device__ KPose camera_from_trig(double distance, double ca, double sa, double cz, double sz) {
  const double pos[3] = {distance * ca * cz, distance * ca * sz, distance * sa};
  double fwd[3] = {-pos[0], -pos[1], -pos[2]};
  dnormalize3(fwd);
  const double d = 0.0 * fwd[0] + (0.0 * fwd[1] + 1.0 * fwd[2]);
  double up[3] = {0.0 - d * fwd[0], 0.0 - d * fwd[1], 1.0 - d * fwd[2]};
  dnormalize3(up);
  const double down[3] = {-up[0], -up[1], -up[2]};
  const double right[3] = {down[1] * fwd[2] - down[2] * fwd[1],
                           down[2] * fwd[0] - down[0] * fwd[2],
                           down[0] * fwd[1] - down[1] * fwd[0]};
  const double m[9] = {right[0], down[0], fwd[0], right[1], down[1],
                       fwd[1],   right[2], down[2], fwd[2]};
  double q[4];
  dquat_from_rot(m, q);
  const double n2 = (q[1] * q[1] + q[2] * q[2]) + (q[3] * q[3] + q[0] * q[0]);
  if (n2 > 0) {
    const double n = sqrt(n2);
    for (int i = 0; i < 4; ++i) q[i] /= n;
  }
  return KPose{q[0], q[1], q[2], q[3], pos[0], pos[1], pos[2]};
}

// tab: 7 rows of n_tab doubles -- d, az, alt, cos(alt), sin(alt), cos(az),
// sin(az) -- per axis value; level s values start at off (the caller's).

// The reference's stage argmax (tracking.cpp:132-137): best = 0, then every
// i with scores[i] > scores[best] takes over.  A NaN never wins a comparison,
// so a NaN at index 0 keeps index 0 and a NaN elsewhere is never picked; keyed
// here as +inf / -inf, after which "first index of the strict maximum" over
// the keys is exactly the reference's pick.  Invalid (out-of-range) points
// score -inf (tracking.cpp:100-101).  Every thread of the CTA calls this; the
// result is valid in thread 0.
__device__ void stage_argmax(const double* __restrict__ scores,
                             const unsigned char* __restrict__ valid, int n, double& best_v,
                             int& best_i) {
  constexpr double kInf = __builtin_huge_val();
  double bv = -kInf;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = valid[i] ? scores[i] : -kInf;
    if (v != v) v = i == 0 ? kInf : -kInf;
    if (bi == 0x7fffffff || v > bv) {
      bv = v;
      bi = i;
    }
  }
  __shared__ double sv[32];
  __shared__ int si[32];
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi != 0x7fffffff && (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi))) {
      bv = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = sv[0];
    bi = si[0];
    for (int w = 1; w < (int)((blockDim.x + 31) / 32); ++w)
      if (si[w] != 0x7fffffff && (bi == 0x7fffffff || sv[w] > bv || (sv[w] == bv && si[w] < bi))) {
        bv = sv[w];
        bi = si[w];
      }
    best_v = bv;
    best_i = bi;
  }
}

// First index of the strict maximum over the valid points (invalid = -inf,
// start at index 0 as the reference's loop); appends the pick to the per-axis
// path; flags a stage whose best score is -inf.
__global__ void cam_argmax_kernel(const double* __restrict__ scores,
                                  const unsigned char* __restrict__ valid, int ppd,
                                  int* __restrict__ state /* path[3], best, err */) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the score kernel's results
  const int n = ppd * ppd * ppd;
  double bv;
  int bi;
  stage_argmax(scores, valid, n, bv, bi);
  if (threadIdx.x == 0) {
    // best score not finite (all -inf, or a NaN / +inf pick): the reference
    // throws (tracking.cpp:135-136)
    if (!isfinite(bv)) state[4] = 1;
    state[3] = bi;
    state[0] = state[0] * ppd + bi / (ppd * ppd);
    state[1] = state[1] * ppd + (bi / ppd) % ppd;
    state[2] = state[2] * ppd + bi % ppd;
  }
}

// One stage of the chain in one CTA: the previous stage's argmax (appended
// to the path; skipped for stage 0, which starts the path at the root), then
// this stage's ppd^3 camera poses.  Launched with programmatic stream
// serialization after the score kernel, so it is resident when that grid
// finishes and waits for its scores here.
__global__ void __launch_bounds__(1024)
cam_stage_kernel(const double* __restrict__ tab, int n_tab, int off, int ppd, int first,
                 const double* __restrict__ prev_scores, const unsigned char* __restrict__ valid_prev,
                 int* __restrict__ state, KPose* __restrict__ cams,
                 unsigned char* __restrict__ valid, KPose fallback) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n = ppd * ppd * ppd;
  __shared__ int s_path[3];
  if (first) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 8; ++i) state[i] = 0;
      s_path[0] = s_path[1] = s_path[2] = 0;
    }
  } else {
    double bv;
    int bi;
    stage_argmax(prev_scores, valid_prev, n, bv, bi);
    if (threadIdx.x == 0) {
      if (!isfinite(bv)) state[4] = 1;
      state[3] = bi;
      state[0] = state[0] * ppd + bi / (ppd * ppd);
      state[1] = state[1] * ppd + (bi / ppd) % ppd;
      state[2] = state[2] * ppd + bi % ppd;
      s_path[0] = state[0];
      s_path[1] = state[1];
      s_path[2] = state[2];
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int i = idx / (ppd * ppd), j = (idx / ppd) % ppd, k = idx % ppd;
    const int id = off + s_path[0] * ppd + i;
    const int iz = off + s_path[1] * ppd + j;
    const int ia = off + s_path[2] * ppd + k;
    const double dist = tab[id], alt = tab[2 * n_tab + ia];
    // score_pose (tracking.cpp:100-108): out-of-range points score -inf
    const bool ok = dist > 0 && alt > 0 && alt < kHalfPiD;
    valid[idx] = ok;
    cams[idx] = ok ? camera_from_trig(dist, tab[3 * n_tab + ia], tab[4 * n_tab + ia],
                                      tab[5 * n_tab + iz], tab[6 * n_tab + iz])
                   : fallback;
  }
}

}  // namespace

cudaError_t launch_cam_stage(const double* tab, int n_tab, int off, int ppd, int first,
                             const double* prev_scores, const unsigned char* valid_prev,
                             int* state, KPose* cams, unsigned char* valid,
                             const KPose& fallback, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(ppd * ppd * ppd >= 1024 ? 1024 : ((ppd * ppd * ppd + 31) / 32) * 32);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = first ? 0 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cam_stage_kernel, tab, n_tab, off, ppd, first,
                                           prev_scores, valid_prev, state, cams, valid, fallback);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_cam_argmax(const double* scores, const unsigned char* valid, int ppd,
                              int* state, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1024);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cam_argmax_kernel, scores, valid, ppd, state);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace b3d200
