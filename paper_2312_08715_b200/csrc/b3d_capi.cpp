// b3d_capi.cpp -- C++ host layer and C ABI (include/b3d_b200.h) of the
// B200-native pose-enumeration hot path.
//
// Mirrors the reference's C API conventions (proj/src/capi/b3d_capi.cpp):
// exceptions are converted to b3d_status by guarded() (b3d_capi.cpp:33-48),
// the message goes to a thread-local string (b3d_capi.cpp:22,118), and the
// argument checks reuse the reference's messages where one exists.
#include "b3d_b200.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <chrono>
#include <limits>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>
#include <atomic>
#include <thread>

#include "b3d_kernels.cuh"

namespace b3d200 {

// kernels (render_score.cu, stage.cu, image_score.cu)
template <bool kIds, bool kScore, bool kOut>
cudaError_t launch_render_score(const KParams& p, int grid, size_t smem, cudaStream_t st,
                                bool pdl = false);
template <bool kIds, bool kScore, bool kOut>
cudaError_t occupancy_render_score(int* blocks, size_t smem, bool vs);
template <bool kIds, bool kScore, bool kOut>
size_t static_smem_render_score();
size_t render_score_staging_bytes(int nt);
// track.cu
cudaError_t launch_cam_argmax(const double* scores, const unsigned char* valid, int ppd,
                              int* state, cudaStream_t st);
cudaError_t launch_cam_stage(const double* tab, int n_tab, int off, int ppd, int first,
                             const double* prev_scores, const unsigned char* valid_prev,
                             int* state, KPose* cams, unsigned char* valid,
                             const KPose& fallback, cudaStream_t st);
// mesh_build.cu
cudaError_t voxel_to_mesh_device(const int* d_vox, unsigned long long n, double res,
                                 const double origin[3], double* d_verts, unsigned* d_tris,
                                 unsigned long long* n_vertices, unsigned long long* n_triangles,
                                 cudaStream_t stream);

cudaError_t launch_obs_prepare(const float* depth, int W, int H, float far_f, float fcx,
                               float fcy, float inv_fx, float inv_fy, float4* out,
                               int* count, cudaStream_t st);
cudaError_t launch_exact_score(const KExactArgs& a, int ctas, cudaStream_t st);
cudaError_t launch_min_merge_f32(float* dst, const float* src, size_t n, cudaStream_t st);
cudaError_t launch_min_merge_u64(unsigned long long* dst, const unsigned long long* src,
                                 size_t n, cudaStream_t st);
cudaError_t launch_keys_to_depth_ids(const unsigned long long* keys, size_t n, float far_f,
                                     float* depth, int32_t* ids, cudaStream_t st);
cudaError_t launch_shard_barrier(const KBarrier& b, cudaStream_t st);
cudaError_t launch_exchange_emulation(unsigned long long* sig, double* arr, int n_ranks,
                                      int rounds, int double_buffered,
                                      unsigned long long hold_ns, unsigned int* errors,
                                      cudaStream_t st);
cudaError_t launch_copy_to_peers(const double* src, long long n_elems, double* const* peers,
                                 int n_peers, long long offset, long long cap, cudaStream_t st);
cudaError_t launch_fill_column(double* s, long long n, int ld, int col, double v, cudaStream_t st);
size_t exact_score_pts_bytes(int W, int H, int ctas);
size_t stage_scratch_bytes(long long n);  // stage.cu: grid-wide reduction partials
size_t obs_count_ints();                 // render_score.cu: obs_prepare count buffer
cudaError_t launch_stage_reduce(const double* x, long long n, int stride, int col,
                                unsigned long long* rng_state, KStageResult* out,
                                double* probs, cudaStream_t st, void* scratch);
cudaError_t launch_sample_many(const double* x, long long n, int stride, int col,
                               const KStageResult* r, unsigned long long* rng_state,
                               int n_samples, double* u_buf, unsigned long long* out,
                               cudaStream_t st, void* scratch);
cudaError_t launch_select_center(const KGrid& g, const KStageResult* r, int use_sample,
                                 KPose* center_out, cudaStream_t st);
cudaError_t launch_base_terms(const KParams& p, const unsigned long long* base_keys,
                              unsigned int* padded, float* sbase, double* G, cudaStream_t st);
cudaError_t launch_image_loglik(const float* obs, const float* rend, int W, int H,
                                double fx, double fy, double cx, double cy, float far_f,
                                double p_outlier, double sigma, double sigma_max,
                                double volume, int window, int prefactor,
                                double* d_partial, double* d_out, int* d_count,
                                cudaStream_t st);
int image_loglik_partials(int n);

// ------------------------------------------------------------------ errors
enum class ErrorCode { invalid = 1, config = 2, io = 3, numeric = 4 };

struct Error : std::runtime_error {
  Error(ErrorCode c, const std::string& w) : std::runtime_error(w), code(c) {}
  ErrorCode code;
};

[[noreturn]] inline void fail(ErrorCode c, const std::string& m) { throw Error(c, m); }
inline void require(bool cond, ErrorCode c, const std::string& m) {
  if (!cond) fail(c, m);
}
inline void check(bool cond, const char* msg) { require(cond, ErrorCode::invalid, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(ErrorCode::numeric, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------- pose math
// geometry.cpp:26-31 inverse (host side, once per call); the per-hypothesis
// compose runs on the device (posemath.cuh).  Same scalar Eigen order.
KPose pose_inverse(const KPose& p) {
  double w = p.qw, x = -p.qx, y = -p.qy, z = -p.qz;
  const double n2 = (x * x + y * y) + (z * z + w * w);
  if (n2 > 0) {
    const double n = std::sqrt(n2);
    w /= n;
    x /= n;
    y /= n;
    z /= n;
  }
  const double v[3] = {p.tx, p.ty, p.tz};
  double uv0 = y * v[2] - z * v[1];
  double uv1 = z * v[0] - x * v[2];
  double uv2 = x * v[1] - y * v[0];
  uv0 += uv0;
  uv1 += uv1;
  uv2 += uv2;
  const double c0 = y * uv2 - z * uv1;
  const double c1 = z * uv0 - x * uv2;
  const double c2 = x * uv1 - y * uv0;
  KPose o;
  o.qw = w;
  o.qx = x;
  o.qy = y;
  o.qz = z;
  o.tx = -(v[0] + w * uv0 + c0);
  o.ty = -(v[1] + w * uv1 + c1);
  o.tz = -(v[2] + w * uv2 + c2);
  return o;
}

// b3d_capi.cpp:66-74 (from_c(b3d_pose)): unit-norm check, then normalize
KPose pose_from_c(const b3d_pose& p) {
  const double n2 = (p.qx * p.qx + p.qy * p.qy) + (p.qz * p.qz + p.qw * p.qw);
  check(std::abs(std::sqrt(n2) - 1.0) < 1e-6, "pose rotation must be a unit quaternion");
  KPose o{p.qw, p.qx, p.qy, p.qz, p.tx, p.ty, p.tz};
  const double n = std::sqrt(n2);
  if (n2 > 0) {
    o.qw /= n;
    o.qx /= n;
    o.qy /= n;
    o.qz /= n;
  }
  return o;
}

// geometry.cpp:38-44
void validate_intrinsics(const b3d_intrinsics& k) {
  check(k.fx > 0 && k.fy > 0, "intrinsics: focal lengths must be positive");
  check(k.width > 0 && k.height > 0, "intrinsics: image dimensions must be positive");
  check(k.cx >= 0 && k.cx < k.width && k.cy >= 0 && k.cy < k.height,
        "intrinsics: principal point outside image bounds");
  check(k.near_m > 0 && k.near_m < k.far_m, "intrinsics: require 0 < near < far");
}

// likelihood.cpp:30-35
double visible_volume(const b3d_intrinsics& k) {
  const double di = (k.far_m * k.far_m * k.far_m - k.near_m * k.near_m * k.near_m) / 3.0;
  return di * (k.width / k.fx) * (k.height / k.fy);
}

// ---------------------------------------------------------- device buffers
// Page-locked host staging (track_camera's per-stage camera / score copies).
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cuda_check(cudaMallocHost(&p, n), "cudaMallocHost");
    bytes = n;
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cuda_check(cudaMalloc(&p, n), "cudaMalloc");
    bytes = n;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Page-locked host memory: copies from it are stream-ordered and need no
// synchronisation before the call returns.
bool is_pinned_host(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Mesh {
  DevBuf verts, tris;
  int nv = 0, nt = 0;
  // +1 / -1: closed and outward / inward wound (back-face culling sign), 0:
  // not closed (no culling)
  int cull = 0;
  // score-mode order (KParams::tris_s): axis classes sorted by plane offset
  DevBuf tris_s, plane_off, plane_end;
  int cls_start[8] = {0};
  int plane_begin[8] = {0};
  double radius = 0;  // max |vertex| (model frame): bounds the projected region
};

// Score-mode triangle order (b3d_kernels.cuh KParams::tris_s).  A triangle
// whose three vertices share one coordinate k exactly (voxel faces) has the
// winding normal +-e_k; with the mesh's winding sign w (closed_mesh_cull_sign)
// its outward normal is s e_k, s = w * sign(n_k), class 2k + (s < 0), plane
// offset o = s * a_k.  Everything else is class 6.
void build_score_order(const double* v, const uint32_t* t, uint64_t nt, int wsign, Mesh& m) {
  struct Item {
    int cls;
    double off;
    uint32_t idx;
  };
  std::vector<Item> items(nt);
  for (uint64_t i = 0; i < nt; ++i) {
    const double* a = v + 3 * t[3 * i];
    const double* b = v + 3 * t[3 * i + 1];
    const double* cc = v + 3 * t[3 * i + 2];
    Item it{6, 0.0, (uint32_t)i};
    if (wsign != 0)
      for (int k = 0; k < 3; ++k) {
        if (a[k] != b[k] || a[k] != cc[k]) continue;
        const int k1 = (k + 1) % 3, k2 = (k + 2) % 3;
        const double nk = (b[k1] - a[k1]) * (cc[k2] - a[k2]) - (b[k2] - a[k2]) * (cc[k1] - a[k1]);
        if (nk == 0) break;
        const int s = (nk > 0 ? 1 : -1) * wsign;
        it.cls = 2 * k + (s < 0);
        it.off = s * a[k];
        break;
      }
    items[i] = it;
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& x, const Item& y) {
    return x.cls != y.cls ? x.cls < y.cls : x.off < y.off;
  });
  std::vector<uint32_t> tri4(4 * nt);
  std::vector<double> poff;
  std::vector<int> pend;
  int cls = -1;
  for (uint64_t i = 0; i < nt; ++i) {
    const Item& it = items[i];
    for (int j = 0; j < 3; ++j) tri4[4 * i + j] = t[3 * it.idx + j];
    tri4[4 * i + 3] = it.idx;
    while (cls < it.cls) {
      ++cls;
      m.cls_start[cls] = (int)i;
      m.plane_begin[cls] = (int)poff.size();
    }
    if (it.cls < 6) {
      if ((int)poff.size() == m.plane_begin[cls] || poff.back() != it.off) {
        poff.push_back(it.off);
        pend.push_back(0);
      }
      pend.back() = (int)i + 1;
    }
  }
  while (cls < 7) {
    ++cls;
    m.cls_start[cls] = (int)nt;
    m.plane_begin[cls] = (int)poff.size();
  }
  m.tris_s.ensure(16 * nt);
  cuda_check(cudaMemcpy(m.tris_s.p, tri4.data(), 16 * nt, cudaMemcpyHostToDevice), "cudaMemcpy");
  m.plane_off.ensure(8 * (poff.size() + 1));
  m.plane_end.ensure(4 * (pend.size() + 1));
  if (!poff.empty()) {
    cuda_check(cudaMemcpy(m.plane_off.p, poff.data(), 8 * poff.size(), cudaMemcpyHostToDevice),
               "cudaMemcpy");
    cuda_check(cudaMemcpy(m.plane_end.p, pend.data(), 4 * pend.size(), cudaMemcpyHostToDevice),
               "cudaMemcpy");
  }
}

// Back faces of a closed mesh never decide a pixel's depth: a ray through a
// pixel centre inside a back face leaves the solid there, so it entered it
// at a strictly nearer front face covering the same pixel.
// Closed = every directed edge (a, b) is matched by as many (b, a); the
// winding sign is the sign of the enclosed volume.  For a triangle with all
// vertices at z > 0, the screen area2 of renderer.cpp:63 has the sign of
// a . ((b - a) x (c - a)), positive for a face turned away from the camera
// when the mesh is outward wound.
int closed_mesh_cull_sign(const double* v, const uint32_t* t, uint64_t nt) {
  std::unordered_map<uint64_t, int> edges;
  edges.reserve(3 * nt);
  for (uint64_t i = 0; i < nt; ++i)
    for (int j = 0; j < 3; ++j) {
      const uint64_t a = t[3 * i + j], b = t[3 * i + (j + 1) % 3];
      if (a == b) return 0;
      edges[(a << 32) | b] += 1;
    }
  for (const auto& kv : edges) {
    const uint64_t rev = (kv.first << 32) | (kv.first >> 32);
    auto it = edges.find(rev);
    if (it == edges.end() || it->second != kv.second) return 0;
  }
  double vol = 0.0, scale = 0.0;
  for (uint64_t i = 0; i < nt; ++i) {
    const double* a = v + 3 * t[3 * i];
    const double* b = v + 3 * t[3 * i + 1];
    const double* c = v + 3 * t[3 * i + 2];
    vol += a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) +
           a[2] * (b[0] * c[1] - b[1] * c[0]);
    scale += std::fabs(a[0]) + std::fabs(a[1]) + std::fabs(a[2]);
  }
  scale /= (double)nt;
  if (!(std::fabs(vol) > 1e-9 * scale * scale * scale)) return 0;
  return vol > 0 ? 1 : -1;
}

}  // namespace b3d200

using namespace b3d200;

// one fused launch's noise entries: output columns [col0, col0 + lik.n_noise)
struct LikChunk {
  int col0 = 0;
  KLik lik{};
  KExactLik ex{};
};

// likelihood settings of a score call (make_spec)
struct LikSpec {
  int n_cols = 0;             // output columns = noise entries
  int window = 0;             // < 0: untruncated likelihood
  bool exact = false;         // fp64 image path (exact_score.cu)
  std::vector<int> gated;     // columns outside the noise support: -inf
  std::vector<LikChunk> chunks;
  // one fused launch writes every column in place
  bool single() const {
    return !exact && gated.empty() && chunks.size() == 1 && chunks[0].lik.n_noise == n_cols;
  }
};

struct b3d_gpu_context {
  int device = 0;
  int sm_count = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  bool has_camera = false;
  b3d_intrinsics k{};
  KPose w2c{1, 0, 0, 0, 0, 0, 0};
  std::vector<std::unique_ptr<Mesh>> meshes;
  bool has_obs = false;
  DevBuf obs_depth, obs_pts, obs_count;
  bool has_lik = false;
  KLik lik{};                 // first fused chunk (window for launch plans)
  LikSpec spec;               // score-cells seam (gated)
  LikSpec cam_spec;           // windowed_log_likelihood_multi seam (camera paths)
  std::string cam_spec_err;   // why cam_spec is unusable ("" = usable)
  DevBuf chunk_scores, ex_depth, ex_pts;
  double sigma_max = 0.1;
  int prefactor = B3D_PREFACTOR_PRINTED;
  DevBuf zscratch, vscratch;
  DevBuf in_stage, out_stage, out_stage2, rot_stage, result, rng;
  DevBuf c2f_scores, c2f_rot, c2f_centers, c2f_results;
  PinnedBuf pin_cams, pin_scores;  // track_camera / enumerate_poses staging
  PinnedBuf trk_tab_pin, trk_state_pin;  // track_camera device chain: tables, picks
  DevBuf stage_part;                     // grid-wide stage reduction partials
  DevBuf trk_tab, trk_state, trk_valid;
  // fixed scene (compose_render)
  bool has_base = false;
  DevBuf base_keys, base_tmp, base_pad, sbase, gnodes, cheb, spin;
  int base_valid = 0;
  uint64_t gen = 0;  // bumped by every setter: cached launch graphs check it
  // b3d_gpu_enumerate_observed with page-locked inputs: the whole step
  // (uploads, observation cache, score kernel, stage reduction, read-back)
  // captured once into a CUDA graph and replayed while its inputs stay
  struct E2E {
    bool valid = false;
    int warm = 0;
    cudaGraphExec_t exec = nullptr;
    std::vector<const void*> key;
  } e2e;
  PinnedBuf pin_rng;
  DevBuf e2e_rng;
  uint32_t base_draw = 0;
  bool culling = true;  // b3d_gpu_set_culling
  // b3d_gpu_set_score_peers: fused score all-gather targets
  double* score_peers[8] = {nullptr};
  int n_score_peers = 0;
  long long score_peer_offset = 0;
  long long score_peer_cap = 0;
  // camera mode scene (b3d_gpu_set_camera_scene): concatenated instances
  // camera scene (b3d_gpu_set_camera_scene): instances in draw order, in
  // groups of up to kMaxInst (one concatenated mesh each; draw indices
  // continue across groups).  One group: the fused camera-mode kernels; more:
  // per-group renders merged per pixel, then the fp64 image likelihood.
  struct CamGroup {
    std::unique_ptr<Mesh> mesh;
    int n = 0;
    int v0[kMaxInst + 1] = {0};
    KPose pose[kMaxInst];
    uint32_t draw_base = 0;
  };
  std::vector<CamGroup> cam_groups;
  DevBuf cam_tmp, cam_keys;
  long long obs_version = 0, base_version = 0;
  std::string base_terms_key;
};

namespace {

thread_local std::string g_last_error;

b3d_status to_status(const Error& e) {
  switch (e.code) {
    case ErrorCode::config: return B3D_ERROR_CONFIG;
    case ErrorCode::io: return B3D_ERROR_IO;
    case ErrorCode::numeric: return B3D_ERROR_NUMERIC;
    default: return B3D_ERROR;
  }
}

template <typename F>
b3d_status guarded(F&& fn) {
  try {
    fn();
    return B3D_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return to_status(e);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return B3D_ERROR;
  } catch (...) {
    g_last_error = "unknown error";
    return B3D_ERROR;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void* stage_scratch(b3d_gpu_context* ctx, long long n) {
  const size_t b = stage_scratch_bytes(n);
  if (!b) return nullptr;
  ctx->stage_part.ensure(b);
  return ctx->stage_part.p;
}

void require_ready(const b3d_gpu_context* ctx, bool need_obs, bool need_lik) {
  check(ctx != nullptr, "bad arguments");
  require(ctx->has_camera, ErrorCode::invalid, "gpu context: intrinsics not set");
  if (need_obs) require(ctx->has_obs, ErrorCode::invalid, "gpu context: observation not set");
  if (need_lik)
    require(ctx->has_lik, ErrorCode::invalid, "gpu context: likelihood settings not set");
}

const Mesh& get_mesh(const b3d_gpu_context* ctx, int32_t id) {
  require(id >= 0 && static_cast<size_t>(id) < ctx->meshes.size(), ErrorCode::invalid,
          "gpu context: unknown mesh id");
  return *ctx->meshes[id];
}

// Copies `bytes` from a host pointer into the staging buffer (or passes a
// device pointer through).
const void* stage_in(b3d_gpu_context* ctx, DevBuf& buf, const void* src, size_t bytes,
                     bool* was_host) {
  if (is_device_ptr(src)) {
    *was_host = false;
    return src;
  }
  *was_host = true;
  buf.ensure(bytes);
  cuda_check(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream),
             "cudaMemcpyAsync H2D");
  return buf.p;
}

struct LaunchPlan {
  long long zstride = 0;
  int grid = 0;
  int cap = 0;
  size_t smem = 0;
  int vcap = 0;
  int zcap = 0;
};

// Bound on a hypothesis's region (pixels incl. the likelihood halo) when its
// model-to-world pose lies within `spread` (m) of `center`: the mesh fits in
// a sphere of radius R, whose projection at depth z has half-width
// <= f R / (z - R).  0 = no useful bound (object may reach the near plane).
double sq3(const double v[3]) { return v[0] * v[0] + (v[1] * v[1] + v[2] * v[2]); }
double cam_z(const b3d_gpu_context* ctx, double tx, double ty, double tz) {
  const KPose& c = ctx->w2c;  // camera-frame depth of a model-to-world translation
  return 2 * (c.qx * c.qz - c.qw * c.qy) * tx + 2 * (c.qy * c.qz + c.qw * c.qx) * ty +
         (1 - 2 * (c.qx * c.qx + c.qy * c.qy)) * tz + c.tz;
}
size_t region_hint_z(const b3d_gpu_context* ctx, const Mesh& m, double zc, int window) {
  const double zmin = zc - m.radius;
  if (!(zmin > std::max(ctx->k.near_m, 1e-6)) || !(m.radius > 0)) return 0;
  const int pad = 2 * std::max(window, 0);
  const double su = 2.0 * ctx->k.fx * m.radius / zmin + 3 + 2 * pad;
  const double sv = 2.0 * ctx->k.fy * m.radius / zmin + 3 + 2 * pad;
  const double px = 1.15 * su * sv;
  return px < 1e9 ? (size_t)px : 0;
}
size_t region_hint(const b3d_gpu_context* ctx, const Mesh& m, const KPose& center, double spread,
                   int window) {
  return region_hint_z(ctx, m, cam_z(ctx, center.tx, center.ty, center.tz) - spread, window);
}
// explicit host poses: the nearest of up to 4,096 evenly spaced samples
// (hypotheses nearer still just take the scratch z-buffer)
size_t region_hint_poses(const b3d_gpu_context* ctx, const Mesh& m, const b3d_pose* poses,
                         uint64_t n, int window) {
  double zc = std::numeric_limits<double>::infinity();
  const uint64_t step = std::max<uint64_t>(1, n / 4096);
  for (uint64_t i = 0; i < n; i += step)
    zc = std::min(zc, cam_z(ctx, poses[i].tx, poses[i].ty, poses[i].tz));
  return std::isfinite(zc) ? region_hint_z(ctx, m, zc, window) : 0;
}

template <bool kIds, bool kScore, bool kOut>
LaunchPlan plan_launch(b3d_gpu_context* ctx, const Mesh& m, long long n, int window = -1,
                       bool full_frame = false, size_t zhint = 0) {
  LaunchPlan lp;
  const size_t key = kIds ? 8 : 4;
  const size_t npx = (size_t)ctx->k.width * ctx->k.height;
  const int pad = kScore ? 2 * (window >= 0 ? window : ctx->lik.window) : 0;
  const size_t padded = (size_t)(ctx->k.width + 2 * pad) * (ctx->k.height + 2 * pad);
  // 2 CTAs/SM; the projected vertices go to shared memory when they fit
  // next to a region z-buffer of at least 2,048 pixels, otherwise to the
  // per-CTA global scratch (L1/L2).  Occupancy wins over the on-chip vertex
  // cache: 1 CTA/SM with the cache on chip measured 29 % slower on cfg4
  // (2,000 voxels) and 12 % on cfg2 (3,000 voxels).  full_frame (camera mode: the table
  // fills the image): prefer the first of (2 CTAs, vertices on chip), (1 CTA,
  // vertices on chip), (1 CTA, vertices in scratch) whose z-buffer holds the
  // whole padded image.
  const size_t vbytes = 32ull * m.nv;  // u, v, 1/z (fp64) + packed int bbox
  const size_t stage = render_score_staging_bytes(m.nt);
  const size_t zmin = std::min<size_t>(2048, npx) * key;
  // shared memory per SM is 228 KB (227 KB max per CTA), 1 KB reserved per
  // CTA, plus the kernel's static shared memory
  const size_t stat = static_smem_render_score<kIds, kScore, kOut>();
  auto budget_for = [&](int b) {
    size_t bud = 233472 / b - 1024 - stat;
    return std::min<size_t>(bud, 232448 - stat);
  };
  size_t budget = 0;
  lp.vcap = 0;
  static const int min_b = [] {
    const char* e = std::getenv("B3D_PLAN_MINB");  // 1: allow 1 CTA/SM (A/B only)
    return e ? std::atoi(e) : 2;
  }();
  static const bool no_vcache = std::getenv("B3D_PLAN_VCAP0") != nullptr;  // A/B only
  static const int max_b = [] {
    const char* e = std::getenv("B3D_PLAN_MAXB");  // A/B only: plan for up to N CTAs/SM
    const int v = e ? std::atoi(e) : 2;
    return v >= 2 && v <= 8 ? v : 2;
  }();
  for (int b = max_b; b >= min_b; --b) {
    budget = budget_for(b);
    if (!no_vcache && vbytes + stage + zmin <= budget) {
      lp.vcap = m.nv;
      break;
    }
  }
  if (lp.vcap == 0) budget = budget_for(max_b);
  if (full_frame && (budget - 32ull * lp.vcap - stage) / key < padded) {
    if (vbytes + stage + padded * key <= budget_for(1)) {
      budget = budget_for(1);
      lp.vcap = m.nv;
    } else if (stage + padded * key <= budget_for(1)) {
      budget = budget_for(1);
      lp.vcap = 0;
    }
  }
  size_t zcap = (budget - 32ull * lp.vcap - stage) / key;
  if (zcap > padded + 64) zcap = padded + 64;
  static const long long zcap_env = [] {
    const char* e = std::getenv("B3D_PLAN_ZCAP");  // A/B only: cap the z-buffer keys
    return e ? std::atoll(e) : 0ll;
  }();
  if (zcap_env > 0 && lp.vcap == 0 && !full_frame && zcap > (size_t)zcap_env) zcap = zcap_env;
  // a z-buffer sized to the batch's projected regions rather than to the
  // whole budget: with the vertex cache in scratch, the shared memory not
  // requested is L1 for it (cfg2 +8 %); regions beyond it take the scratch
  // z-buffer, so the hint only moves speed, never results
  if (zhint > 0 && lp.vcap == 0 && !full_frame) zcap = std::min(zcap, std::max<size_t>(zhint, 2048));
  zcap &= ~size_t(7);  // the vertex cache after the z-buffer stays 32-byte aligned
  lp.zcap = (int)zcap;
  lp.smem = 32ull * lp.vcap + stage + key * zcap;
  int per_sm = 0;
  cuda_check(occupancy_render_score<kIds, kScore, kOut>(&per_sm, lp.smem, lp.vcap >= m.nv), "occupancy");
  if (per_sm < 1) per_sm = 1;
  long long grid = (long long)per_sm * ctx->sm_count;
  lp.cap = (int)grid;  // resident capacity: score launches may pair CTAs on the batch tail
  if (grid > n) grid = n;
  if (grid < 1) grid = 1;
  lp.grid = (int)grid;
  // overflow scratch for hypotheses whose region / mesh exceeds shared memory
  lp.zstride = (long long)(ctx->k.width + 2 * pad) * (ctx->k.height + 2 * pad);
  const size_t ctas = kScore ? (size_t)lp.cap : (size_t)lp.grid;
  ctx->zscratch.ensure(ctas * lp.zstride * 8);
  if (lp.vcap < m.nv) ctx->vscratch.ensure(ctas * 32 * m.nv);
  return lp;
}

KParams base_params(b3d_gpu_context* ctx, const Mesh& m) {
  KParams p{};
  // big projected faces: only 1x1 bboxes stay in the tile queue; 2x2 and
  // 3x3 take the per-lane loop too (cfg4 173 -> 180 FPS, cfg3 +3 % vs
  // queueing 2x2; B3D_Q1_SMALL overrides for A/B)
  // (A/B overrides; out-of-range values are ignored: the 3x3 tile queue
  // covers at most 3 columns / rows and the packed bh-1 field is 2 bits)
  static const int q1_small = [] {
    const char* e = std::getenv("B3D_Q1_SMALL");
    const int v = e ? std::atoi(e) : 1;
    if (e) std::fprintf(stderr, "b3d: B3D_Q1_SMALL=%s %s\n", e,
                        v >= 1 && v <= 3 ? "(A/B override)" : "ignored (must be 1..3)");
    return v >= 1 && v <= 3 ? v : 1;
  }();
  p.q1_small = q1_small;
  static const int q1_ratio = [] {  // region px per 100 triangles (B3D_Q1_RATIO: A/B)
    const char* e = std::getenv("B3D_Q1_RATIO");
    const int v = e ? std::atoi(e) : 20;
    if (e) std::fprintf(stderr, "b3d: B3D_Q1_RATIO=%s %s\n", e,
                        v >= 0 ? "(A/B override)" : "ignored (must be >= 0)");
    return v >= 0 ? v : 20;
  }();
  p.q1_ratio = q1_ratio;
  static const int obs_stage = [] {  // B3D_OBS_STAGE=0/1 (A/B of the bulk-copy staging)
    const char* e = std::getenv("B3D_OBS_STAGE");
    return e ? (std::atoi(e) != 0) : 0;
  }();
  p.obs_stage = obs_stage;

  const b3d_intrinsics& k = ctx->k;
  p.fx = k.fx;
  p.fy = k.fy;
  p.cx = k.cx;
  p.cy = k.cy;
  p.near_m = k.near_m;
  p.far_m = k.far_m;
  p.near_lim = k.near_m * (1.0 - 1e-12);
  p.far_f = static_cast<float>(k.far_m);

  p.W = (int)k.width;
  p.H = (int)k.height;
  p.fcx = (float)k.cx;
  p.fcy = (float)k.cy;
  p.inv_fx = (float)(1.0 / k.fx);
  p.inv_fy = (float)(1.0 / k.fy);
  p.w2c = ctx->w2c;
  p.verts = m.verts.as<double>();
  p.tris = m.tris.as<uint4>();
  p.nv = m.nv;
  p.nt = m.nt;
  p.draw_base = 0;
  p.cull = ctx->culling ? m.cull : 0;
  p.n_score_peers = 0;  // set per call by the peer-enabled score paths only
  p.tris_s = m.tris_s.as<uint4>();
  p.plane_off = m.plane_off.as<double>();
  p.plane_end = m.plane_end.as<int>();
  for (int i = 0; i < 8; ++i) {
    p.cls_start[i] = m.cls_start[i];
    p.plane_begin[i] = m.plane_begin[i];
  }
  p.obs = ctx->obs_pts.as<float4>();
  p.obs_count = ctx->obs_count.as<int>();
  p.lik = ctx->lik;
  p.zscratch = ctx->zscratch.as<unsigned long long>();
  p.vscratch = ctx->vscratch.as<double>();
  return p;
}

// Base-scene terms for the likelihood settings in p.lik:
// S_base per observed pixel and sigma slot, and the Chebyshev coefficients of
// G_e(log |y|) = sum_p log(floor_e + coef_e(|y|) * S_base(p)) on [0, log(W*H)].
// Cached per (observation, base scene, likelihood settings).
void attach_base(b3d_gpu_context* ctx, KParams& p) {
  p.draw_base = ctx->base_draw;
  if (!ctx->has_base) {
    p.base_keys = nullptr;
    return;
  }
  p.base_keys = ctx->base_keys.as<unsigned long long>();
  p.base_valid = ctx->base_valid;
  p.cheb_lo = 0.0;
  p.cheb_hi = std::log((double)ctx->k.width * ctx->k.height);
  if (p.lik.n_noise == 0) return;  // render-only use
  std::string key(reinterpret_cast<const char*>(&p.lik), sizeof(KLik));
  key += std::to_string(ctx->obs_version) + "/" + std::to_string(ctx->base_version);
  const size_t npx = (size_t)ctx->k.width * ctx->k.height;
  if (key != ctx->base_terms_key) {
    const int pad = p.lik.window;
    ctx->base_pad.ensure(4ull * (ctx->k.width + 2 * pad) * (ctx->k.height + 2 * pad));
    ctx->sbase.ensure(4ull * kMaxSlots * npx);
    ctx->gnodes.ensure(8ull * kMaxNoise * kCheb);
    ctx->cheb.ensure(8ull * kMaxNoise * kCheb);
    cuda_check(launch_base_terms(p, p.base_keys, ctx->base_pad.as<unsigned int>(),
                                 ctx->sbase.as<float>(), ctx->gnodes.as<double>(), ctx->stream),
               "base terms launch");
    std::vector<double> f(kMaxNoise * kCheb), coef(kMaxNoise * kCheb, 0.0);
    cuda_check(cudaMemcpyAsync(f.data(), ctx->gnodes.p, 8ull * p.lik.n_noise * kCheb,
                               cudaMemcpyDeviceToHost, ctx->stream),
               "cudaMemcpyAsync G nodes");
    cuda_check(cudaStreamSynchronize(ctx->stream), "base terms");
    const double pi = 3.14159265358979323846;
    for (int e = 0; e < p.lik.n_noise; ++e)
      for (int j = 0; j < kCheb; ++j) {
        double s = 0.0;
        for (int k = 0; k < kCheb; ++k)
          s += f[e * kCheb + k] * std::cos(pi * j * (k + 0.5) / kCheb);
        coef[e * kCheb + j] = 2.0 * s / kCheb;
      }
    cuda_check(cudaMemcpyAsync(ctx->cheb.p, coef.data(), 8ull * kMaxNoise * kCheb,
                               cudaMemcpyHostToDevice, ctx->stream),
               "cudaMemcpyAsync cheb");
    ctx->base_terms_key = key;
  }
  p.sbase = ctx->sbase.as<float>();
  p.cheb = ctx->cheb.as<double>();
}

void finish_copy_out(b3d_gpu_context* ctx, void* dst, const void* src, size_t bytes) {
  cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream),
             "cudaMemcpyAsync D2H");
}

// windowed_log_likelihood_multi settings (likelihood.cpp:14-26,162-186) for
// one fused launch: per-noise coefficients and the distinct-sigma slots.
KLik make_lik(const b3d_intrinsics& k, const b3d_noise* noise, uint32_t n_noise,
              double sigma_max, int window, int prefactor) {
  const double vol = visible_volume(k);
  KLik L{};
  L.n_noise = (int)n_noise;
  L.window = window;
  std::vector<double> slots;
  for (uint32_t e = 0; e < n_noise; ++e) {
    const b3d_noise& np = noise[e];
    const double sigma2 = np.sigma_noise * np.sigma_noise;
    L.one_minus_p[e] = 1.0 - np.p_outlier;
    L.norm3[e] = std::pow(6.283185307179586476925287 * sigma2, -1.5);
    L.floor_term[e] = np.p_outlier / vol;
    L.log_floor[e] = std::log(L.floor_term[e]);
    L.prefactor[e] = prefactor == B3D_PREFACTOR_PRINTED ? std::log(np.sigma_noise / sigma_max)
                                                        : -std::log(sigma_max);
    size_t s = 0;
    while (s < slots.size() && slots[s] != np.sigma_noise) ++s;
    if (s == slots.size()) slots.push_back(np.sigma_noise);
    L.slot_of[e] = (int)s;
  }
  L.n_slots = (int)slots.size();
  for (size_t s = 0; s < slots.size(); ++s) {
    L.slot_scale[s] = (float)(1.4426950408889634 / (2.0 * slots[s] * slots[s]));
    L.slot_root[s] = (float)std::sqrt(1.4426950408889634 / (2.0 * slots[s] * slots[s]));
  }
  return L;
}

// The same entries for the fp64 image path (exact_score.cu), with each
// form's own rounding of 1/(2 sigma^2): windowed 1/((2 s) s)
// (likelihood.cpp:186-187), full 1/(2 (s s)) (likelihood.cpp:91-92).
KExactLik make_exact_lik(const KLik& L, const b3d_noise* noise, int window) {
  KExactLik X{};
  X.n_noise = L.n_noise;
  X.n_slots = L.n_slots;
  X.window = window;
  for (int e = 0; e < L.n_noise; ++e) {
    X.slot_of[e] = L.slot_of[e];
    X.one_minus_p[e] = L.one_minus_p[e];
    X.norm3[e] = L.norm3[e];
    X.floor_term[e] = L.floor_term[e];
    X.prefactor[e] = L.prefactor[e];
    const double sg = noise[e].sigma_noise;
    X.inv2s2[L.slot_of[e]] = window >= 0 ? 1.0 / (2.0 * sg * sg) : 1.0 / (2.0 * (sg * sg));
  }
  return X;
}

// Outlier probabilities below this take the fp64 image path: with the floor
// p/V that small, an fp32 window sum that underflows to 0 (exp of < -103)
// changes the pixel's term from log(coef * S) (finite in fp64 down to exp of
// -745) to log(floor); above it coef * S at fp32 underflow is < 1e-25 of
// the floor and the fused kernel's terms are exact to its tolerance.
constexpr double kExactOutlierP = 1e-6;

// Likelihood settings of one score call (b3d_gpu_set_likelihood, a
// coarse-to-fine stage): the noise entries split into launches the fused
// kernel supports -- contiguous runs of <= kMaxNoise entries with <=
// kMaxSlots distinct sigmas -- plus the columns that score -inf.
//
// gate = true is the inference seam (score_cells -> observation_loglik_cached_multi,
// inference.cpp:40-45,59-83): an entry outside the noise support (p_outlier
// outside [0,1], sigma_noise <= 0 or > sigma_max) scores -inf and the others
// are scored; window < 0 selects the untruncated likelihood (inference.cpp:51-56).
// gate = false is windowed_log_likelihood_multi itself (likelihood.cpp:137-141):
// validate_noise errors, sigma_noise > sigma_max is scored, window >= 0.
LikSpec make_spec(const b3d_intrinsics& k, const b3d_noise* noise, uint32_t n_noise,
                  double sigma_max, int window, int prefactor, bool gate) {
  require(n_noise >= 1, ErrorCode::invalid, "no noise settings given");
  require(gate || window >= 0, ErrorCode::invalid, "window radius must be >= 0");
  require(prefactor == B3D_PREFACTOR_PRINTED || prefactor == B3D_PREFACTOR_UNIFORM,
          ErrorCode::invalid, "unknown prefactor");
  const double vol = visible_volume(k);
  require(vol > 0, ErrorCode::invalid, "scene volume must be positive");
  require(sigma_max > 0, ErrorCode::invalid, "sigma_max must be positive");
  LikSpec spec;
  spec.n_cols = (int)n_noise;
  spec.window = window;
  spec.exact = window < 0;
  std::vector<uint32_t> live;
  for (uint32_t e = 0; e < n_noise; ++e) {
    const b3d_noise& np = noise[e];
    if (gate) {
      if (!(np.p_outlier >= 0 && np.p_outlier <= 1 && np.sigma_noise > 0 &&
            np.sigma_noise <= sigma_max)) {
        spec.gated.push_back((int)e);
        continue;
      }
    } else {
      require(np.sigma_noise > 0, ErrorCode::invalid, "sigma_noise must be positive");
      require(np.p_outlier >= 0 && np.p_outlier <= 1, ErrorCode::invalid,
              "p_outlier must be in [0,1]");
    }
    if (np.p_outlier < kExactOutlierP) spec.exact = true;
    live.push_back(e);
  }
  // contiguous runs of live entries, cut at kMaxNoise entries / kMaxSlots sigmas
  size_t i = 0;
  while (i < live.size()) {
    size_t j = i;
    std::vector<double> slots;
    while (j < live.size() && (j == i || live[j] == live[j - 1] + 1) && j - i < (size_t)kMaxNoise) {
      const double sg = noise[live[j]].sigma_noise;
      if (std::find(slots.begin(), slots.end(), sg) == slots.end()) {
        if (slots.size() == (size_t)kMaxSlots) break;
        slots.push_back(sg);
      }
      ++j;
    }
    LikChunk c;
    c.col0 = (int)live[i];
    c.lik = make_lik(k, noise + live[i], (uint32_t)(j - i), sigma_max, window < 0 ? 0 : window,
                     prefactor);
    c.ex = make_exact_lik(c.lik, noise + live[i], window);
    spec.chunks.push_back(c);
    i = j;
  }
  return spec;
}

// ------------------------------------------------ table contact (host side)
constexpr double kTwoPiD = 6.283185307179586476925287;

// Eigen AngleAxis -> Quaternion with a unit axis (scene_graph.cpp:60-71,116).
void axis_angle_q(const double ax[3], double angle, double q[4]) {
  const double ha = 0.5 * angle;
  const double s = std::sin(ha);
  q[0] = std::cos(ha);
  q[1] = s * ax[0];
  q[2] = s * ax[1];
  q[3] = s * ax[2];
}

// scene_graph.cpp:60-71
void face_rotation(int face, double q[4]) {
  const double half_pi = kTwoPiD / 4.0;
  static const double ux[3] = {1, 0, 0}, uy[3] = {0, 1, 0};
  switch (face) {
    case 1: q[0] = 1; q[1] = q[2] = q[3] = 0; return;
    case 2: axis_angle_q(ux, 2 * half_pi, q); return;
    case 3: axis_angle_q(uy, -half_pi, q); return;
    case 4: axis_angle_q(uy, half_pi, q); return;
    case 5: axis_angle_q(ux, half_pi, q); return;
    default: axis_angle_q(ux, -half_pi, q); return;
  }
}

// scene_graph.cpp:73-89 (Eigen scalar order, as the oracle)
void rotated_bounds(const double amin[3], const double amax[3], int face, double lo[3],
                    double hi[3]) {
  double q[4];
  face_rotation(face, q);
  const double tx = 2.0 * q[1], ty = 2.0 * q[2], tz = 2.0 * q[3];
  const double twx = tx * q[0], twy = ty * q[0], twz = tz * q[0];
  const double txx = tx * q[1], txy = ty * q[1], txz = tz * q[1];
  const double tyy = ty * q[2], tyz = tz * q[2], tzz = tz * q[3];
  const double m[9] = {1.0 - (tyy + tzz), txy - twz,         txz + twy,
                       txy + twz,         1.0 - (txx + tzz), tyz - twx,
                       txz - twy,         tyz + twx,         1.0 - (txx + tyy)};
  for (int i = 0; i < 8; ++i) {
    const double c[3] = {i & 1 ? amax[0] : amin[0], i & 2 ? amax[1] : amin[1],
                         i & 4 ? amax[2] : amin[2]};
    for (int a = 0; a < 3; ++a) {
      const double r = m[3 * a] * c[0] + (m[3 * a + 1] * c[1] + m[3 * a + 2] * c[2]);
      if (i == 0) {
        lo[a] = hi[a] = r;
      } else {
        lo[a] = r < lo[a] ? r : lo[a];
        hi[a] = r > hi[a] ? r : hi[a];
      }
    }
  }
}

// Host quaternion helpers in Eigen's evaluation order (posemath.cuh restates
// the same on the device).
struct HQ {
  double w, x, y, z;
};
HQ hq_mul(const HQ& a, const HQ& b) {
  return HQ{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
            a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z,
            a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}
HQ hq_normalized(HQ q) {
  const double n2 = (q.x * q.x + q.y * q.y) + (q.z * q.z + q.w * q.w);
  if (n2 > 0) {
    const double n = std::sqrt(n2);
    q.w /= n;
    q.x /= n;
    q.y /= n;
    q.z /= n;
  }
  return q;
}
void hq_rotate(const HQ& q, const double v[3], double o[3]) {
  double uv0 = q.y * v[2] - q.z * v[1];
  double uv1 = q.z * v[0] - q.x * v[2];
  double uv2 = q.x * v[1] - q.y * v[0];
  uv0 += uv0;
  uv1 += uv1;
  uv2 += uv2;
  const double c0 = q.y * uv2 - q.z * uv1;
  const double c1 = q.z * uv0 - q.x * uv2;
  const double c2 = q.x * uv1 - q.y * uv0;
  o[0] = v[0] + q.w * uv0 + c0;
  o[1] = v[1] + q.w * uv1 + c1;
  o[2] = v[2] + q.w * uv2 + c2;
}

// scene_graph.cpp:97-121 contact_to_pose (table extents given directly)
KPose contact_to_pose_host(double table_w, double table_h, const double amin[3],
                           const double amax[3], int face, double dx, double dy, double dtheta) {
  require(face >= 1 && face <= 6, ErrorCode::invalid, "face must be in 1..6");
  double lo[3], hi[3];
  rotated_bounds(amin, amax, face, lo, hi);
  const double w = hi[0] - lo[0];
  const double h = hi[1] - lo[1];
  require(dx >= 0 && dx <= table_w - w && dy >= 0 && dy <= table_h - h && dtheta >= 0 &&
              dtheta < kTwoPiD,
          ErrorCode::invalid, "contact params out of valid range");
  const double corner[3] = {-table_w / 2, -table_h / 2, 0.0};
  const double bt[3] = {corner[0] + (dx - lo[0]), corner[1] + (dy - lo[1]), corner[2] + -lo[2]};
  const double pivot[3] = {corner[0] + (dx + w / 2), corner[1] + (dy + h / 2), corner[2] + 0.0};
  static const double uz[3] = {0, 0, 1};
  double s[4], f[4];
  axis_angle_q(uz, dtheta, s);
  face_rotation(face, f);
  const HQ spin{s[0], s[1], s[2], s[3]};
  const HQ q = hq_normalized(hq_mul(spin, HQ{f[0], f[1], f[2], f[3]}));
  const double rel[3] = {bt[0] - pivot[0], bt[1] - pivot[1], bt[2] - pivot[2]};
  double r[3];
  hq_rotate(spin, rel, r);
  return KPose{q.w, q.x, q.y, q.z, r[0] + pivot[0], r[1] + pivot[1], r[2] + pivot[2]};
}

// KGrid (mode 2) for the children of a contact cell (subdivide_cell): face
// rotation, footprint and the per-cell spin cos/sin computed here with
// libm; the rest runs on device.  cells.grid alone (stage 0) is the parent
// [0, table - footprint] x [0, 2 pi).
KGrid make_contact_cells(const b3d_contact_cells& cells, std::vector<double>& spin) {
  const b3d_contact_grid& g = cells.grid;
  check(g.face >= 1 && g.face <= 6, "face must be in 1..6");
  check(g.count[0] >= 1 && g.count[1] >= 1 && g.count[2] >= 1,
        "schedule stage: subdivision counts must be >= 1");
  KGrid k{};
  k.mode = 2;
  for (int a = 0; a < 3; ++a) k.count[a] = (int)g.count[a];
  KContact& c = k.contact;
  face_rotation(g.face, c.face_q);
  double lo[3], hi[3];
  rotated_bounds(g.aabb_min, g.aabb_max, g.face, lo, hi);
  for (int a = 0; a < 3; ++a) c.lo[a] = lo[a];
  c.w = hi[0] - lo[0];
  c.h = hi[1] - lo[1];
  c.table_w = g.table_w;
  c.table_h = g.table_h;
  c.dx_lo = cells.dx_lo;
  c.dx_w = cells.dx_hi - cells.dx_lo;
  c.dy_lo = cells.dy_lo;
  c.dy_w = cells.dy_hi - cells.dy_lo;
  spin.resize(2 * g.count[2]);
  const double tw = cells.dtheta_hi - cells.dtheta_lo;
  for (uint32_t it = 0; it < g.count[2]; ++it) {
    const double dlo = cells.dtheta_lo + tw * it / g.count[2];
    const double dhi = cells.dtheta_lo + tw * (it + 1) / g.count[2];
    const double dtheta = 0.5 * (dlo + dhi);
    const double ha = 0.5 * dtheta;
    spin[2 * it] = std::cos(ha);
    spin[2 * it + 1] = std::sin(ha);
  }
  return k;
}

// stage 0 of one (object, face): the full contact support as parent cell
b3d_contact_cells stage0_parent(const b3d_contact_grid& g) {
  check(g.face >= 1 && g.face <= 6, "face must be in 1..6");
  double lo[3], hi[3];
  rotated_bounds(g.aabb_min, g.aabb_max, g.face, lo, hi);
  b3d_contact_cells cells{};
  cells.grid = g;
  cells.dx_lo = 0.0;
  cells.dx_hi = g.table_w - (hi[0] - lo[0]);
  cells.dy_lo = 0.0;
  cells.dy_hi = g.table_h - (hi[1] - lo[1]);
  cells.dtheta_lo = 0.0;
  cells.dtheta_hi = kTwoPiD;
  require(cells.dx_hi > 0 && cells.dy_hi > 0, ErrorCode::numeric,
          "stage 0: empty proposal support (no object fits the table)");
  return cells;
}

// Host pose of child (ix, iy, it): the operations of posemath.cuh contact_pose.
b3d_pose contact_cell_pose(const KGrid& g, const std::vector<double>& spin, uint32_t ix,
                           uint32_t iy, uint32_t it) {
  const KContact& c = g.contact;
  const uint32_t nx = g.count[0], ny = g.count[1];
  const double dx = 0.5 * ((c.dx_lo + c.dx_w * ix / nx) + (c.dx_lo + c.dx_w * (ix + 1) / nx));
  const double dy = 0.5 * ((c.dy_lo + c.dy_w * iy / ny) + (c.dy_lo + c.dy_w * (iy + 1) / ny));
  const HQ spin_q{spin[2 * it], spin[2 * it + 1] * 0.0, spin[2 * it + 1] * 0.0,
                  spin[2 * it + 1] * 1.0};
  const double cx = -c.table_w / 2, cy = -c.table_h / 2, cz = 0.0;
  const double bt[3] = {cx + (dx - c.lo[0]), cy + (dy - c.lo[1]), cz + -c.lo[2]};
  const double pv[3] = {cx + (dx + c.w / 2), cy + (dy + c.h / 2), cz + 0.0};
  const HQ q = hq_normalized(
      hq_mul(spin_q, HQ{c.face_q[0], c.face_q[1], c.face_q[2], c.face_q[3]}));
  const double rel[3] = {bt[0] - pv[0], bt[1] - pv[1], bt[2] - pv[2]};
  double r[3];
  hq_rotate(spin_q, rel, r);
  return b3d_pose{q.w, q.x, q.y, q.z, r[0] + pv[0], r[1] + pv[1], r[2] + pv[2]};
}

// The fp64 image path (exact_score.cu): render the hypotheses of p in chunks
// (render-mode kernel, depth to HBM), then score every image per chunk of
// noise entries.  p is a score-mode parameter block (object or camera mode,
// base attached); d_scores n x spec.n_cols and d_status are device memory.
void exact_scores(b3d_gpu_context* ctx, const Mesh& m, const KParams& p, const LikSpec& spec,
                  long long n, double* d_scores, uint8_t* d_status, bool camera) {
  const size_t npx = (size_t)ctx->k.width * ctx->k.height;
  const long long chunk = std::max<long long>(1, std::min<long long>(n, (256ll << 20) / (4 * npx)));
  ctx->ex_depth.ensure(4 * npx * (size_t)chunk);
  const int ctas = (int)std::min<long long>(chunk, 4ll * ctx->sm_count);
  if (spec.window < 0) ctx->ex_pts.ensure(exact_score_pts_bytes((int)ctx->k.width, (int)ctx->k.height, ctas));
  for (long long h0 = 0; h0 < n; h0 += chunk) {
    const long long c = std::min(chunk, n - h0);
    KParams q = p;
    q.lik.n_noise = 0;  // render only
    if (!camera) attach_base(ctx, q);
    q.scores = nullptr;
    q.status = nullptr;
    q.n_score_peers = 0;
    q.rng_dst = nullptr;
    q.n_hyp = c;
    if (camera)
      q.cams = p.cams + h0;
    else if (p.poses)
      q.poses = p.poses + h0;
    else
      q.index0 = p.index0 + h0;
    q.out_depth = ctx->ex_depth.as<float>();
    q.out_ids = nullptr;
    q.out_keys = nullptr;
    LaunchPlan lp = plan_launch<false, false, true>(ctx, m, c);
    q.zscratch = ctx->zscratch.as<unsigned long long>();
    q.vscratch = ctx->vscratch.as<double>();
    q.vcap = lp.vcap;
    q.zcap = lp.zcap;
    q.zstride = lp.zstride;
    cuda_check(launch_render_score<false, false, true>(q, lp.grid, lp.smem, ctx->stream),
               "render launch (fp64 path)");
    for (const LikChunk& ch : spec.chunks) {
      KExactArgs a{};
      a.obs = ctx->obs_pts.as<float4>();
      a.rend = ctx->ex_depth.as<float>();
      a.W = (int)ctx->k.width;
      a.H = (int)ctx->k.height;
      a.fx = ctx->k.fx;
      a.fy = ctx->k.fy;
      a.cx = ctx->k.cx;
      a.cy = ctx->k.cy;
      a.far_f = static_cast<float>(ctx->k.far_m);
      a.n = c;
      a.scores = d_scores + (size_t)h0 * spec.n_cols;
      a.ld = spec.n_cols;
      a.col0 = ch.col0;
      a.status = d_status ? d_status + h0 : nullptr;
      a.pts = spec.window < 0 ? ctx->ex_pts.as<double>() : nullptr;
      a.lik = ch.ex;
      cuda_check(launch_exact_score(a, (int)std::min<long long>(c, ctas), ctx->stream),
                 "exact_score launch");
    }
  }
}

// Scores the n hypotheses of p (score mode, everything set but lik / scores /
// status / plan) under `spec` into device arrays: one fused launch when the
// spec fits it, else one launch per chunk of entries (columns copied into
// place), -inf for gated columns, or the fp64 image path.
void run_scores(b3d_gpu_context* ctx, const Mesh& m, KParams p, const LikSpec& spec, long long n,
                double* d_scores, uint8_t* d_status, bool camera, size_t zhint,
                bool pdl = false) {
  const int nc = spec.n_cols;
  for (int col : spec.gated)
    cuda_check(launch_fill_column(d_scores, n, nc, col, -std::numeric_limits<double>::infinity(),
                                  ctx->stream),
               "fill launch");
  if (spec.chunks.empty()) {  // every entry outside the support: nothing rendered
    if (d_status) cuda_check(cudaMemsetAsync(d_status, 0, (size_t)n, ctx->stream), "memset");
    if (p.n_score_peers)
      cuda_check(launch_copy_to_peers(d_scores, n * nc, p.score_peers, p.n_score_peers,
                                      p.score_peer_offset * nc, p.score_peer_cap, ctx->stream),
                 "copy_to_peers launch");
    return;
  }
  // peers requested but the scores do not come out of one fused launch:
  // store them to the peers after the fact (same elements, same capacity)
  auto copy_to_peers = [&] {
    if (!p.n_score_peers) return;
    cuda_check(launch_copy_to_peers(d_scores, n * nc, p.score_peers, p.n_score_peers,
                                    p.score_peer_offset * nc, p.score_peer_cap, ctx->stream),
               "copy_to_peers launch");
  };
  if (spec.exact) {
    exact_scores(ctx, m, p, spec, n, d_scores, d_status, camera);
    copy_to_peers();
    return;
  }
  const bool in_place = spec.single();
  if (!in_place) {
    size_t widest = 0;
    for (const LikChunk& ch : spec.chunks) widest = std::max(widest, (size_t)ch.lik.n_noise);
    ctx->chunk_scores.ensure(8 * widest * (size_t)n);
  }
  const int peers = p.n_score_peers;
  if (!in_place) p.n_score_peers = 0;
  for (const LikChunk& ch : spec.chunks) {
    p.lik = ch.lik;
    if (!camera) attach_base(ctx, p);
    p.scores = in_place ? d_scores : ctx->chunk_scores.as<double>();
    p.status = d_status;
    LaunchPlan lp = plan_launch<false, true, false>(ctx, m, n, ch.lik.window, camera, zhint);
    p.zscratch = ctx->zscratch.as<unsigned long long>();
    p.vscratch = ctx->vscratch.as<double>();
    p.vcap = lp.vcap;
    p.zcap = lp.zcap;
    p.zstride = lp.zstride;
    cuda_check(launch_render_score<false, true, false>(p, lp.cap, lp.smem, ctx->stream, pdl),
               camera ? "render_score launch (cameras)" : "render_score launch");
    if (!in_place)
      cuda_check(cudaMemcpy2DAsync(d_scores + ch.col0, 8ull * nc, p.scores,
                                   8ull * ch.lik.n_noise, 8ull * ch.lik.n_noise, (size_t)n,
                                   cudaMemcpyDeviceToDevice, ctx->stream),
                 "cudaMemcpy2DAsync scores");
  }
  if (!in_place) {
    p.n_score_peers = peers;
    copy_to_peers();
  }
}

void score_common(b3d_gpu_context* ctx, int32_t mesh_id, const b3d_pose* poses,
                  const b3d_pose_grid* grid, uint64_t n, double* scores, uint8_t* status,
                  const b3d_contact_cells* contact = nullptr, uint64_t first = 0,
                  uint64_t grid_n = 0, unsigned long long* stage_rng = nullptr,
                  KStageResult* stage_out = nullptr, bool peers = false) {
  require_ready(ctx, true, true);
  check(scores != nullptr, "bad arguments");
  check(n > 0, "score_cells: no cells");
  DeviceGuard dg(ctx->device);
  const Mesh& m = get_mesh(ctx, mesh_id);
  KParams p = base_params(ctx, m);
  bool host_in = false;
  if (poses) {
    p.poses = static_cast<const KPose*>(
        stage_in(ctx, ctx->in_stage, poses, sizeof(b3d_pose) * n, &host_in));
  } else if (contact) {
    std::vector<double> spin;
    p.poses = nullptr;
    p.grid = make_contact_cells(*contact, spin);
    const uint32_t* cnt = contact->grid.count;
    check((uint64_t)cnt[0] * cnt[1] * cnt[2] == n, "contact grid: n does not match the grid size");
    ctx->spin.ensure(8 * spin.size());
    cuda_check(cudaMemcpyAsync(ctx->spin.p, spin.data(), 8 * spin.size(), cudaMemcpyHostToDevice,
                               ctx->stream),
               "cudaMemcpyAsync spin");
    p.grid.contact.spin = ctx->spin.as<double>();
    host_in = true;
  } else {
    check(grid != nullptr && grid->rotations && grid->n_rot > 0, "bad arguments");
    const uint64_t nt = (uint64_t)grid->count[0] * grid->count[1] * grid->count[2];
    check(nt > 0, "pose grid: counts must be >= 1");
    const uint64_t gn = grid->mode == B3D_GRID_PRODUCT ? nt * grid->n_rot : nt;
    check(grid->mode == B3D_GRID_PRODUCT || nt == grid->n_rot,
          "pose grid: zip mode needs nx*ny*nz == n_rot");
    check(grid_n ? (gn == grid_n && first + n <= gn) : gn == n,
          "pose grid: n does not match the grid size");
    bool h2 = false;
    p.poses = nullptr;
    p.grid.center = pose_from_c(grid->center);
    p.grid.center_dev = nullptr;
    for (int a = 0; a < 3; ++a) {
      p.grid.extent[a] = grid->extent[a];
      p.grid.count[a] = (int)grid->count[a];
    }
    p.grid.rotations = static_cast<const double*>(
        stage_in(ctx, ctx->rot_stage, grid->rotations, 32ull * grid->n_rot, &h2));
    p.grid.n_rot = (int)grid->n_rot;
    p.grid.mode = (int)grid->mode;
    host_in = host_in || h2;
  }
  p.n_hyp = (long long)n;
  p.index0 = (long long)first;
  const LikSpec& spec = ctx->spec;
  const int nn = spec.n_cols;
  const bool dev_scores = is_device_ptr(scores);
  const bool dev_status = status && is_device_ptr(status);
  if (dev_scores) {
    p.scores = scores;
  } else {
    ctx->out_stage.ensure(sizeof(double) * n * nn);
    p.scores = ctx->out_stage.as<double>();
  }
  if (status) {
    if (dev_status) {
      p.status = status;
    } else {
      ctx->out_stage2.ensure(n);
      p.status = ctx->out_stage2.as<uint8_t>();
    }
  }
  size_t zhint = 0;
  if (poses && host_in) {
    zhint = region_hint_poses(ctx, m, poses, n, std::max(spec.window, 0));
  } else if (!poses && !contact) {
    zhint = region_hint(ctx, m, p.grid.center,
                        std::sqrt(sq3(grid->extent)), std::max(spec.window, 0));
  }
  if (peers && ctx->n_score_peers) {  // b3d_gpu_set_score_peers: the fused all-gather
    for (int r = 0; r < 8; ++r) p.score_peers[r] = ctx->score_peers[r];
    p.n_score_peers = ctx->n_score_peers;
    p.score_peer_offset = ctx->score_peer_offset;
    p.score_peer_cap = ctx->score_peer_cap;
  }
  run_scores(ctx, m, p, spec, (long long)n, p.scores, p.status, false, zhint);
  if (stage_out)
    cuda_check(launch_stage_reduce(p.scores, (long long)n, nn, 0, stage_rng, stage_out, nullptr,
                                   ctx->stream, stage_scratch(ctx, (long long)n)),
               "stage_reduce launch");
  bool sync = host_in;
  if (!dev_scores) {
    finish_copy_out(ctx, scores, p.scores, sizeof(double) * n * nn);
    sync = true;
  }
  if (status && !dev_status) {
    finish_copy_out(ctx, status, p.status, n);
    sync = true;
  }
  if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "score_poses");
}


// ---------------------------------------------------------------- camera mode
constexpr double kHalfPi = 1.5707963267948966;

// Eigen 3-vector reductions split as a0 + (a1 + a2) (redux unroller halves)

void normalize3(double v[3]) {
  const double n2 = sq3(v);
  if (n2 > 0) {
    const double n = std::sqrt(n2);
    v[0] /= n;
    v[1] /= n;
    v[2] /= n;
  }
}

// Eigen Quaternion(const Matrix3&) (trace / largest-diagonal branches),
// m row-major
void quat_from_rot(const double m[9], double q[4]) {
  auto M = [&](int i, int j) { return m[3 * i + j]; };
  double t = M(0, 0) + (M(1, 1) + M(2, 2));
  if (t > 0) {
    t = std::sqrt(t + 1.0);
    q[0] = 0.5 * t;
    t = 0.5 / t;
    q[1] = (M(2, 1) - M(1, 2)) * t;
    q[2] = (M(0, 2) - M(2, 0)) * t;
    q[3] = (M(1, 0) - M(0, 1)) * t;
  } else {
    int i = 0;
    if (M(1, 1) > M(0, 0)) i = 1;
    if (M(2, 2) > M(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    double c[3];
    t = std::sqrt(M(i, i) - M(j, j) - M(k, k) + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (M(k, j) - M(j, k)) * t;
    c[j] = (M(j, i) + M(i, j)) * t;
    c[k] = (M(k, i) + M(i, k)) * t;
    q[1] = c[0];
    q[2] = c[1];
    q[3] = c[2];
  }
}

// generative.cpp:35-59: camera on a sphere around the origin, optical axis
// through it, image "down" = -(world +z projected off the axis)
KPose camera_from_spherical(double distance, double azimuth, double altitude) {
  require(distance > 0, ErrorCode::invalid, "camera distance must be positive");
  require(altitude > 0 && altitude < kHalfPi, ErrorCode::invalid,
          "camera altitude must lie within (0, pi/2)");
  const double pos[3] = {distance * std::cos(altitude) * std::cos(azimuth),
                         distance * std::cos(altitude) * std::sin(azimuth),
                         distance * std::sin(altitude)};
  double fwd[3] = {-pos[0], -pos[1], -pos[2]};
  normalize3(fwd);
  const double d = 0.0 * fwd[0] + (0.0 * fwd[1] + 1.0 * fwd[2]);
  double up[3] = {0.0 - d * fwd[0], 0.0 - d * fwd[1], 1.0 - d * fwd[2]};
  require(std::sqrt(sq3(up)) > 1e-12, ErrorCode::invalid,
          "camera pose degenerate: looking along world z");
  normalize3(up);
  const double down[3] = {-up[0], -up[1], -up[2]};
  const double right[3] = {down[1] * fwd[2] - down[2] * fwd[1],
                           down[2] * fwd[0] - down[0] * fwd[2],
                           down[0] * fwd[1] - down[1] * fwd[0]};
  const double m[9] = {right[0], down[0], fwd[0], right[1], down[1],
                       fwd[1],   right[2], down[2], fwd[2]};
  double q[4];
  quat_from_rot(m, q);
  const double n2 = (q[1] * q[1] + q[2] * q[2]) + (q[3] * q[3] + q[0] * q[0]);
  if (n2 > 0) {
    const double n = std::sqrt(n2);
    for (double& x : q) x /= n;
  }
  return KPose{q[0], q[1], q[2], q[3], pos[0], pos[1], pos[2]};
}

// generative.cpp:61-85
bool camera_to_spherical(const KPose& pose, double tol, double& distance, double& azimuth,
                         double& altitude) {
  const double t[3] = {pose.tx, pose.ty, pose.tz};
  const double d = std::sqrt(sq3(t));
  if (d <= 0) return false;
  const double sin_alt = std::clamp(t[2] / d, -1.0, 1.0);
  const double alt = std::asin(sin_alt);
  if (alt <= 0 || alt >= kHalfPi) return false;
  double az = std::fmod(std::atan2(t[1], t[0]), kTwoPiD);
  if (az < 0) az += kTwoPiD;
  const KPose e = camera_from_spherical(d, az, alt);
  const double dt[3] = {e.tx - t[0], e.ty - t[1], e.tz - t[2]};
  if (std::sqrt(sq3(dt)) > tol * std::max(1.0, d)) return false;
  // coeffs() order (x, y, z, w), 4-term redux (x2 + y2) + (z2 + w2)
  const double a[4] = {e.qx - pose.qx, e.qy - pose.qy, e.qz - pose.qz, e.qw - pose.qw};
  const double b[4] = {e.qx + pose.qx, e.qy + pose.qy, e.qz + pose.qz, e.qw + pose.qw};
  const double qa = std::sqrt((a[0] * a[0] + a[1] * a[1]) + (a[2] * a[2] + a[3] * a[3]));
  const double qb = std::sqrt((b[0] * b[0] + b[1] * b[1]) + (b[2] * b[2] + b[3] * b[3]));
  if (std::min(qa, qb) > tol) return false;
  distance = d;
  azimuth = az;
  altitude = alt;
  return true;
}

// tracking.cpp:27-37
double lattice_at(double center, double extent, int n, int i) {
  if (n == 1) return center;
  return center - extent + 2.0 * extent * i / (n - 1);
}

void cam_params(b3d_gpu_context* ctx, KParams& p, const b3d_gpu_context::CamGroup& g) {
  (void)ctx;
  p.cams = nullptr;
  p.n_inst = g.n;
  for (int i = 0; i <= kMaxInst; ++i) p.inst_v0[i] = g.v0[i];
  for (int i = 0; i < kMaxInst; ++i) p.inst_pose[i] = g.pose[i];
  p.draw_base = g.draw_base;
  p.base_keys = nullptr;
}

// Render-many of hypotheses cams[0..n) over every camera group: depth (or,
// with keys, 64-bit (depth, draw) keys) of group 0 into out, each further
// group into a scratch image set merged per pixel (the z-test's minimum is
// the same whatever the instance order; ties keep the lower draw index).
void render_camera_groups(b3d_gpu_context* ctx, const KPose* cams, long long n, float* depth,
                          unsigned long long* keys) {
  const size_t npx = (size_t)ctx->k.width * ctx->k.height;
  for (size_t gi = 0; gi < ctx->cam_groups.size(); ++gi) {
    const auto& g = ctx->cam_groups[gi];
    const Mesh& m = *g.mesh;
    KParams q = base_params(ctx, m);
    cam_params(ctx, q, g);
    q.cams = cams;
    q.n_hyp = n;
    q.lik.n_noise = 0;
    q.scores = nullptr;
    q.status = nullptr;
    q.rng_dst = nullptr;
    q.n_score_peers = 0;
    float* od = nullptr;
    unsigned long long* ok = nullptr;
    if (gi == 0) {
      od = depth;
      ok = keys;
    } else if (keys) {
      ctx->cam_tmp.ensure(8 * npx * (size_t)n);
      ok = ctx->cam_tmp.as<unsigned long long>();
    } else {
      ctx->cam_tmp.ensure(4 * npx * (size_t)n);
      od = ctx->cam_tmp.as<float>();
    }
    q.out_depth = keys ? nullptr : od;
    q.out_ids = nullptr;
    q.out_keys = ok;
    if (keys) {
      LaunchPlan lp = plan_launch<true, false, true>(ctx, m, n);
      q.zscratch = ctx->zscratch.as<unsigned long long>();
      q.vscratch = ctx->vscratch.as<double>();
      q.vcap = lp.vcap;
      q.zcap = lp.zcap;
      q.zstride = lp.zstride;
      cuda_check(launch_render_score<true, false, true>(q, lp.grid, lp.smem, ctx->stream),
                 "render launch (camera groups)");
    } else {
      LaunchPlan lp = plan_launch<false, false, true>(ctx, m, n);
      q.zscratch = ctx->zscratch.as<unsigned long long>();
      q.vscratch = ctx->vscratch.as<double>();
      q.vcap = lp.vcap;
      q.zcap = lp.zcap;
      q.zstride = lp.zstride;
      cuda_check(launch_render_score<false, false, true>(q, lp.grid, lp.smem, ctx->stream),
                 "render launch (camera groups)");
    }
    if (gi > 0) {
      if (keys)
        cuda_check(launch_min_merge_u64(keys, ok, npx * (size_t)n, ctx->stream), "merge keys");
      else
        cuda_check(launch_min_merge_f32(depth, od, npx * (size_t)n, ctx->stream), "merge depth");
    }
  }
}

// score-many over camera poses (device-resident `cams` of n entries) into
// device buffers scores/status
void launch_score_cameras(b3d_gpu_context* ctx, const KPose* cams, long long n, double* scores,
                          uint8_t* status, bool pdl = false) {
  require(ctx->cam_spec_err.empty(), ErrorCode::invalid, ctx->cam_spec_err);
  if (ctx->cam_groups.size() == 1) {  // the fused camera-mode kernel
    const auto& g = ctx->cam_groups.front();
    const Mesh& m = *g.mesh;
    KParams p = base_params(ctx, m);
    cam_params(ctx, p, g);
    p.cams = cams;
    p.n_hyp = n;
    run_scores(ctx, m, p, ctx->cam_spec, n, scores, status, true, 0, pdl);
    return;
  }
  // more instances than one launch holds: merged group renders, then the
  // fp64 image likelihood (exact_score.cu) of each hypothesis
  const LikSpec& spec = ctx->cam_spec;
  const size_t npx = (size_t)ctx->k.width * ctx->k.height;
  const long long chunk =
      std::max<long long>(1, std::min<long long>(n, (256ll << 20) / (4 * (long long)npx)));
  ctx->ex_depth.ensure(4 * npx * (size_t)chunk);
  const int ctas = (int)std::min<long long>(chunk, 4ll * ctx->sm_count);
  if (spec.window < 0)
    ctx->ex_pts.ensure(exact_score_pts_bytes((int)ctx->k.width, (int)ctx->k.height, ctas));
  for (long long h0 = 0; h0 < n; h0 += chunk) {
    const long long c = std::min(chunk, n - h0);
    render_camera_groups(ctx, cams + h0, c, ctx->ex_depth.as<float>(), nullptr);
    for (const LikChunk& ch : spec.chunks) {
      KExactArgs a{};
      a.obs = ctx->obs_pts.as<float4>();
      a.rend = ctx->ex_depth.as<float>();
      a.W = (int)ctx->k.width;
      a.H = (int)ctx->k.height;
      a.fx = ctx->k.fx;
      a.fy = ctx->k.fy;
      a.cx = ctx->k.cx;
      a.cy = ctx->k.cy;
      a.far_f = static_cast<float>(ctx->k.far_m);
      a.n = c;
      a.scores = scores + (size_t)h0 * spec.n_cols;
      a.ld = spec.n_cols;
      a.col0 = ch.col0;
      a.status = status ? status + h0 : nullptr;
      a.pts = spec.window < 0 ? ctx->ex_pts.as<double>() : nullptr;
      a.lik = ch.ex;
      cuda_check(launch_exact_score(a, (int)std::min<long long>(c, ctas), ctx->stream),
                 "exact_score launch (camera groups)");
    }
  }
}
}  // namespace

// the thread-local error channel, shared with smc.cpp (not exported)
void b3d200_set_last_error(const char* msg) { g_last_error = msg; }

// CameraIntrinsics::validate (geometry.cpp:38-44) for the handle layer
void b3d200_validate_intrinsics(const b3d_intrinsics& k) { validate_intrinsics(k); }

// render_instances (renderer.cpp:174-184) for scenes with more instances than
// the camera-mode kernel holds: the instances rasterized one after another
// into the base-scene key buffer (object mode, the same arithmetic, draw
// order table -> children), read back as depth with the far sentinel.
void b3d200_render_scene_keys(b3d_gpu_context* ctx, const b3d_intrinsics* k,
                              const b3d_pose* camera, const int32_t* ids, const b3d_pose* poses,
                              uint32_t n, float* out) {
  auto ok = [](b3d_status s) {
    if (s != B3D_OK) throw Error(static_cast<ErrorCode>(s), b3d_last_error());
  };
  ok(b3d_gpu_set_camera(ctx, k, camera));
  ok(b3d_gpu_set_base_scene(ctx, ids, poses, n));
  const size_t npx = (size_t)k->width * k->height;
  std::vector<unsigned long long> keys(npx);
  {
    DeviceGuard dg(ctx->device);
    cuda_check(cudaMemcpyAsync(keys.data(), ctx->base_keys.p, 8 * npx, cudaMemcpyDeviceToHost,
                               ctx->stream),
               "cudaMemcpyAsync keys");
    cuda_check(cudaStreamSynchronize(ctx->stream), "render_scene_keys");
  }
  const float far_f = static_cast<float>(k->far_m);
  for (size_t i = 0; i < npx; ++i) {
    const unsigned int bits = (unsigned int)(keys[i] >> 32);
    float z;
    std::memcpy(&z, &bits, 4);
    out[i] = z < far_f ? z : far_f;
  }
  ok(b3d_gpu_set_base_scene(ctx, nullptr, nullptr, 0));
}

// =================================================================== C ABI
extern "C" {

const char* b3d_version(void) { return "0.1.0-b200"; }

const char* b3d_last_error(void) { return g_last_error.c_str(); }

struct b3d_depth_image {
  uint32_t width = 0, height = 0;
  std::vector<float> depth;
};

b3d_status b3d_depth_image_create(uint32_t width, uint32_t height, const float* depth,
                                  b3d_depth_image** out) {
  return guarded([&] {
    check(out && depth && width > 0 && height > 0, "bad arguments");
    auto h = std::make_unique<b3d_depth_image>();
    h->width = width;
    h->height = height;
    h->depth.assign(depth, depth + static_cast<size_t>(width) * height);
    *out = h.release();
  });
}

// load_depth_image (io.cpp:104-116) builds the image without
// b3d_depth_image_create's argument checks: a 0 x N file loads (handle layer)
}  // extern "C"
b3d_depth_image* b3d200_depth_image_new(uint32_t width, uint32_t height,
                                        std::vector<float>&& depth) {
  auto h = std::make_unique<b3d_depth_image>();
  h->width = width;
  h->height = height;
  h->depth = std::move(depth);
  return h.release();
}
extern "C" {

uint32_t b3d_depth_image_width(const b3d_depth_image* img) { return img ? img->width : 0; }
uint32_t b3d_depth_image_height(const b3d_depth_image* img) { return img ? img->height : 0; }
const float* b3d_depth_image_data(const b3d_depth_image* img) {
  return img ? img->depth.data() : nullptr;
}
void b3d_depth_image_destroy(b3d_depth_image* img) { delete img; }

}  // extern "C"
namespace {
struct LoglikScratch {
  int device = -1;
  cudaStream_t st = nullptr;
  DevBuf img, res;
  PinnedBuf pin;
  ~LoglikScratch() {
    if (st) cudaStreamDestroy(st);  // thread exit: errors at teardown are moot
  }
};
LoglikScratch& loglik_scratch() {
  thread_local LoglikScratch s;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (s.device != dev) {  // first use on this thread, or the device changed
    if (s.st) cudaStreamDestroy(s.st);
    s.st = nullptr;
    for (DevBuf* b : {&s.img, &s.res}) {
      if (b->p) cudaFree(b->p);
      b->p = nullptr;
      b->bytes = 0;
    }
    cuda_check(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking), "cudaStreamCreate");
    s.device = dev;
  }
  return s;
}
}  // namespace
extern "C" {

b3d_status b3d_log_likelihood(const b3d_depth_image* observed, const b3d_depth_image* rendered,
                              const b3d_intrinsics* k, double p_outlier, double sigma_noise,
                              double sigma_max, int window, double* out) {
  return guarded([&] {
    check(observed && rendered && k && out, "bad arguments");
    validate_intrinsics(*k);  // from_c + visible_volume (b3d_capi.cpp:283-285)
    auto validate_noise = [&] {  // likelihood.cpp:21-26
      require(sigma_max > 0, ErrorCode::invalid, "sigma_max must be positive");
      require(sigma_noise > 0, ErrorCode::invalid, "sigma_noise must be positive");
      require(p_outlier >= 0 && p_outlier <= 1, ErrorCode::invalid,
              "p_outlier must be in [0,1]");
    };
    const float far_f = static_cast<float>(k->far_m);
    size_t rend_valid = 0;
    for (float z : rendered->depth) rend_valid += z < far_f;
    if (window >= 0) {  // ObservationCache::build, then windowed_log_likelihood_multi
      require(observed->width == k->width && observed->height == k->height,
              ErrorCode::invalid, "observation dimensions do not match intrinsics");
      require(observed->width == rendered->width && observed->height == rendered->height,
              ErrorCode::invalid, "windowed likelihood: image dimension mismatch");
      validate_noise();
      require(rend_valid > 0, ErrorCode::invalid, "windowed likelihood: empty rendered cloud");
    } else {  // depth_to_cloud(rendered), depth_to_cloud(observed) -- gcc's
              // right-to-left argument order -- then full_log_likelihood
      require(rendered->width == k->width && rendered->height == k->height,
              ErrorCode::invalid, "depth_to_cloud: image dimensions do not match intrinsics");
      require(observed->width == k->width && observed->height == k->height,
              ErrorCode::invalid, "depth_to_cloud: image dimensions do not match intrinsics");
      validate_noise();
      require(rend_valid > 0, ErrorCode::invalid, "full_log_likelihood: empty rendered cloud");
    }
    // the calling thread's device state, kept across calls: buffers that
    // only grow, page-locked staging, a private stream (one copy in, one
    // launch, one copy out, one synchronisation per call)
    LoglikScratch& s = loglik_scratch();
    const size_t npx = (size_t)k->width * k->height;
    s.img.ensure(npx * 8);
    s.res.ensure(32 + 8 * (size_t)image_loglik_partials((int)npx));
    s.pin.ensure(npx * 8 + 32);
    float* h_img = s.pin.as<float>();
    std::memcpy(h_img, observed->depth.data(), npx * 4);
    std::memcpy(h_img + npx, rendered->depth.data(), npx * 4);
    cuda_check(cudaMemcpyAsync(s.img.p, h_img, npx * 8, cudaMemcpyHostToDevice, s.st),
               "cudaMemcpyAsync");
    char* d_res = s.res.as<char>();
    cuda_check(launch_image_loglik(s.img.as<float>(), s.img.as<float>() + npx, (int)k->width,
                                   (int)k->height, k->fx, k->fy, k->cx, k->cy,
                                   static_cast<float>(k->far_m), p_outlier, sigma_noise,
                                   sigma_max, visible_volume(*k), window, 0,
                                   reinterpret_cast<double*>(d_res + 32),
                                   reinterpret_cast<double*>(d_res + 16),
                                   reinterpret_cast<int*>(d_res + 24), s.st),
               "image_loglik launch");
    char* h_res = s.pin.as<char>() + npx * 8;
    cuda_check(cudaMemcpyAsync(h_res, d_res + 16, 16, cudaMemcpyDeviceToHost, s.st),
               "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(s.st), "b3d_log_likelihood");
    double v = 0;
    int cnt = 0;
    std::memcpy(&v, h_res, 8);
    std::memcpy(&cnt, h_res + 8, 4);
    if (window >= 0)
      require(cnt > 0, ErrorCode::invalid, "windowed likelihood: empty rendered cloud");
    else
      require(cnt > 0, ErrorCode::invalid, "full_log_likelihood: empty rendered cloud");
    *out = v;
  });
}

b3d_status b3d_gpu_context_create(int device, b3d_gpu_context** out) {
  return guarded([&] {
    check(out != nullptr, "bad arguments");
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    require(device >= 0 && device < n, ErrorCode::invalid, "gpu context: no such device");
    DeviceGuard dg(device);
    auto c = std::make_unique<b3d_gpu_context>();
    c->device = device;
    cuda_check(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device),
               "cudaDeviceGetAttribute");
    // blocking: ordered with the legacy default stream (b3d_b200.h)
    cuda_check(cudaStreamCreateWithFlags(&c->own, cudaStreamDefault), "cudaStreamCreate");
    c->stream = c->own;
    c->obs_count.ensure(sizeof(int) * obs_count_ints());
    cuda_check(cudaMemset(c->obs_count.p, 0, sizeof(int) * obs_count_ints()), "cudaMemset");
    static_assert(sizeof(KStageResult) <= 64, "rng slot at +64");
    c->result.ensure(128);  // KStageResult, then an Rng state at +64
    c->rng.ensure(5 * sizeof(uint64_t));
    *out = c.release();
  });
}

void b3d_gpu_context_destroy(b3d_gpu_context* ctx) {
  if (ctx && ctx->e2e.exec) cudaGraphExecDestroy(ctx->e2e.exec);
  if (!ctx) return;
  DeviceGuard dg(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStream_t own = ctx->own;
  delete ctx;  // device buffers are released with the device current
  if (own) cudaStreamDestroy(own);
}

b3d_status b3d_gpu_set_stream(b3d_gpu_context* ctx, void* cuda_stream) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx != nullptr, "bad arguments");
    ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own;
  });
}

b3d_status b3d_gpu_synchronize(b3d_gpu_context* ctx) {
  return guarded([&] {
    check(ctx != nullptr, "bad arguments");
    DeviceGuard dg(ctx->device);
    cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  });
}

b3d_status b3d_mesh_cull_sign(const double* vertices, uint64_t n_vertices,
                              const uint32_t* triangles, uint64_t n_triangles, int32_t* out) {
  return guarded([&] {
    check(vertices && triangles && out, "bad arguments");
    for (uint64_t i = 0; i < 3 * n_triangles; ++i)
      check(triangles[i] < n_vertices, "mesh: triangle index out of range");
    *out = closed_mesh_cull_sign(vertices, triangles, n_triangles);
  });
}

b3d_status b3d_gpu_set_score_peers(b3d_gpu_context* ctx, const uint64_t* peer_ptrs,
                                   uint32_t n_peers, uint64_t offset, uint64_t capacity) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx != nullptr && (n_peers == 0 || peer_ptrs != nullptr), "bad arguments");
    require(n_peers <= 8, ErrorCode::invalid, "score peers: at most 8 ranks");
    for (uint32_t r = 0; r < n_peers; ++r)
      check(peer_ptrs[r] != 0, "score peers: null peer array");
    for (uint32_t r = 0; r < 8; ++r)
      ctx->score_peers[r] = r < n_peers ? reinterpret_cast<double*>(peer_ptrs[r]) : nullptr;
    ctx->n_score_peers = (int)n_peers;
    ctx->score_peer_offset = (long long)offset;
    ctx->score_peer_cap = (long long)capacity;
  });
}

b3d_status b3d_gpu_shard_barrier(b3d_gpu_context* ctx, const uint64_t* signal_ptrs,
                                 uint32_t n_ranks, uint32_t rank, uint64_t epoch) {
  return guarded([&] {
    check(ctx && signal_ptrs && n_ranks >= 1 && n_ranks <= 8 && rank < n_ranks && epoch > 0,
          "bad arguments");
    DeviceGuard dg(ctx->device);
    KBarrier b{};
    for (uint32_t r = 0; r < n_ranks; ++r) {
      check(signal_ptrs[r] != 0, "shard barrier: null signal pad");
      b.sig[r] = reinterpret_cast<unsigned long long*>(signal_ptrs[r]);
    }
    b.n_ranks = (int)n_ranks;
    b.rank = (int)rank;
    b.epoch = epoch;
    cuda_check(launch_shard_barrier(b, ctx->stream), "shard barrier launch");
  });
}

b3d_status b3d_gpu_test_exchange_emulation(b3d_gpu_context* ctx, uint32_t n_ranks,
                                           uint32_t rounds, int32_t double_buffered,
                                           uint64_t hold_ns, uint32_t* errors) {
  return guarded([&] {
    check(ctx && errors && n_ranks >= 1 && n_ranks <= 8 && rounds >= 1, "bad arguments");
    check(hold_ns <= 100000000ull, "exchange emulation: hold at most 0.1 s");
    DeviceGuard dg(ctx->device);
    DevBuf sig, arr, err;
    sig.ensure(8 * 64);
    arr.ensure(8 * 8 * 2 * 8);
    err.ensure(4);
    cuda_check(cudaMemsetAsync(sig.p, 0, 8 * 64, ctx->stream), "cudaMemsetAsync");
    cuda_check(cudaMemsetAsync(arr.p, 0xff, 8 * 8 * 2 * 8, ctx->stream), "cudaMemsetAsync");
    cuda_check(cudaMemsetAsync(err.p, 0, 4, ctx->stream), "cudaMemsetAsync");
    cuda_check(launch_exchange_emulation(sig.as<unsigned long long>(), arr.as<double>(),
                                         (int)n_ranks, (int)rounds, double_buffered ? 1 : 0,
                                         hold_ns, err.as<unsigned int>(), ctx->stream),
               "exchange emulation launch");
    cuda_check(cudaMemcpyAsync(errors, err.p, 4, cudaMemcpyDeviceToHost, ctx->stream),
               "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(ctx->stream), "exchange emulation");
  });
}

b3d_status b3d_gpu_enumerate_shard(b3d_gpu_context* ctx, int32_t mesh_id, const float* depth,
                                   const b3d_pose* poses, const b3d_pose_grid* grid,
                                   uint64_t n_local, const b3d_shard_exchange* ex,
                                   uint64_t* rng_state, b3d_stage_result* out) {
  return guarded([&] {
    check(ctx && ex && out && n_local > 0 && ((poses != nullptr) != (grid != nullptr)),
          "bad arguments");
    check(ex->n_ranks >= 1 && ex->n_ranks <= 8 && ex->rank < ex->n_ranks && ex->epoch > 0,
          "shard exchange: bad ranks / epoch");
    check(ex->offset + n_local <= ex->n_total, "shard exchange: shard outside the global array");
    for (uint32_t r = 0; r < ex->n_ranks; ++r)
      check(ex->scores[r] != 0 && ex->signals[r] != 0, "shard exchange: null peer buffer");
    if (depth) {
      const b3d_status st = b3d_gpu_set_observation(ctx, depth);
      if (st != B3D_OK) throw Error(ErrorCode::invalid, b3d_last_error());
    }
    require_ready(ctx, true, true);
    DeviceGuard dg(ctx->device);
    const long long nn = ctx->spec.n_cols;
    const long long half = (long long)(ex->epoch & 1) * (long long)ex->n_total * nn;
    double* own = reinterpret_cast<double*>(ex->scores[ex->rank]) + half;
    // this rank's scores land in its own array directly; the kernel stores
    // them into the other ranks' arrays (the fused all-gather)
    double* const saved[8] = {ctx->score_peers[0], ctx->score_peers[1], ctx->score_peers[2],
                              ctx->score_peers[3], ctx->score_peers[4], ctx->score_peers[5],
                              ctx->score_peers[6], ctx->score_peers[7]};
    const int saved_n = ctx->n_score_peers;
    const long long saved_off = ctx->score_peer_offset, saved_cap = ctx->score_peer_cap;
    int np = 0;
    for (uint32_t r = 0; r < ex->n_ranks; ++r)
      if (r != ex->rank) ctx->score_peers[np++] = reinterpret_cast<double*>(ex->scores[r]) + half;
    ctx->n_score_peers = np;
    ctx->score_peer_offset = (long long)ex->offset;
    ctx->score_peer_cap = (long long)ex->n_total * nn;
    try {
      if (poses)
        score_common(ctx, mesh_id, poses, nullptr, n_local, own + (long long)ex->offset * nn,
                     nullptr, nullptr, 0, 0, nullptr, nullptr, true);
      else {
        // a grid of n_total rows is the global one (this shard = rows offset +
        // i); any other size is this rank's own grid (rows i)
        const uint64_t gn = (uint64_t)grid->count[0] * grid->count[1] * grid->count[2] *
                            (grid->mode == B3D_GRID_PRODUCT ? grid->n_rot : 1);
        score_common(ctx, mesh_id, nullptr, grid, n_local, own + (long long)ex->offset * nn,
                     nullptr, nullptr, gn == ex->n_total ? ex->offset : 0, gn, nullptr, nullptr,
                     true);
      }
    } catch (...) {
      for (int r = 0; r < 8; ++r) ctx->score_peers[r] = saved[r];
      ctx->n_score_peers = saved_n;
      ctx->score_peer_offset = saved_off;
      ctx->score_peer_cap = saved_cap;
      throw;
    }
    for (int r = 0; r < 8; ++r) ctx->score_peers[r] = saved[r];
    ctx->n_score_peers = saved_n;
    ctx->score_peer_offset = saved_off;
    ctx->score_peer_cap = saved_cap;
    KBarrier b{};
    for (uint32_t r = 0; r < ex->n_ranks; ++r)
      b.sig[r] = reinterpret_cast<unsigned long long*>(ex->signals[r]);
    b.n_ranks = (int)ex->n_ranks;
    b.rank = (int)ex->rank;
    b.epoch = ex->epoch;
    cuda_check(launch_shard_barrier(b, ctx->stream), "shard barrier launch");
    // stage reduction of the complete array; result + Rng come back in one copy
    ctx->result.ensure(128);
    char* tail = static_cast<char*>(ctx->result.p);
    const bool dev_out = is_device_ptr(out);
    const bool dev_rng = rng_state && is_device_ptr(rng_state);
    KStageResult* d_out = dev_out ? reinterpret_cast<KStageResult*>(out)
                                  : reinterpret_cast<KStageResult*>(tail);
    unsigned long long* d_rng = nullptr;
    if (rng_state) {
      if (dev_rng) {
        d_rng = reinterpret_cast<unsigned long long*>(rng_state);
      } else {
        d_rng = reinterpret_cast<unsigned long long*>(tail + 64);
        cuda_check(cudaMemcpyAsync(d_rng, rng_state, 40, cudaMemcpyHostToDevice, ctx->stream),
                   "cudaMemcpyAsync rng");
      }
    }
    cuda_check(launch_stage_reduce(own, (long long)ex->n_total, (int)nn, 0, d_rng, d_out, nullptr,
                                   ctx->stream, stage_scratch(ctx, (long long)ex->n_total)),
               "stage_reduce launch");
    if (!dev_out || (rng_state && !dev_rng)) {
      ctx->pin_scores.ensure(128);
      cuda_check(cudaMemcpyAsync(ctx->pin_scores.p, tail, 104, cudaMemcpyDeviceToHost,
                                 ctx->stream),
                 "cudaMemcpyAsync result");
      cuda_check(cudaStreamSynchronize(ctx->stream), "enumerate_shard");
      const char* pin = static_cast<const char*>(ctx->pin_scores.p);
      if (!dev_out) std::memcpy(out, pin, sizeof(KStageResult));
      if (rng_state && !dev_rng) std::memcpy(rng_state, pin + 64, 40);
    }
  });
}

b3d_status b3d_gpu_set_culling(b3d_gpu_context* ctx, int enable) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx != nullptr, "bad arguments");
    ctx->culling = enable != 0;
  });
}

b3d_status b3d_gpu_mesh_cull_sign(const b3d_gpu_context* ctx, int32_t mesh_id, int32_t* out) {
  return guarded([&] {
    check(ctx && out, "bad arguments");
    *out = get_mesh(ctx, mesh_id).cull;
  });
}

b3d_status b3d_gpu_set_camera(b3d_gpu_context* ctx, const b3d_intrinsics* k,
                              const b3d_pose* camera) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx && k, "bad arguments");
    validate_intrinsics(*k);
    require(k->width <= 16384 && k->height <= 16384, ErrorCode::invalid,
            "gpu context: image dimensions above 16384 are not supported");
    if (ctx->has_camera && (k->width != ctx->k.width || k->height != ctx->k.height))
      ctx->has_obs = false;
    ctx->k = *k;
    const KPose cam = camera ? pose_from_c(*camera) : KPose{1, 0, 0, 0, 0, 0, 0};
    ctx->w2c = pose_inverse(cam);
    ctx->has_camera = true;
  });
}

b3d_status b3d_gpu_upload_mesh(b3d_gpu_context* ctx, const double* vertices,
                               uint64_t n_vertices, const uint32_t* triangles,
                               uint64_t n_triangles, int32_t* out_mesh_id) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx && vertices && triangles && out_mesh_id, "bad arguments");
    check(n_vertices > 0 && n_triangles > 0, "mesh: empty");
    check(n_vertices < (1u << 30) && n_triangles < (1u << 30), "mesh: too large");
    for (uint64_t i = 0; i < 3 * n_triangles; ++i)
      check(triangles[i] < n_vertices, "mesh: triangle index out of range");
    for (uint64_t i = 0; i < 3 * n_vertices; ++i)
      check(std::isfinite(vertices[i]), "mesh: non-finite vertex coordinate");
    DeviceGuard dg(ctx->device);
    auto m = std::make_unique<Mesh>();
    m->nv = (int)n_vertices;
    m->nt = (int)n_triangles;
    m->cull = closed_mesh_cull_sign(vertices, triangles, n_triangles);
    for (uint64_t i = 0; i < n_vertices; ++i)
      m->radius = std::max(m->radius, std::sqrt(sq3(vertices + 3 * i)));
    build_score_order(vertices, triangles, n_triangles, m->cull, *m);
    m->verts.ensure(24 * n_vertices);
    m->tris.ensure(16 * n_triangles);
    // triangles padded to 16 bytes: one 128-bit load per triangle
    std::vector<uint32_t> padded(4 * n_triangles, 0u);
    for (uint64_t i = 0; i < n_triangles; ++i)
      for (int j = 0; j < 3; ++j) padded[4 * i + j] = triangles[3 * i + j];
    cuda_check(cudaMemcpy(m->verts.p, vertices, 24 * n_vertices, cudaMemcpyHostToDevice),
               "cudaMemcpy");
    cuda_check(cudaMemcpy(m->tris.p, padded.data(), 16 * n_triangles, cudaMemcpyHostToDevice),
               "cudaMemcpy");
    ctx->meshes.push_back(std::move(m));
    *out_mesh_id = (int32_t)(ctx->meshes.size() - 1);
  });
}

b3d_status b3d_gpu_set_observation(b3d_gpu_context* ctx, const float* depth) {
  return guarded([&] {
    check(ctx && depth, "bad arguments");
    require(ctx->has_camera, ErrorCode::invalid, "gpu context: intrinsics not set");
    DeviceGuard dg(ctx->device);
    const b3d_intrinsics& k = ctx->k;
    const size_t npx = (size_t)k.width * k.height;
    bool host = false;
    const float* d = static_cast<const float*>(stage_in(ctx, ctx->obs_depth, depth, npx * 4, &host));
    ctx->obs_pts.ensure(npx * sizeof(float4));
    cuda_check(launch_obs_prepare(d, (int)k.width, (int)k.height, static_cast<float>(k.far_m),
                                  (float)k.cx, (float)k.cy, (float)(1.0 / k.fx),
                                  (float)(1.0 / k.fy), ctx->obs_pts.as<float4>(),
                                  ctx->obs_count.as<int>(), ctx->stream),
               "obs_prepare launch");
    // pageable host memory must be consumed before returning; pinned host
    // memory is read in stream order (see b3d_b200.h)
    if (host && !is_pinned_host(depth))
      cuda_check(cudaStreamSynchronize(ctx->stream), "set_observation");
    ctx->has_obs = true;
    ++ctx->obs_version;
  });
}

b3d_status b3d_gpu_set_likelihood(b3d_gpu_context* ctx, const b3d_noise* noise,
                                  uint32_t n_noise, double sigma_max, int window,
                                  int prefactor) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx && noise, "bad arguments");
    require(ctx->has_camera, ErrorCode::invalid, "gpu context: intrinsics not set");
    ctx->spec = make_spec(ctx->k, noise, n_noise, sigma_max, window, prefactor, true);
    try {
      ctx->cam_spec = make_spec(ctx->k, noise, n_noise, sigma_max, window, prefactor, false);
      ctx->cam_spec_err.clear();
    } catch (const Error& e) {
      ctx->cam_spec = LikSpec{};
      ctx->cam_spec_err = e.what();
    }
    ctx->lik = ctx->spec.chunks.empty() ? KLik{} : ctx->spec.chunks[0].lik;
    ctx->lik.window = std::max(window, 0);
    ctx->sigma_max = sigma_max;
    ctx->prefactor = prefactor;
    ctx->has_lik = true;
  });
}

b3d_status b3d_gpu_score_poses(b3d_gpu_context* ctx, int32_t mesh_id, const b3d_pose* poses,
                               uint64_t n, double* scores, uint8_t* status) {
  return guarded([&] {
    check(poses != nullptr, "bad arguments");
    score_common(ctx, mesh_id, poses, nullptr, n, scores, status, nullptr, 0, 0, nullptr,
                 nullptr, true);
  });
}

b3d_status b3d_gpu_score_grid(b3d_gpu_context* ctx, int32_t mesh_id, const b3d_pose_grid* grid,
                              double* scores, uint8_t* status) {
  return guarded([&] {
    check(grid != nullptr, "bad arguments");
    const uint64_t nt = (uint64_t)grid->count[0] * grid->count[1] * grid->count[2];
    const uint64_t n = grid->mode == B3D_GRID_PRODUCT ? nt * grid->n_rot : nt;
    score_common(ctx, mesh_id, nullptr, grid, n, scores, status, nullptr, 0, 0, nullptr,
                 nullptr, true);
  });
}

b3d_status b3d_gpu_render_poses(b3d_gpu_context* ctx, int32_t mesh_id, const b3d_pose* poses,
                                uint64_t n, float* depth, int32_t* draw_index) {
  return guarded([&] {
    require_ready(ctx, false, false);
    check(poses && depth && n > 0, "bad arguments");
    DeviceGuard dg(ctx->device);
    const Mesh& m = get_mesh(ctx, mesh_id);
    KParams p = base_params(ctx, m);
    bool host_in = false;
    p.poses = static_cast<const KPose*>(
        stage_in(ctx, ctx->in_stage, poses, sizeof(b3d_pose) * n, &host_in));
    p.n_hyp = (long long)n;
    p.lik.n_noise = 0;  // render only
    attach_base(ctx, p);
    const size_t npx = (size_t)ctx->k.width * ctx->k.height;
    const bool dev_d = is_device_ptr(depth);
    const bool dev_i = draw_index && is_device_ptr(draw_index);
    if (dev_d) {
      p.out_depth = depth;
    } else {
      ctx->out_stage.ensure(4 * npx * n);
      p.out_depth = ctx->out_stage.as<float>();
    }
    if (draw_index) {
      if (dev_i) {
        p.out_ids = draw_index;
      } else {
        ctx->out_stage2.ensure(4 * npx * n);
        p.out_ids = ctx->out_stage2.as<int32_t>();
      }
    }
    bool sync = host_in;
    if (draw_index) {
      LaunchPlan lp = plan_launch<true, false, true>(ctx, m, (long long)n);
      p.zscratch = ctx->zscratch.as<unsigned long long>();
      p.vscratch = ctx->vscratch.as<double>();
      p.vcap = lp.vcap;
      p.zcap = lp.zcap;
      p.zstride = lp.zstride;
      cuda_check(launch_render_score<true, false, true>(p, lp.grid, lp.smem, ctx->stream),
                 "render launch");
    } else {
      LaunchPlan lp = plan_launch<false, false, true>(ctx, m, (long long)n);
      p.zscratch = ctx->zscratch.as<unsigned long long>();
      p.vscratch = ctx->vscratch.as<double>();
      p.vcap = lp.vcap;
      p.zcap = lp.zcap;
      p.zstride = lp.zstride;
      cuda_check(launch_render_score<false, false, true>(p, lp.grid, lp.smem, ctx->stream),
                 "render launch");
    }
    if (!dev_d) {
      finish_copy_out(ctx, depth, p.out_depth, 4 * npx * n);
      sync = true;
    }
    if (draw_index && !dev_i) {
      finish_copy_out(ctx, draw_index, p.out_ids, 4 * npx * n);
      sync = true;
    }
    if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "render_poses");
  });
}

b3d_status b3d_rotated_bounds(const double aabb_min[3], const double aabb_max[3], int32_t face,
                              double lo[3], double hi[3]) {
  return guarded([&] {
    check(aabb_min && aabb_max && lo && hi, "bad arguments");
    check(face >= 1 && face <= 6, "face must be in 1..6");
    rotated_bounds(aabb_min, aabb_max, face, lo, hi);
  });
}

b3d_status b3d_box_mesh(const double lo[3], const double hi[3], double vertices[24],
                        uint32_t triangles[36]) {
  return guarded([&] {
    check(lo && hi && vertices && triangles, "bad arguments");
    // scene_graph.cpp:37-58: corners by bit layout (x=1, y=2, z=4), outward
    // quads split (0,1,2), (0,2,3)
    for (int i = 0; i < 8; ++i) {
      vertices[3 * i + 0] = (i & 1) ? hi[0] : lo[0];
      vertices[3 * i + 1] = (i & 2) ? hi[1] : lo[1];
      vertices[3 * i + 2] = (i & 4) ? hi[2] : lo[2];
    }
    static const uint32_t quads[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4},
                                         {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
    for (int f = 0; f < 6; ++f) {
      const uint32_t* q = quads[f];
      const uint32_t t[6] = {q[0], q[1], q[2], q[0], q[2], q[3]};
      for (int j = 0; j < 6; ++j) triangles[6 * f + j] = t[j];
    }
  });
}

b3d_status b3d_contact_to_pose(double table_w, double table_h, const double aabb_min[3],
                               const double aabb_max[3], int32_t face, double dx, double dy,
                               double dtheta, b3d_pose* out) {
  return guarded([&] {
    check(aabb_min && aabb_max && out, "bad arguments");
    const KPose k =
        contact_to_pose_host(table_w, table_h, aabb_min, aabb_max, face, dx, dy, dtheta);
    *out = b3d_pose{k.qw, k.qx, k.qy, k.qz, k.tx, k.ty, k.tz};
  });
}

b3d_status b3d_camera_pose_from_spherical(double distance, double azimuth, double altitude,
                                          b3d_pose* out) {
  return guarded([&] {
    check(out != nullptr, "bad arguments");
    const KPose k = camera_from_spherical(distance, azimuth, altitude);
    *out = b3d_pose{k.qw, k.qx, k.qy, k.qz, k.tx, k.ty, k.tz};
  });
}

int b3d_camera_pose_to_spherical(const b3d_pose* pose, double tol, double* distance,
                                 double* azimuth, double* altitude) {
  if (!pose || !distance || !azimuth || !altitude) return 0;
  try {
    const KPose k{pose->qw, pose->qx, pose->qy, pose->qz, pose->tx, pose->ty, pose->tz};
    return camera_to_spherical(k, tol, *distance, *azimuth, *altitude) ? 1 : 0;
  } catch (...) {
    return 0;
  }
}

b3d_status b3d_gpu_set_camera_scene(b3d_gpu_context* ctx, const int32_t* mesh_ids,
                                    const b3d_pose* model_to_world, uint32_t n) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    check(ctx && mesh_ids && model_to_world, "bad arguments");
    require(n >= 1, ErrorCode::invalid, "camera scene: at least one instance");
    for (uint32_t i = 0; i < n; ++i) get_mesh(ctx, mesh_ids[i]);  // ids valid
    DeviceGuard dg(ctx->device);
    std::vector<b3d_gpu_context::CamGroup> groups;
    long long draw = 0;
    for (uint32_t g0 = 0; g0 < n; g0 += (uint32_t)kMaxInst) {
      const uint32_t gn = std::min<uint32_t>((uint32_t)kMaxInst, n - g0);
      b3d_gpu_context::CamGroup grp;
      grp.n = (int)gn;
      grp.draw_base = (uint32_t)draw;
      auto sm = std::make_unique<Mesh>();
      long long nv = 0, nt = 0;
      int sign = 2;
      for (uint32_t i = 0; i < gn; ++i) {
        const Mesh& m = get_mesh(ctx, mesh_ids[g0 + i]);
        grp.v0[i] = (int)nv;
        nv += m.nv;
        nt += m.nt;
        sign = (sign == 2 || sign == m.cull) ? m.cull : 0;
      }
      require(nv < (1ll << 30) && nt < (1ll << 30) && draw + nt < (1ll << 31),
              ErrorCode::invalid, "camera scene: too large");
      for (uint32_t i = gn; i <= (uint32_t)kMaxInst; ++i) grp.v0[i] = (int)nv;
      sm->nv = (int)nv;
      sm->nt = (int)nt;
      sm->cull = sign == 2 ? 0 : sign;  // per-triangle culling only if every mesh shares a sign
      sm->verts.ensure(24 * nv);
      sm->tris.ensure(16 * nt);
      std::vector<uint32_t> tri(4 * nt);
      long long vo = 0, to = 0;
      for (uint32_t i = 0; i < gn; ++i) {
        const Mesh& m = get_mesh(ctx, mesh_ids[g0 + i]);
        cuda_check(cudaMemcpy(sm->verts.as<char>() + 24 * vo, m.verts.p, 24ull * m.nv,
                              cudaMemcpyDeviceToDevice),
                   "cudaMemcpy");
        cuda_check(cudaMemcpy(tri.data() + 4 * to, m.tris.p, 16ull * m.nt,
                              cudaMemcpyDeviceToHost),
                   "cudaMemcpy");
        for (long long k = 0; k < m.nt; ++k)
          for (int j = 0; j < 3; ++j) tri[4 * (to + k) + j] += (uint32_t)vo;
        vo += m.nv;
        to += m.nt;
        const b3d_pose& q = model_to_world[g0 + i];
        grp.pose[i] = KPose{q.qw, q.qx, q.qy, q.qz, q.tx, q.ty, q.tz};
      }
      cuda_check(cudaMemcpy(sm->tris.p, tri.data(), 16ull * nt, cudaMemcpyHostToDevice),
                 "cudaMemcpy");
      grp.mesh = std::move(sm);
      draw += nt;
      groups.push_back(std::move(grp));
    }
    ctx->cam_groups = std::move(groups);
  });
}

b3d_status b3d_gpu_render_cameras(b3d_gpu_context* ctx, const b3d_pose* cameras, uint64_t n,
                                  float* depth, int32_t* draw_index) {
  return guarded([&] {
    require_ready(ctx, false, false);
    check(cameras && depth && n > 0, "bad arguments");
    require(!ctx->cam_groups.empty(), ErrorCode::invalid, "gpu context: camera scene not set");
    DeviceGuard dg(ctx->device);
    const Mesh& m = *ctx->cam_groups.front().mesh;
    KParams p = base_params(ctx, m);
    cam_params(ctx, p, ctx->cam_groups.front());
    bool host_in = false;
    p.cams = static_cast<const KPose*>(
        stage_in(ctx, ctx->in_stage, cameras, sizeof(b3d_pose) * n, &host_in));
    p.n_hyp = (long long)n;
    p.lik.n_noise = 0;  // render only
    const size_t npx = (size_t)ctx->k.width * ctx->k.height;
    const bool dev_d = is_device_ptr(depth);
    const bool dev_i = draw_index && is_device_ptr(draw_index);
    if (dev_d) {
      p.out_depth = depth;
    } else {
      ctx->out_stage.ensure(4 * npx * n);
      p.out_depth = ctx->out_stage.as<float>();
    }
    if (draw_index) {
      if (dev_i) {
        p.out_ids = draw_index;
      } else {
        ctx->out_stage2.ensure(4 * npx * n);
        p.out_ids = ctx->out_stage2.as<int32_t>();
      }
    }
    if (ctx->cam_groups.size() > 1) {  // merged per-group renders
      if (draw_index) {
        ctx->cam_keys.ensure(8 * npx * n);
        render_camera_groups(ctx, p.cams, (long long)n, nullptr,
                             ctx->cam_keys.as<unsigned long long>());
        cuda_check(launch_keys_to_depth_ids(ctx->cam_keys.as<unsigned long long>(), npx * n,
                                            static_cast<float>(ctx->k.far_m), p.out_depth,
                                            p.out_ids, ctx->stream),
                   "keys_to_depth_ids launch");
      } else {
        render_camera_groups(ctx, p.cams, (long long)n, p.out_depth, nullptr);
      }
    } else if (draw_index) {
      LaunchPlan lp = plan_launch<true, false, true>(ctx, m, (long long)n);
      p.zscratch = ctx->zscratch.as<unsigned long long>();
      p.vscratch = ctx->vscratch.as<double>();
      p.vcap = lp.vcap;
      p.zcap = lp.zcap;
      p.zstride = lp.zstride;
      cuda_check(launch_render_score<true, false, true>(p, lp.grid, lp.smem, ctx->stream),
                 "render launch (cameras)");
    } else {
      LaunchPlan lp = plan_launch<false, false, true>(ctx, m, (long long)n);
      p.zscratch = ctx->zscratch.as<unsigned long long>();
      p.vscratch = ctx->vscratch.as<double>();
      p.vcap = lp.vcap;
      p.zcap = lp.zcap;
      p.zstride = lp.zstride;
      cuda_check(launch_render_score<false, false, true>(p, lp.grid, lp.smem, ctx->stream),
                 "render launch (cameras)");
    }
    bool sync = host_in;
    if (!dev_d) {
      finish_copy_out(ctx, depth, p.out_depth, 4 * npx * n);
      sync = true;
    }
    if (draw_index && !dev_i) {
      finish_copy_out(ctx, draw_index, p.out_ids, 4 * npx * n);
      sync = true;
    }
    if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "render_cameras");
  });
}

b3d_status b3d_gpu_score_cameras(b3d_gpu_context* ctx, const b3d_pose* cameras, uint64_t n,
                                 double* scores, uint8_t* status) {
  return guarded([&] {
    require_ready(ctx, true, true);
    check(cameras && scores && n > 0, "bad arguments");
    require(!ctx->cam_groups.empty(), ErrorCode::invalid, "gpu context: camera scene not set");
    DeviceGuard dg(ctx->device);
    bool host_in = false;
    const KPose* cams = static_cast<const KPose*>(
        stage_in(ctx, ctx->in_stage, cameras, sizeof(b3d_pose) * n, &host_in));
    require(ctx->cam_spec_err.empty(), ErrorCode::invalid, ctx->cam_spec_err);
    const int nn = ctx->cam_spec.n_cols;
    const bool dev_scores = is_device_ptr(scores);
    const bool dev_status = status && is_device_ptr(status);
    double* d_scores = scores;
    uint8_t* d_status = status;
    if (!dev_scores) {
      ctx->out_stage.ensure(sizeof(double) * n * nn);
      d_scores = ctx->out_stage.as<double>();
    }
    if (status && !dev_status) {
      ctx->out_stage2.ensure(n);
      d_status = ctx->out_stage2.as<uint8_t>();
    }
    launch_score_cameras(ctx, cams, (long long)n, d_scores, d_status);
    bool sync = host_in;
    if (!dev_scores) {
      finish_copy_out(ctx, scores, d_scores, sizeof(double) * n * nn);
      sync = true;
    }
    if (status && !dev_status) {
      finish_copy_out(ctx, status, d_status, n);
      sync = true;
    }
    if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "score_cameras");
  });
}

b3d_status b3d_gpu_track_camera(b3d_gpu_context* ctx, const float* frames, uint32_t n_frames,
                                const b3d_pose* initial, const b3d_track_search* search,
                                b3d_pose* out_poses, double* out_frame_ms) {
  return guarded([&] {
    check(ctx && frames && initial && search && out_poses, "bad arguments");
    require(n_frames >= 1, ErrorCode::invalid, "track_camera: empty frame list");
    require_ready(ctx, false, true);
    require(!ctx->cam_groups.empty(), ErrorCode::invalid, "gpu context: camera scene not set");
    require(ctx->cam_spec_err.empty(), ErrorCode::invalid, ctx->cam_spec_err);
    require(ctx->cam_spec.n_cols == 1, ErrorCode::invalid, "track_camera: one noise setting");
    const b3d_track_search& s = *search;
    // TrackSearch::validate (tracking.cpp:49-57)
    require(s.pos_extent > 0 && s.angle_extent > 0, ErrorCode::invalid,
            "track search: extents must be positive");
    require(s.points_per_dim >= 2, ErrorCode::invalid,
            "track search: need at least 2 points per dimension");
    require(s.refine_stages >= 0 && s.refine_factor > 1, ErrorCode::invalid,
            "track search: bad refinement settings");
    require(s.beam_width >= 1, ErrorCode::invalid, "track search: beam width must be >= 1");
    DeviceGuard dg(ctx->device);
    using Clock = std::chrono::steady_clock;
    auto frame_start = Clock::now();
    auto close_frame = [&](uint32_t f) {
      const double ms =
          std::chrono::duration<double, std::milli>(Clock::now() - frame_start).count();
      if (out_frame_ms) out_frame_ms[f] = std::max(ms, 1e-6);
      frame_start = Clock::now();
    };
    struct Sph {
      double d, az, alt;
    };
    struct Cand {
      Sph c;
      double score;
    };
    const KPose init{initial->qw, initial->qx, initial->qy, initial->qz,
                     initial->tx, initial->ty, initial->tz};
    Sph start{};
    require(camera_to_spherical(init, 1e-6, start.d, start.az, start.alt), ErrorCode::invalid,
            "track_camera: initial pose must look at the origin with up = +z");
    out_poses[0] = *initial;
    close_frame(0);
    std::vector<Cand> beam{{start, 0.0}};
    const int ppd = s.points_per_dim;
    const size_t n_grid = (size_t)ppd * ppd * ppd;
    const size_t npx = (size_t)ctx->k.width * ctx->k.height;
    const bool dev_frames = is_device_ptr(frames);
    std::vector<KPose> cams;
    std::vector<int> slot;
    ctx->c2f_scores.ensure(8 * n_grid);
    ctx->c2f_centers.ensure(sizeof(KPose) * n_grid);
    constexpr double kNegInf = -std::numeric_limits<double>::infinity();
    for (uint32_t f = 1; f < n_frames; ++f) {
      const float* fr = frames + (size_t)f * npx;
      {  // ObservationCache::build for this frame (tracking.cpp:112)
        bool host = false;
        const float* d = dev_frames ? fr
                                    : static_cast<const float*>(stage_in(
                                          ctx, ctx->obs_depth, fr, npx * 4, &host));
        ctx->obs_pts.ensure(npx * sizeof(float4));
        cuda_check(launch_obs_prepare(d, (int)ctx->k.width, (int)ctx->k.height,
                                      static_cast<float>(ctx->k.far_m), (float)ctx->k.cx,
                                      (float)ctx->k.cy, (float)(1.0 / ctx->k.fx),
                                      (float)(1.0 / ctx->k.fy), ctx->obs_pts.as<float4>(),
                                      ctx->obs_count.as<int>(), ctx->stream),
                   "obs_prepare launch");
        ctx->has_obs = true;
        ++ctx->obs_version;
      }
      // tables of ppd + ppd^2 + ... + ppd^(S+1) values per axis: the device
      // chain is used while that stays small (always at the defaults: 155)
      double tab_n = 0;
      for (int st = 0, w = 1; st <= s.refine_stages && tab_n <= (1 << 20); ++st) {
        w = (int)std::min<double>((double)w * ppd, 1 << 21);
        tab_n += w;
      }
      if (s.beam_width == 1 && tab_n <= (1 << 20) && ctx->cam_spec.single()) {
        // the frame's stages chained on the device (track.cu): every lattice
        // value the frame can visit and its sin / cos from this libm, one
        // upload, ppd^3 poses / score / argmax per stage, one read-back
        const Sph c0 = beam.front().c;
        const int S = s.refine_stages;
        std::vector<int> off(S + 2, 0);
        for (int st = 0, w = ppd; st <= S; ++st, w *= ppd) off[st + 1] = off[st] + w;
        const int n_tab = off[S + 1];
        ctx->trk_tab_pin.ensure(sizeof(double) * 7 * n_tab);
        double* tab = ctx->trk_tab_pin.as<double>();
        double* td = tab;
        double* taz = tab + n_tab;
        double* talt = tab + 2 * n_tab;
        double pe = s.pos_extent, ae = s.angle_extent;
        for (int st = 0; st <= S; ++st) {
          const int parents = st == 0 ? 1 : off[st] - off[st - 1];
          for (int q = 0; q < parents; ++q) {
            const double cd = st == 0 ? c0.d : td[off[st - 1] + q];
            const double caz = st == 0 ? c0.az : taz[off[st - 1] + q];
            const double calt = st == 0 ? c0.alt : talt[off[st - 1] + q];
            for (int i = 0; i < ppd; ++i) {
              const int o = off[st] + q * ppd + i;
              td[o] = lattice_at(cd, pe, ppd, i);
              taz[o] = lattice_at(caz, ae, ppd, i);
              talt[o] = lattice_at(calt, ae, ppd, i);
            }
          }
          pe /= s.refine_factor;
          ae /= s.refine_factor;
        }
        for (int o = 0; o < n_tab; ++o) {  // generative.cpp:40-43's trig, host libm
          tab[3 * n_tab + o] = std::cos(talt[o]);
          tab[4 * n_tab + o] = std::sin(talt[o]);
          tab[5 * n_tab + o] = std::cos(taz[o]);
          tab[6 * n_tab + o] = std::sin(taz[o]);
        }
        ctx->trk_tab.ensure(sizeof(double) * 7 * n_tab);
        ctx->trk_state.ensure(8 * sizeof(int));
        ctx->trk_valid.ensure(n_grid);
        ctx->trk_state_pin.ensure(8 * sizeof(int));
        cuda_check(cudaMemcpyAsync(ctx->trk_tab.p, tab, sizeof(double) * 7 * n_tab,
                                   cudaMemcpyHostToDevice, ctx->stream),
                   "cudaMemcpyAsync track tables");
        const KPose fallback = camera_from_spherical(c0.d, c0.az, c0.alt);
        int* dstate = ctx->trk_state.as<int>();
        for (int st = 0; st <= S; ++st) {  // stage 0's kernel also zeroes the state
          cuda_check(launch_cam_stage(ctx->trk_tab.as<double>(), n_tab, off[st], ppd, st == 0,
                                      ctx->c2f_scores.as<double>(),
                                      ctx->trk_valid.as<unsigned char>(), dstate,
                                      ctx->c2f_centers.as<KPose>(),
                                      ctx->trk_valid.as<unsigned char>(), fallback, ctx->stream),
                     "cam_stage launch");
          launch_score_cameras(ctx, ctx->c2f_centers.as<KPose>(), (long long)n_grid,
                               ctx->c2f_scores.as<double>(), nullptr, /*pdl=*/true);
        }
        cuda_check(launch_cam_argmax(ctx->c2f_scores.as<double>(),
                                     ctx->trk_valid.as<unsigned char>(), ppd, dstate,
                                     ctx->stream),
                   "cam_argmax launch");
        int* hs = ctx->trk_state_pin.as<int>();
        cuda_check(cudaMemcpyAsync(hs, dstate, 8 * sizeof(int), cudaMemcpyDeviceToHost,
                                   ctx->stream),
                   "cudaMemcpyAsync track state");
        cuda_check(cudaStreamSynchronize(ctx->stream), "track_camera frame");
        require(hs[4] == 0, ErrorCode::numeric, "track_camera: every candidate pose scored -inf");
        const Sph top{td[off[S] + hs[0]], taz[off[S] + hs[1]], talt[off[S] + hs[2]]};
        beam = {{top, 0.0}};
        const KPose cp = camera_from_spherical(top.d, top.az, top.alt);
        out_poses[f] = b3d_pose{cp.qw, cp.qx, cp.qy, cp.qz, cp.tx, cp.ty, cp.tz};
        close_frame(f);
        continue;
      }
      std::vector<Cand> next;
      for (const Cand& seed : beam) {
        Sph center = seed.c;
        double pe = s.pos_extent, ae = s.angle_extent;
        Cand stage_best{center, kNegInf};
        for (int st = 0; st <= s.refine_stages; ++st) {
          std::vector<Sph> grid;
          grid.reserve(n_grid);
          for (int i = 0; i < ppd; ++i)
            for (int j = 0; j < ppd; ++j)
              for (int k = 0; k < ppd; ++k)
                grid.push_back({lattice_at(center.d, pe, ppd, i), lattice_at(center.az, ae, ppd, j),
                                lattice_at(center.alt, ae, ppd, k)});
          // score_pose (tracking.cpp:100-108): out-of-range coordinates score -inf
          cams.clear();
          slot.assign(grid.size(), -1);
          for (size_t i = 0; i < grid.size(); ++i) {
            const Sph& g = grid[i];
            if (g.d <= 0 || g.alt <= 0 || g.alt >= kHalfPi) continue;
            slot[i] = (int)cams.size();
            cams.push_back(camera_from_spherical(g.d, g.az, g.alt));
          }
          std::vector<double> scores(grid.size(), kNegInf);
          if (!cams.empty()) {  // pinned staging: asynchronous copies, one sync per stage
            ctx->pin_cams.ensure(sizeof(KPose) * n_grid);
            ctx->pin_scores.ensure(8 * n_grid);
            std::copy(cams.begin(), cams.end(), ctx->pin_cams.as<KPose>());
            cuda_check(cudaMemcpyAsync(ctx->c2f_centers.p, ctx->pin_cams.p,
                                       sizeof(KPose) * cams.size(), cudaMemcpyHostToDevice,
                                       ctx->stream),
                       "cudaMemcpyAsync cameras");
            launch_score_cameras(ctx, ctx->c2f_centers.as<KPose>(), (long long)cams.size(),
                                 ctx->c2f_scores.as<double>(), nullptr);
            cuda_check(cudaMemcpyAsync(ctx->pin_scores.p, ctx->c2f_scores.p, 8 * cams.size(),
                                       cudaMemcpyDeviceToHost, ctx->stream),
                       "cudaMemcpyAsync scores");
            cuda_check(cudaStreamSynchronize(ctx->stream), "track_camera stage");
            const double* ds = ctx->pin_scores.as<double>();
            for (size_t i = 0; i < grid.size(); ++i)
              if (slot[i] >= 0) scores[i] = ds[slot[i]];
          }
          size_t best = 0;  // tracking.cpp:132-134 (strict >, first index)
          for (size_t i = 1; i < scores.size(); ++i)
            if (scores[i] > scores[best]) best = i;
          require(std::isfinite(scores[best]), ErrorCode::numeric,
                  "track_camera: every candidate pose scored -inf");
          center = grid[best];
          stage_best = {center, scores[best]};
          if (s.beam_width > 1 && st == s.refine_stages) {
            std::vector<size_t> order(grid.size());
            for (size_t i = 0; i < order.size(); ++i) order[i] = i;
            std::stable_sort(order.begin(), order.end(),
                             [&](size_t a, size_t b) { return scores[a] > scores[b]; });
            const size_t keep = std::min<size_t>((size_t)s.beam_width, order.size());
            for (size_t i = 0; i < keep; ++i) next.push_back({grid[order[i]], scores[order[i]]});
          }
          pe /= s.refine_factor;
          ae /= s.refine_factor;
        }
        if (s.beam_width == 1) next.push_back(stage_best);
      }
      std::stable_sort(next.begin(), next.end(),
                       [](const Cand& a, const Cand& b) { return a.score > b.score; });
      if (next.size() > (size_t)s.beam_width) next.resize(s.beam_width);
      beam = std::move(next);
      const Sph& top = beam.front().c;
      const KPose cp = camera_from_spherical(top.d, top.az, top.alt);
      out_poses[f] = b3d_pose{cp.qw, cp.qx, cp.qy, cp.qz, cp.tx, cp.ty, cp.tz};
      close_frame(f);
    }
  });
}

b3d_status b3d_gpu_stage_reduce(b3d_gpu_context* ctx, const double* scores, uint64_t n,
                                uint32_t stride, uint32_t col, uint64_t* rng_state,
                                b3d_stage_result* out, double* probs) {
  return guarded([&] {
    check(ctx && scores && out && n > 0, "bad arguments");
    check(stride >= 1 && col < stride, "stage_reduce: bad stride/column");
    DeviceGuard dg(ctx->device);
    bool host_in = false;
    const double* d_scores = static_cast<const double*>(
        stage_in(ctx, ctx->in_stage, scores, sizeof(double) * n * stride, &host_in));
    unsigned long long* d_rng = nullptr;
    const bool dev_rng = rng_state && is_device_ptr(rng_state);
    if (rng_state) {
      if (dev_rng) {
        d_rng = reinterpret_cast<unsigned long long*>(rng_state);
      } else {
        cuda_check(cudaMemcpyAsync(ctx->rng.p, rng_state, 40, cudaMemcpyHostToDevice,
                                   ctx->stream),
                   "cudaMemcpyAsync");
        d_rng = ctx->rng.as<unsigned long long>();
        host_in = true;
      }
    }
    const bool dev_out = is_device_ptr(out);
    KStageResult* d_out = dev_out ? reinterpret_cast<KStageResult*>(out)
                                  : ctx->result.as<KStageResult>();
    const bool dev_probs = probs && is_device_ptr(probs);
    double* d_probs = nullptr;
    if (probs) {
      if (dev_probs) {
        d_probs = probs;
      } else {
        ctx->out_stage2.ensure(8 * n);
        d_probs = ctx->out_stage2.as<double>();
      }
    }
    cuda_check(launch_stage_reduce(d_scores, (long long)n, (int)stride, (int)col, d_rng, d_out,
                                   d_probs, ctx->stream, stage_scratch(ctx, (long long)n)),
               "stage_reduce launch");
    bool sync = host_in;
    if (!dev_out) {
      finish_copy_out(ctx, out, d_out, sizeof(KStageResult));
      sync = true;
    }
    if (rng_state && !dev_rng) finish_copy_out(ctx, rng_state, d_rng, 40);
    if (probs && !dev_probs) {
      finish_copy_out(ctx, probs, d_probs, 8 * n);
      sync = true;
    }
    if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "stage_reduce");
  });
}

b3d_status b3d_gpu_coarse_to_fine(b3d_gpu_context* ctx, int32_t mesh_id, const b3d_pose* center,
                                  const b3d_stage_spec* stages, uint32_t n_stages,
                                  uint64_t* rng_state, b3d_stage_result* results,
                                  b3d_pose* centers) {
  return guarded([&] {
    require_ready(ctx, true, true);
    check(center && stages && n_stages > 0 && results, "bad arguments");
    DeviceGuard dg(ctx->device);
    const Mesh& m = get_mesh(ctx, mesh_id);
    // stage sizes, rotation tables (staged once), scratch sized for the
    // largest stage / window
    std::vector<uint64_t> n(n_stages), rot_off(n_stages);
    uint64_t n_max = 0, rot_total = 0;
    int w_max = 0;
    bool any_sample = false;
    for (uint32_t s = 0; s < n_stages; ++s) {
      const b3d_stage_spec& g = stages[s];
      check(g.rotations && g.n_rot > 0, "stage: rotation table required");
      const uint64_t nt = (uint64_t)g.count[0] * g.count[1] * g.count[2];
      check(nt > 0, "pose grid: counts must be >= 1");
      check(g.mode == B3D_GRID_PRODUCT || nt == g.n_rot,
            "pose grid: zip mode needs nx*ny*nz == n_rot");
      n[s] = g.mode == B3D_GRID_PRODUCT ? nt * g.n_rot : nt;
      n_max = std::max(n_max, n[s]);
      w_max = std::max(w_max, (int)g.window);
      rot_off[s] = rot_total;
      rot_total += g.n_rot;
      any_sample = any_sample || g.select == B3D_SELECT_SAMPLE;
    }
    if (any_sample) check(rng_state != nullptr, "stage: SAMPLE selection needs rng_state");
    ctx->c2f_scores.ensure(8 * n_max);
    ctx->c2f_rot.ensure(32 * rot_total);
    ctx->c2f_centers.ensure(sizeof(KPose) * (n_stages + 1));
    ctx->c2f_results.ensure(sizeof(KStageResult) * n_stages);
    for (uint32_t s = 0; s < n_stages; ++s)
      cuda_check(cudaMemcpyAsync(ctx->c2f_rot.as<double>() + 4 * rot_off[s], stages[s].rotations,
                                 32ull * stages[s].n_rot, cudaMemcpyDefault, ctx->stream),
                 "cudaMemcpyAsync rotations");
    KPose* d_centers = ctx->c2f_centers.as<KPose>();
    const KPose c0 = pose_from_c(*center);
    cuda_check(cudaMemcpyAsync(d_centers, &c0, sizeof(KPose), cudaMemcpyHostToDevice,
                               ctx->stream),
               "cudaMemcpyAsync centre");
    unsigned long long* d_rng = nullptr;
    const bool dev_rng = rng_state && is_device_ptr(rng_state);
    if (rng_state) {
      if (dev_rng) {
        d_rng = reinterpret_cast<unsigned long long*>(rng_state);
      } else {
        cuda_check(cudaMemcpyAsync(ctx->rng.p, rng_state, 40, cudaMemcpyHostToDevice,
                                   ctx->stream),
                   "cudaMemcpyAsync rng");
        d_rng = ctx->rng.as<unsigned long long>();
      }
    }
    KStageResult* d_res = ctx->c2f_results.as<KStageResult>();
    double spread = 0;  // the chained centres stay within the summed extents
    for (uint32_t s = 0; s < n_stages; ++s) spread += std::sqrt(sq3(stages[s].extent));
    LaunchPlan lp = plan_launch<false, true, false>(ctx, m, (long long)n_max, w_max, false,
                                                    region_hint(ctx, m, c0, spread, w_max));
    for (uint32_t s = 0; s < n_stages; ++s) {
      const b3d_stage_spec& g = stages[s];
      // coarse_to_fine_propose scores through score_cells (inference.cpp:381):
      // the gated inference seam
      const LikSpec spec =
          make_spec(ctx->k, &g.noise, 1, ctx->sigma_max, g.window, ctx->prefactor, true);
      KParams p = base_params(ctx, m);
      p.poses = nullptr;
      p.grid.center_dev = d_centers + s;
      for (int a = 0; a < 3; ++a) {
        p.grid.extent[a] = g.extent[a];
        p.grid.count[a] = (int)g.count[a];
      }
      p.grid.rotations = ctx->c2f_rot.as<double>() + 4 * rot_off[s];
      p.grid.n_rot = (int)g.n_rot;
      p.grid.mode = (int)g.mode;
      p.n_hyp = (long long)n[s];
      p.scores = ctx->c2f_scores.as<double>();
      p.status = nullptr;
      if (spec.single()) {
        p.lik = spec.chunks[0].lik;
        attach_base(ctx, p);
        p.zscratch = ctx->zscratch.as<unsigned long long>();
        p.vscratch = ctx->vscratch.as<double>();
        p.vcap = lp.vcap;
        p.zcap = lp.zcap;
        p.zstride = lp.zstride;
        cuda_check(launch_render_score<false, true, false>(p, lp.cap, lp.smem, ctx->stream),
                   "render_score launch");
      } else {
        run_scores(ctx, m, p, spec, (long long)n[s], p.scores, nullptr, false, 0);
      }
      const bool sample = g.select == B3D_SELECT_SAMPLE;
      cuda_check(launch_stage_reduce(p.scores, (long long)n[s], 1, 0, sample ? d_rng : nullptr,
                                     d_res + s, nullptr, ctx->stream,
                                     stage_scratch(ctx, (long long)n[s])),
                 "stage_reduce launch");
      cuda_check(launch_select_center(p.grid, d_res + s, sample ? 1 : 0, d_centers + s + 1,
                                      ctx->stream),
                 "select_center launch");
    }
    bool sync = !dev_rng && rng_state != nullptr;
    cuda_check(cudaMemcpyAsync(results, d_res, sizeof(KStageResult) * n_stages, cudaMemcpyDefault,
                               ctx->stream),
               "cudaMemcpyAsync results");
    if (!is_device_ptr(results)) sync = true;
    if (centers) {
      cuda_check(cudaMemcpyAsync(centers, d_centers, sizeof(KPose) * (n_stages + 1),
                                 cudaMemcpyDefault, ctx->stream),
                 "cudaMemcpyAsync centres");
      if (!is_device_ptr(centers)) sync = true;
    }
    if (rng_state && !dev_rng)
      cuda_check(cudaMemcpyAsync(rng_state, d_rng, 40, cudaMemcpyDeviceToHost, ctx->stream),
                 "cudaMemcpyAsync rng");
    if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "coarse_to_fine");
  });
}

b3d_status b3d_gpu_set_base_scene(b3d_gpu_context* ctx, const int32_t* mesh_ids,
                                  const b3d_pose* model_to_world, uint32_t n) {
  return guarded([&] {
    if (ctx) ++ctx->gen;
    require_ready(ctx, false, false);
    DeviceGuard dg(ctx->device);
    ++ctx->base_version;
    ctx->base_terms_key.clear();
    if (n == 0) {
      ctx->has_base = false;
      ctx->base_draw = 0;
      ctx->base_valid = 0;
      return;
    }
    check(mesh_ids && model_to_world, "bad arguments");
    const size_t npx = (size_t)ctx->k.width * ctx->k.height;
    ctx->base_keys.ensure(8 * npx);
    ctx->base_tmp.ensure(8 * npx);
    ctx->has_base = false;
    ctx->base_draw = 0;
    unsigned long long* cur = nullptr;  // first instance composes onto the background
    for (uint32_t i = 0; i < n; ++i) {
      const Mesh& m = get_mesh(ctx, mesh_ids[i]);
      KParams p = base_params(ctx, m);
      const KPose pose = pose_from_c(model_to_world[i]);
      ctx->in_stage.ensure(sizeof(KPose));
      cuda_check(cudaMemcpyAsync(ctx->in_stage.p, &pose, sizeof(KPose), cudaMemcpyHostToDevice,
                                 ctx->stream),
                 "cudaMemcpyAsync pose");
      p.poses = ctx->in_stage.as<KPose>();
      p.n_hyp = 1;
      p.lik.n_noise = 0;
      p.draw_base = ctx->base_draw;
      p.base_keys = cur;
      // ping-pong: the last instance must land in base_keys
      unsigned long long* dst = ((n - 1 - i) % 2 == 0) ? ctx->base_keys.as<unsigned long long>()
                                                       : ctx->base_tmp.as<unsigned long long>();
      p.out_keys = dst;
      p.out_depth = nullptr;
      p.out_ids = nullptr;
      LaunchPlan lp = plan_launch<true, false, true>(ctx, m, 1);
      p.zscratch = ctx->zscratch.as<unsigned long long>();
      p.vscratch = ctx->vscratch.as<double>();
      p.vcap = lp.vcap;
      p.zcap = lp.zcap;
      p.zstride = lp.zstride;
      cuda_check(launch_render_score<true, false, true>(p, 1, lp.smem, ctx->stream),
                 "base render launch");
      cur = dst;
      ctx->base_draw += (uint32_t)m.nt;
    }
    std::vector<unsigned long long> keys(npx);
    cuda_check(cudaMemcpyAsync(keys.data(), ctx->base_keys.p, 8 * npx, cudaMemcpyDeviceToHost,
                               ctx->stream),
               "cudaMemcpyAsync base");
    cuda_check(cudaStreamSynchronize(ctx->stream), "set_base_scene");
    const float far_f = static_cast<float>(ctx->k.far_m);
    int valid = 0;
    for (unsigned long long k : keys) {
      const unsigned int bits = (unsigned int)(k >> 32);
      float z;
      std::memcpy(&z, &bits, 4);
      valid += z < far_f;
    }
    ctx->base_valid = valid;
    ctx->has_base = true;
  });
}

b3d_status b3d_gpu_score_contact_grid(b3d_gpu_context* ctx, int32_t mesh_id,
                                      const b3d_contact_grid* grid, double* scores,
                                      uint8_t* status) {
  return guarded([&] {
    check(grid != nullptr, "bad arguments");
    const b3d_contact_cells cells = stage0_parent(*grid);
    const uint64_t n = (uint64_t)grid->count[0] * grid->count[1] * grid->count[2];
    score_common(ctx, mesh_id, nullptr, nullptr, n, scores, status, &cells);
  });
}

b3d_status b3d_gpu_score_contact_cells(b3d_gpu_context* ctx, int32_t mesh_id,
                                       const b3d_contact_cells* cells, double* scores,
                                       uint8_t* status) {
  return guarded([&] {
    check(cells != nullptr, "bad arguments");
    const uint64_t n =
        (uint64_t)cells->grid.count[0] * cells->grid.count[1] * cells->grid.count[2];
    score_common(ctx, mesh_id, nullptr, nullptr, n, scores, status, cells);
  });
}

namespace {
void cells_poses(const b3d_contact_cells& cells, b3d_pose* out) {
  std::vector<double> spin;
  const KGrid g = make_contact_cells(cells, spin);
  const uint32_t nx = g.count[0], ny = g.count[1], nt = g.count[2];
  for (uint32_t ix = 0; ix < nx; ++ix)
    for (uint32_t iy = 0; iy < ny; ++iy)
      for (uint32_t it = 0; it < nt; ++it)
        out[((size_t)ix * ny + iy) * nt + it] = contact_cell_pose(g, spin, ix, iy, it);
}
}  // namespace

b3d_status b3d_contact_grid_poses(const b3d_contact_grid* grid, b3d_pose* out) {
  return guarded([&] {
    check(grid && out, "bad arguments");
    cells_poses(stage0_parent(*grid), out);
  });
}

b3d_status b3d_contact_cells_poses(const b3d_contact_cells* cells, b3d_pose* out) {
  return guarded([&] {
    check(cells && out, "bad arguments");
    cells_poses(*cells, out);
  });
}

b3d_status b3d_gpu_enumerate_poses(b3d_gpu_context* ctx, int32_t mesh_id,
                                   const b3d_pose* poses, uint64_t n, uint64_t* rng_state,
                                   b3d_stage_result* out, double* scores) {
  return guarded([&] {
    require_ready(ctx, true, true);
    check(poses && out && n > 0, "bad arguments");
    DeviceGuard dg(ctx->device);
    const Mesh& m = get_mesh(ctx, mesh_id);
    KParams p = base_params(ctx, m);
    bool host_in = false;
    p.poses = static_cast<const KPose*>(
        stage_in(ctx, ctx->in_stage, poses, sizeof(b3d_pose) * n, &host_in));
    p.n_hyp = (long long)n;
    const LikSpec& spec = ctx->spec;
    const int nn = spec.n_cols;
    // device layout: scores (n x n_noise), then the stage result (64 B) and
    // the Rng state (40 B), so one read-back returns everything
    const size_t sbytes = sizeof(double) * n * nn;
    ctx->c2f_scores.ensure(sbytes + 128);
    p.scores = ctx->c2f_scores.as<double>();
    p.status = nullptr;
    attach_base(ctx, p);
    LaunchPlan lp = plan_launch<false, true, false>(ctx, m, (long long)n);
    p.zscratch = ctx->zscratch.as<unsigned long long>();
    p.vscratch = ctx->vscratch.as<double>();
    p.vcap = lp.vcap;
    p.zcap = lp.zcap;
    p.zstride = lp.zstride;
    char* const tail = static_cast<char*>(ctx->c2f_scores.p) + sbytes;
    KStageResult* d_out = reinterpret_cast<KStageResult*>(tail);
    unsigned long long* d_rng = nullptr;
    const bool dev_rng = rng_state && is_device_ptr(rng_state);
    if (rng_state) {
      if (dev_rng) {
        d_rng = reinterpret_cast<unsigned long long*>(rng_state);
      } else {  // the render kernel stores the state as it starts (KParams::rng_dst)
        d_rng = reinterpret_cast<unsigned long long*>(tail + 64);
        p.rng_dst = d_rng;
        std::memcpy(p.rng_init, rng_state, 40);
      }
    }
    if (spec.single()) {
      cuda_check(launch_render_score<false, true, false>(p, lp.cap, lp.smem, ctx->stream),
                 "render_score launch");
    } else {
      if (p.rng_dst)
        cuda_check(cudaMemcpyAsync(p.rng_dst, rng_state, 40, cudaMemcpyHostToDevice, ctx->stream),
                   "cudaMemcpyAsync rng");
      p.rng_dst = nullptr;
      run_scores(ctx, m, p, spec, (long long)n, p.scores, nullptr, false, 0);
    }
    cuda_check(launch_stage_reduce(p.scores, (long long)n, nn, 0, d_rng, d_out, nullptr,
                                   ctx->stream, stage_scratch(ctx, (long long)n)),
               "stage_reduce launch");
    const bool host_out = !is_device_ptr(out);
    const bool host_rng = rng_state && !dev_rng;
    const bool host_scores = scores && !is_device_ptr(scores);
    if (!host_out)
      cuda_check(cudaMemcpyAsync(out, d_out, sizeof(KStageResult), cudaMemcpyDeviceToDevice,
                                 ctx->stream),
                 "cudaMemcpyAsync result");
    if (scores && !host_scores)
      cuda_check(cudaMemcpyAsync(scores, p.scores, sbytes, cudaMemcpyDeviceToDevice, ctx->stream),
                 "cudaMemcpyAsync scores");
    if (host_out || host_rng || host_scores) {
      // one read-back into pinned staging: [scores if wanted] + result + Rng
      const size_t from = host_scores ? 0 : sbytes;
      ctx->pin_scores.ensure(sbytes + 128);
      char* const pin = static_cast<char*>(ctx->pin_scores.p);
      cuda_check(cudaMemcpyAsync(pin + from, static_cast<char*>(ctx->c2f_scores.p) + from,
                                 sbytes + 128 - from, cudaMemcpyDeviceToHost, ctx->stream),
                 "cudaMemcpyAsync results");
      cuda_check(cudaStreamSynchronize(ctx->stream), "enumerate_poses");
      if (host_out) std::memcpy(out, pin + sbytes, sizeof(KStageResult));
      if (host_rng) std::memcpy(rng_state, pin + sbytes + 64, 40);
      if (host_scores) std::memcpy(scores, pin, sbytes);
    } else if (host_in) {
      cuda_check(cudaStreamSynchronize(ctx->stream), "enumerate_poses");
    }
  });
}

namespace {

// The graph-replayed form of b3d_gpu_enumerate_observed (all inputs
// page-locked host memory, one fused launch, no base scene, no peers):
// captured on the second call with the same buffers and context state,
// replayed afterwards -- one host launch instead of seven stream operations,
// and the score kernel launched with programmatic serialization right
// behind the observation cache (it waits for it before its window sums).
// Returns false when the form does not apply (the caller runs the plain path).
bool enumerate_observed_graph(b3d_gpu_context* ctx, int32_t mesh_id, const float* depth,
                              const b3d_pose* poses, uint64_t n, uint64_t* rng_state,
                              b3d_stage_result* out, double* scores) {
  static const bool enabled = [] {
    const char* e = std::getenv("B3D_E2E_GRAPH");  // 0 disables (A/B)
    return !e || std::atoi(e) != 0;
  }();
  if (!enabled || !ctx || !depth || !poses || !out || n == 0) return false;
  if (!ctx->has_camera || !ctx->has_lik || ctx->has_base || ctx->n_score_peers) return false;
  if (!ctx->spec.single()) return false;
  if (!is_pinned_host(depth) || !is_pinned_host(poses) || is_device_ptr(out)) return false;
  if (scores && !is_pinned_host(scores)) return false;
  if (rng_state && is_device_ptr(rng_state)) return false;
  if (mesh_id < 0 || mesh_id >= (int)ctx->meshes.size()) return false;
  const size_t npx = (size_t)ctx->k.width * ctx->k.height;
  const int nn = ctx->spec.n_cols;
  const size_t sbytes = sizeof(double) * n * nn;
  ctx->obs_depth.ensure(npx * 4);
  ctx->obs_pts.ensure(npx * sizeof(float4));
  ctx->in_stage.ensure(sizeof(b3d_pose) * n);
  ctx->c2f_scores.ensure(sbytes + 128);
  ctx->pin_scores.ensure(128);
  ctx->pin_rng.ensure(64);
  ctx->e2e_rng.ensure(64);
  const Mesh& m = get_mesh(ctx, mesh_id);
  std::vector<const void*> key{reinterpret_cast<const void*>(ctx->gen),
                               reinterpret_cast<const void*>((uintptr_t)mesh_id),
                               reinterpret_cast<const void*>((uintptr_t)n),
                               reinterpret_cast<const void*>((uintptr_t)(rng_state != nullptr)),
                               depth, poses, scores, ctx->stream, ctx->obs_depth.p,
                               ctx->obs_pts.p, ctx->obs_count.p, ctx->in_stage.p,
                               ctx->c2f_scores.p, ctx->pin_scores.p, ctx->pin_rng.p,
                               ctx->e2e_rng.p, ctx->zscratch.p, ctx->vscratch.p,
                               ctx->stage_part.p, m.verts.p};
  static const bool dbg = std::getenv("B3D_E2E_DEBUG") != nullptr;
  if (dbg && !(ctx->e2e.valid && ctx->e2e.key == key)) {
    std::fprintf(stderr, "b3d e2e graph: (re)capture needed, warm %d valid %d, differing key slots:",
                 ctx->e2e.warm, (int)ctx->e2e.valid);
    for (size_t i = 0; i < key.size() && i < ctx->e2e.key.size(); ++i)
      if (key[i] != ctx->e2e.key[i]) std::fprintf(stderr, " %zu", i);
    std::fprintf(stderr, "\n");
  }
  if (!(ctx->e2e.valid && ctx->e2e.key == key)) {
    // first sight of this configuration: run the plain path once (it sizes
    // every buffer and sets the kernels' attributes), capture on the next
    if (ctx->e2e.warm == 0 || ctx->e2e.key != key) {
      if (ctx->e2e.exec) cudaGraphExecDestroy(ctx->e2e.exec);
      ctx->e2e = b3d_gpu_context::E2E{};
      ctx->e2e.key = key;
      ctx->e2e.warm = 1;
      return false;
    }
    // zero-copy: the page-locked inputs are read by the kernels through
    // their device mappings (no upload copies), the stage result and the Rng
    // state live in mapped page-locked memory
    void *d_depth = nullptr, *d_poses = nullptr, *d_pin = nullptr, *d_pin_rng = nullptr,
         *d_scores_host = nullptr;
    if ((scores && cudaHostGetDevicePointer(&d_scores_host, scores, 0) != cudaSuccess) ||
        cudaHostGetDevicePointer(&d_depth, const_cast<float*>(depth), 0) != cudaSuccess ||
        cudaHostGetDevicePointer(&d_poses, const_cast<b3d_pose*>(poses), 0) != cudaSuccess ||
        cudaHostGetDevicePointer(&d_pin, ctx->pin_scores.p, 0) != cudaSuccess ||
        cudaHostGetDevicePointer(&d_pin_rng, ctx->pin_rng.p, 0) != cudaSuccess) {
      cudaGetLastError();
      ctx->e2e.warm = 2;
      return false;
    }
    KStageResult* d_out = static_cast<KStageResult*>(d_pin);
    unsigned long long* d_rng = static_cast<unsigned long long*>(d_pin_rng);
    KParams p = base_params(ctx, m);
    p.poses = static_cast<const KPose*>(d_poses);
    p.n_hyp = (long long)n;
    p.scores = ctx->c2f_scores.as<double>();
    p.scores_mirror = static_cast<double*>(d_scores_host);  // the caller's scores, zero-copy
    p.status = nullptr;
    attach_base(ctx, p);
    LaunchPlan lp = plan_launch<false, true, false>(ctx, m, (long long)n, -1, false,
                                                    region_hint_poses(ctx, m, poses, n,
                                                                      ctx->lik.window));
    p.zscratch = ctx->zscratch.as<unsigned long long>();
    p.vscratch = ctx->vscratch.as<double>();
    p.vcap = lp.vcap;
    p.zcap = lp.zcap;
    p.zstride = lp.zstride;
    void* const scratch = stage_scratch(ctx, (long long)n);
    // the key as captured (plan_launch / stage_scratch may have grown buffers)
    key[16] = ctx->zscratch.p;
    key[17] = ctx->vscratch.p;
    key[18] = ctx->stage_part.p;
    cudaGraph_t graph = nullptr;
    cuda_check(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal),
               "begin capture");
    cudaError_t e = launch_obs_prepare(static_cast<const float*>(d_depth), (int)ctx->k.width,
                                       (int)ctx->k.height, static_cast<float>(ctx->k.far_m),
                                       (float)ctx->k.cx, (float)ctx->k.cy,
                                       (float)(1.0 / ctx->k.fx), (float)(1.0 / ctx->k.fy),
                                       ctx->obs_pts.as<float4>(), ctx->obs_count.as<int>(),
                                       ctx->stream);
    if (e == cudaSuccess)
      e = launch_render_score<false, true, false>(p, lp.cap, lp.smem, ctx->stream, true);
    if (e == cudaSuccess)
      e = launch_stage_reduce(p.scores, (long long)n, nn, 0, rng_state ? d_rng : nullptr, d_out,
                              nullptr, ctx->stream, scratch);
    const cudaError_t e2 = cudaStreamEndCapture(ctx->stream, &graph);
    cudaGetLastError();
    static const bool dbg = std::getenv("B3D_E2E_DEBUG") != nullptr;
    if (dbg)
      std::fprintf(stderr, "b3d e2e graph capture: %s / %s\n", cudaGetErrorString(e),
                   cudaGetErrorString(e2));
    if (e != cudaSuccess || e2 != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      ctx->e2e.warm = 2;  // this configuration cannot be captured: plain path
      return false;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e3 = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e3 != cudaSuccess) {
      cudaGetLastError();
      ctx->e2e.warm = 2;
      return false;
    }
    ctx->e2e.exec = exec;
    ctx->e2e.valid = true;
    ctx->e2e.key = key;
  }
  if (rng_state) std::memcpy(ctx->pin_rng.p, rng_state, 40);
  cuda_check(cudaGraphLaunch(ctx->e2e.exec, ctx->stream), "cudaGraphLaunch");
  cuda_check(cudaStreamSynchronize(ctx->stream), "enumerate_observed");
  std::memcpy(out, ctx->pin_scores.p, sizeof(KStageResult));
  if (rng_state) std::memcpy(rng_state, ctx->pin_rng.p, 40);
  ctx->has_obs = true;
  ++ctx->obs_version;
  return true;
}

}  // namespace

b3d_status b3d_gpu_enumerate_observed(b3d_gpu_context* ctx, int32_t mesh_id, const float* depth,
                                      const b3d_pose* poses, uint64_t n, uint64_t* rng_state,
                                      b3d_stage_result* out, double* scores) {
  bool done = false;
  const b3d_status g = guarded([&] {
    if (ctx && ctx->e2e.warm != 2) {
      DeviceGuard dg(ctx->device);
      done = enumerate_observed_graph(ctx, mesh_id, depth, poses, n, rng_state, out, scores);
    }
  });
  if (g != B3D_OK) return g;
  if (done) return B3D_OK;
  const b3d_status st = b3d_gpu_set_observation(ctx, depth);
  if (st != B3D_OK) return st;
  return b3d_gpu_enumerate_poses(ctx, mesh_id, poses, n, rng_state, out, scores);
}

b3d_status b3d_gpu_enumerate_grid(b3d_gpu_context* ctx, int32_t mesh_id,
                                  const b3d_pose_grid* grid, uint64_t* rng_state,
                                  b3d_stage_result* out, double* scores) {
  return guarded([&] {
    require_ready(ctx, true, true);
    check(grid && out && scores, "bad arguments");
    check(is_device_ptr(scores) && is_device_ptr(out) && (!rng_state || is_device_ptr(rng_state)),
          "enumerate_grid: scores, out and rng_state must be device memory");
    DeviceGuard dg(ctx->device);
    const uint64_t nt = (uint64_t)grid->count[0] * grid->count[1] * grid->count[2];
    const uint64_t n = grid->mode == B3D_GRID_PRODUCT ? nt * grid->n_rot : nt;
    score_common(ctx, mesh_id, nullptr, grid, n, scores, nullptr, nullptr, 0, 0,
                 reinterpret_cast<unsigned long long*>(rng_state),
                 reinterpret_cast<KStageResult*>(out), true);
  });
}

b3d_status b3d_gpu_score_grid_range(b3d_gpu_context* ctx, int32_t mesh_id,
                                    const b3d_pose_grid* grid, uint64_t first, uint64_t n,
                                    double* scores, uint8_t* status) {
  return guarded([&] {
    check(grid != nullptr, "bad arguments");
    const uint64_t nt = (uint64_t)grid->count[0] * grid->count[1] * grid->count[2];
    const uint64_t gn = grid->mode == B3D_GRID_PRODUCT ? nt * grid->n_rot : nt;
    score_common(ctx, mesh_id, nullptr, grid, n, scores, status, nullptr, first, gn, nullptr,
                 nullptr, true);
  });
}

b3d_status b3d_gpu_sample_many(b3d_gpu_context* ctx, const double* scores, uint64_t n,
                               uint32_t stride, uint32_t col, uint64_t* rng_state,
                               uint32_t n_samples, uint64_t* samples, b3d_stage_result* out) {
  return guarded([&] {
    check(ctx && scores && rng_state && samples && out && n > 0 && n_samples > 0,
          "bad arguments");
    check(stride >= 1 && col < stride, "stage_reduce: bad stride/column");
    DeviceGuard dg(ctx->device);
    bool host_in = false;
    const double* d_scores = static_cast<const double*>(
        stage_in(ctx, ctx->in_stage, scores, sizeof(double) * n * stride, &host_in));
    const bool dev_rng = is_device_ptr(rng_state);
    unsigned long long* d_rng = reinterpret_cast<unsigned long long*>(rng_state);
    if (!dev_rng) {
      cuda_check(cudaMemcpyAsync(ctx->rng.p, rng_state, 40, cudaMemcpyHostToDevice, ctx->stream),
                 "cudaMemcpyAsync rng");
      d_rng = ctx->rng.as<unsigned long long>();
    }
    KStageResult* d_out = ctx->result.as<KStageResult>();
    ctx->out_stage.ensure(8ull * n_samples);
    ctx->out_stage2.ensure(8ull * n_samples);
    const bool dev_samples = is_device_ptr(samples);
    unsigned long long* d_samples = dev_samples ? reinterpret_cast<unsigned long long*>(samples)
                                                : ctx->out_stage2.as<unsigned long long>();
    // reduction without a draw, then the draws
    void* scr = stage_scratch(ctx, (long long)n);
    cuda_check(launch_stage_reduce(d_scores, (long long)n, (int)stride, (int)col, nullptr, d_out,
                                   nullptr, ctx->stream, scr),
               "stage_reduce launch");
    cuda_check(launch_sample_many(d_scores, (long long)n, (int)stride, (int)col, d_out, d_rng,
                                  (int)n_samples, ctx->out_stage.as<double>(), d_samples,
                                  ctx->stream, scr),
               "sample_many launch");
    cuda_check(cudaMemcpyAsync(&d_out->sample, d_samples, 8, cudaMemcpyDeviceToDevice,
                               ctx->stream),
               "cudaMemcpyAsync");
    cuda_check(cudaMemcpyAsync(out, d_out, sizeof(KStageResult), cudaMemcpyDefault, ctx->stream),
               "cudaMemcpyAsync result");
    if (!dev_samples)
      cuda_check(cudaMemcpyAsync(samples, d_samples, 8ull * n_samples, cudaMemcpyDeviceToHost,
                                 ctx->stream),
                 "cudaMemcpyAsync samples");
    if (!dev_rng)
      cuda_check(cudaMemcpyAsync(rng_state, d_rng, 40, cudaMemcpyDeviceToHost, ctx->stream),
                 "cudaMemcpyAsync rng");
    if (host_in || !dev_samples || !dev_rng || !is_device_ptr(out))
      cuda_check(cudaStreamSynchronize(ctx->stream), "sample_many");
  });
}

// rng.hpp:8-13, rng.cpp:13-28
static uint64_t splitmix64_next(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void b3d_rng_seed(uint64_t seed, uint64_t state[5]) {
  uint64_t s = seed;
  state[0] = seed;
  for (int i = 0; i < 4; ++i) state[1 + i] = splitmix64_next(s);
}

void b3d_rng_split(const uint64_t state[5], uint64_t k0, uint64_t k1, uint64_t k2,
                   uint64_t out[5]) {
  auto mix = [](uint64_t a, uint64_t b) {
    uint64_t s = a ^ (0x9e3779b97f4a7c15ull + (b << 6) + (b >> 2));
    return splitmix64_next(s);
  };
  b3d_rng_seed(mix(mix(mix(state[0], k0), k1), k2), out);
}

b3d_status b3d_voxel_to_mesh(const int32_t* voxels, uint64_t n, double resolution,
                             const double origin[3], double* vertices, uint32_t* triangles,
                             uint64_t* n_vertices, uint64_t* n_triangles) {
  return guarded([&] {
    check(voxels && origin && vertices && triangles && n_vertices && n_triangles,
          "bad arguments");
    require(n > 0, ErrorCode::invalid, "voxel_to_mesh: empty grid");
    // geometry.cpp:128-138
    static const int kCorners[6][4][3] = {
        {{0, 0, 0}, {0, 0, 1}, {0, 1, 1}, {0, 1, 0}},
        {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}, {1, 0, 1}},
        {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}, {0, 0, 1}},
        {{0, 1, 0}, {0, 1, 1}, {1, 1, 1}, {1, 1, 0}},
        {{0, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 0, 0}},
        {{0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}},
    };
    static const int kOff[6][3] = {{-1, 0, 0}, {1, 0, 0},  {0, -1, 0},
                                   {0, 1, 0},  {0, 0, -1}, {0, 0, 1}};
    struct K3 {
      int x, y, z;
      bool operator==(const K3& o) const { return x == o.x && y == o.y && z == o.z; }
    };
    struct H3 {
      size_t operator()(const K3& k) const {
        uint64_t h = 1469598103934665603ull;
        for (int v : {k.x, k.y, k.z}) {
          h ^= (uint64_t)(uint32_t)v;
          h *= 1099511628211ull;
        }
        return (size_t)h;
      }
    };
    std::unordered_map<K3, uint8_t, H3> occ;
    occ.reserve(2 * n);
    for (uint64_t i = 0; i < n; ++i)
      occ.emplace(K3{voxels[3 * i], voxels[3 * i + 1], voxels[3 * i + 2]}, 1);
    std::unordered_map<K3, uint32_t, H3> corner;
    uint64_t nv = 0, nt = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const int* v = voxels + 3 * i;
      for (int f = 0; f < 6; ++f) {
        if (occ.count(K3{v[0] + kOff[f][0], v[1] + kOff[f][1], v[2] + kOff[f][2]})) continue;
        uint32_t quad[4];
        for (int c = 0; c < 4; ++c) {
          const K3 cc{v[0] + kCorners[f][c][0], v[1] + kCorners[f][c][1],
                      v[2] + kCorners[f][c][2]};
          auto it = corner.find(cc);
          if (it == corner.end()) {
            it = corner.emplace(cc, (uint32_t)nv).first;
            vertices[3 * nv + 0] = origin[0] + resolution * (double)cc.x;
            vertices[3 * nv + 1] = origin[1] + resolution * (double)cc.y;
            vertices[3 * nv + 2] = origin[2] + resolution * (double)cc.z;
            ++nv;
          }
          quad[c] = it->second;
        }
        uint32_t* t = triangles + 3 * nt;
        t[0] = quad[0];
        t[1] = quad[1];
        t[2] = quad[2];
        t[3] = quad[0];
        t[4] = quad[2];
        t[5] = quad[3];
        nt += 2;
      }
    }
    *n_vertices = nv;
    *n_triangles = nt;
  });
}

b3d_status b3d_gpu_voxel_to_mesh(b3d_gpu_context* ctx, const int32_t* voxels, uint64_t n,
                                 double resolution, const double origin[3], double* vertices,
                                 uint32_t* triangles, uint64_t* n_vertices,
                                 uint64_t* n_triangles) {
  return guarded([&] {
    check(ctx && voxels && origin && vertices && triangles && n_vertices && n_triangles,
          "bad arguments");
    require(n > 0, ErrorCode::invalid, "voxel_to_mesh: empty grid");
    check(n < (1ull << 26), "voxel_to_mesh: too many voxels");
    DeviceGuard dg(ctx->device);
    bool host_in = false;
    DevBuf vin, vout, tout;
    const int* d_vox = static_cast<const int*>(stage_in(ctx, vin, voxels, 12 * n, &host_in));
    const bool host_v = !is_device_ptr(vertices), host_t = !is_device_ptr(triangles);
    if (host_v) vout.ensure(24 * 8 * n);
    if (host_t) tout.ensure(12 * 12 * n);
    double* dv = host_v ? vout.as<double>() : vertices;
    unsigned* dt = host_t ? tout.as<unsigned>() : reinterpret_cast<unsigned*>(triangles);
    unsigned long long nv = 0, nt = 0;
    const cudaError_t e =
        voxel_to_mesh_device(d_vox, n, resolution, origin, dv, dt, &nv, &nt, ctx->stream);
    check(e != cudaErrorInvalidValue, "voxel_to_mesh: coordinates outside [-2^20+1, 2^20-2]");
    cuda_check(e, "voxel_to_mesh_device");
    if (host_v)
      cuda_check(cudaMemcpyAsync(vertices, dv, 24 * nv, cudaMemcpyDeviceToHost, ctx->stream),
                 "cudaMemcpyAsync vertices");
    if (host_t)
      cuda_check(cudaMemcpyAsync(triangles, dt, 12 * nt, cudaMemcpyDeviceToHost, ctx->stream),
                 "cudaMemcpyAsync triangles");
    cuda_check(cudaStreamSynchronize(ctx->stream), "voxel_to_mesh");
    *n_vertices = nv;
    *n_triangles = nt;
  });
}

// ---- synthetic observations (likelihood.cpp:44-80, tracking.cpp:174-206)
//
// sample_observation consumes ONE Rng stream with a data-dependent number of
// draws per point (outlier test, rejection-sampled index, Box-Muller loops),
// so it cannot be split across threads without changing the stream; it runs
// on the host with the reference's libm calls (cbrt, log, cos, sqrt, lround),
// which makes it bitwise the reference's.  Frames of a sequence use
// independent split streams and run one thread per frame.
namespace {

struct HostRng {
  uint64_t s[5];
  uint64_t next() {  // rng.cpp:30-40 (xoshiro256**)
    uint64_t* q = s + 1;
    auto rotl = [](uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
    const uint64_t r = rotl(q[1] * 5, 7) * 9;
    const uint64_t t = q[1] << 17;
    q[2] ^= q[0];
    q[3] ^= q[1];
    q[1] ^= q[2];
    q[0] ^= q[3];
    q[2] ^= t;
    q[3] = rotl(q[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t uniform_int(uint64_t n) {  // rng.cpp:48-57
    const uint64_t limit = n * (UINT64_MAX / n);
    uint64_t x;
    do {
      x = next();
    } while (x >= limit);
    return x % n;
  }
  double normal() {  // rng.cpp:59-64
    double u1 = uniform();
    double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925287 * u2);
  }
};

void check_noise(const b3d_intrinsics& k, const b3d_noise& np) {
  // validate_noise(np, k.far) (likelihood.cpp:21-27)
  check(k.far_m > 0, "sigma_max must be positive");
  check(np.sigma_noise > 0, "sigma_noise must be positive");
  check(np.p_outlier >= 0 && np.p_outlier <= 1, "p_outlier must be in [0,1]");
}

void sample_one(const b3d_intrinsics& k, const float* rendered, const b3d_noise& np,
                HostRng& rng, float* out) {
  // depth_to_cloud (geometry.cpp:54-70)
  const float sentinel = static_cast<float>(k.far_m);
  std::vector<double> cloud;
  cloud.reserve(3 * (size_t)k.width * k.height);
  for (uint32_t v = 0; v < k.height; ++v)
    for (uint32_t u = 0; u < k.width; ++u) {
      const float z = rendered[(size_t)v * k.width + u];
      if (z >= sentinel) continue;
      const double zd = z;
      cloud.push_back((u - k.cx) * zd / k.fx);
      cloud.push_back((v - k.cy) * zd / k.fy);
      cloud.push_back(zd);
    }
  const size_t n = cloud.size() / 3;
  check(n > 0, "sample_observation: all-sentinel render");
  const double near3 = k.near_m * k.near_m * k.near_m;
  const double far3 = k.far_m * k.far_m * k.far_m;
  std::fill(out, out + (size_t)k.width * k.height, sentinel);
  for (size_t i = 0; i < n; ++i) {
    double x, y, z;
    if (rng.uniform() < np.p_outlier) {
      // uniform in the viewing frustum: depth density ~ z^2
      z = std::cbrt(near3 + rng.uniform() * (far3 - near3));
      x = rng.uniform((0.0 - k.cx) * z / k.fx, (k.width - k.cx) * z / k.fx);
      y = rng.uniform((0.0 - k.cy) * z / k.fy, (k.height - k.cy) * z / k.fy);
    } else {
      const size_t j = (size_t)rng.uniform_int(n);
      x = cloud[3 * j];
      y = cloud[3 * j + 1];
      z = cloud[3 * j + 2];
      x += 0.0 + np.sigma_noise * rng.normal();
      y += 0.0 + np.sigma_noise * rng.normal();
      z += 0.0 + np.sigma_noise * rng.normal();
    }
    if (z < k.near_m || z >= k.far_m) continue;
    const long u = std::lround(k.fx * x / z + k.cx);
    const long v = std::lround(k.fy * y / z + k.cy);
    if (u < 0 || u >= static_cast<long>(k.width) || v < 0 || v >= static_cast<long>(k.height))
      continue;
    float& cell = out[(size_t)v * k.width + (size_t)u];
    cell = std::min(cell, static_cast<float>(z));
  }
}

}  // namespace

b3d_status b3d_sample_observation(const b3d_intrinsics* k, const float* rendered,
                                  const b3d_noise* noise, uint64_t rng_state[5], float* out) {
  return guarded([&] {
    check(k && rendered && noise && rng_state && out, "bad arguments");
    check(k->width > 0 && k->height > 0, "bad intrinsics");
    check_noise(*k, *noise);
    HostRng rng;
    std::memcpy(rng.s, rng_state, sizeof(rng.s));
    sample_one(*k, rendered, *noise, rng, out);
    std::memcpy(rng_state, rng.s, sizeof(rng.s));
  });
}

b3d_status b3d_sample_observations(const b3d_intrinsics* k, const float* rendered, uint64_t n,
                                   const b3d_noise* noise, const uint64_t rng_state[5],
                                   uint64_t split_key, float* out) {
  return guarded([&] {
    check(k && rendered && noise && rng_state && out, "bad arguments");
    check(k->width > 0 && k->height > 0, "bad intrinsics");
    check_noise(*k, *noise);
    const size_t npx = (size_t)k->width * k->height;
    std::vector<uint8_t> empty(n, 0);
    const float sentinel = static_cast<float>(k->far_m);
    for (uint64_t i = 0; i < n; ++i) {
      const float* r = rendered + i * npx;
      empty[i] = std::none_of(r, r + npx, [&](float z) { return z < sentinel; });
    }
    check(std::find(empty.begin(), empty.end(), 1) == empty.end(),
          "sample_observation: all-sentinel render");
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nth = (unsigned)std::min<uint64_t>(n, hw);
    std::vector<std::thread> pool;
    std::atomic<uint64_t> next{0};
    for (unsigned t = 0; t < nth; ++t)
      pool.emplace_back([&] {
        for (uint64_t i; (i = next.fetch_add(1)) < n;) {
          // Rng frame_rng = rng.split(split_key, i) (tracking.cpp:200)
          HostRng rng;
          b3d_rng_split(rng_state, split_key, i, 0, rng.s);
          sample_one(*k, rendered + i * npx, *noise, rng, out + i * npx);
        }
      });
    for (auto& th : pool) th.join();
  });
}

}  // extern "C"
