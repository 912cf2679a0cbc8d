// b3d_kernels.cuh -- device-side data structures shared by the B200 kernels
// and the C++ host layer.  No torch types: the host side is plain CUDA C++.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b3d200 {

// Same layout as b3d_pose (reference b3d.h:52-55).
struct KPose {
  double qw, qx, qy, qz;
  double tx, ty, tz;
};

// BASELINE 6-DoF hypothesis grid (no reference equivalent):
// translation lattice (tracking.cpp:27-37 formula) around the centre times a
// table of rotation perturbations, q = normalized(center.q * dq[r]).
// Table-contact hypotheses (stage0_cells / contact_to_pose,
// inference.cpp:208-238, scene_graph.cpp:97-121): the cell centres of an
// n_dx x n_dy x n_dtheta partition of one (object, face) support.  Values that
// need libm (face rotation, per-cell spin cos/sin, rotated bounds) are
// computed once on the host with the same formulas as the oracle.
struct KContact {
  double face_q[4];        // face_rotation(face), (w,x,y,z)
  double lo[3];            // rotated_bounds lo
  double w, h;             // footprint (hi - lo) in x, y
  double table_w, table_h;
  // parent cell (subdivide_cell, inference.cpp:240-259): child ix spans
  // [dx_lo + dx_w*ix/n, dx_lo + dx_w*(ix+1)/n); stage 0 is the parent
  // [0, table_w - w] (stage0_cells, inference.cpp:208-238)
  double dx_lo, dx_w, dy_lo, dy_w;
  const double* spin;      // n_dtheta x 2: cos, sin of half the cell-centre angle
};

struct KGrid {
  KPose center;             // used when center_dev == nullptr
  const KPose* center_dev;  // device-resident centre (stage chaining)
  double extent[3];
  int count[3];             // contact mode: n_dx, n_dy, n_dtheta
  const double* rotations;  // n_rot x 4 (w,x,y,z), device
  int n_rot;
  int mode;                 // 0 product, 1 zip, 2 table contact
  KContact contact;
};

constexpr int kMaxNoise = 12;  // noise entries per call (the default noise grid has 9)
constexpr int kMaxSlots = 4;   // distinct sigmas per call
constexpr int kMaxInst = 16;
constexpr int kCheb = 64;

struct KLik {
  int n_noise;
  int n_slots;
  int window;
  int slot_of[kMaxNoise];
  float slot_scale[kMaxSlots];   // log2(e)/(2 sigma^2) per distinct sigma (exp2 form)
  float slot_root[kMaxSlots];    // sqrt(slot_scale): single-sigma taps scale the points
  double one_minus_p[kMaxNoise]; // 1 - p_outlier
  double norm3[kMaxNoise];       // pow(2 pi sigma^2, -1.5)
  double floor_term[kMaxNoise];  // p_outlier / V
  double log_floor[kMaxNoise];   // log(floor_term)
  double prefactor[kMaxNoise];   // log(sigma/sigma_max) or -log(sigma_max)
};

struct KParams {
  // intrinsics (geometry.hpp:40-47)
  double fx, fy, cx, cy, near_m, far_m, near_lim;
  float far_f;
  int W, H;
  float fcx, fcy, inv_fx, inv_fy;  // fp32 back-projection for the likelihood
  KPose w2c;                       // inverse(camera)
  // mesh of the enumerated object
  const double* verts;
  const uint4* tris;  // (i0, i1, i2, 0) per triangle
  int nv, nt;
  uint32_t draw_base;
  // back-face culling of a closed mesh in score mode:
  // +1 = skip triangles with screen area2 > 0 (outward-wound mesh), -1 =
  // area2 < 0 (inward-wound), 0 = off; ignored for hypotheses with a vertex
  // in front of z = near
  int cull;
  // score-mode triangle order (depth = min over fragments does not depend
  // on draw order): 6 axis-aligned classes (+x,-x,+y,-y,+z,-z outward
  // normal), each sorted by plane offset o = n . a, then the rest (class 6).
  // A face of class c is turned away from the camera centre C (model frame)
  // iff o > n . C, so the back faces of a class are a suffix found per
  // hypothesis from the class's distinct plane offsets.
  const uint4* tris_s;
  int cls_start[8];         // class c = tris_s[cls_start[c], cls_start[c+1])
  const double* plane_off;  // distinct offsets per class, ascending
  const int* plane_end;     // tris_s index one past each plane's triangles
  int plane_begin[8];       // class c's planes = [plane_begin[c], plane_begin[c+1])
  // camera mode (render_instances under per-hypothesis cameras,
  // renderer.cpp:153-189 / tracking.cpp:100-108): hypothesis h is the
  // camera-to-world pose cams[h]; the mesh is the concatenation of n_inst
  // instances in draw order, instance i = vertices [inst_v0[i], inst_v0[i+1])
  // with model-to-world pose inst_pose[i]
  const KPose* cams;
  int n_inst;
  int inst_v0[kMaxInst + 1];
  KPose inst_pose[kMaxInst];
  // hypotheses
  const KPose* poses;  // nullptr => grid
  KGrid grid;
  long long n_hyp;
  long long index0;    // grid index of hypothesis 0 (shards of a large grid)
  // observation (per pixel: x, y, z, valid) + device count of valid pixels
  const float4* obs;
  const int* obs_count;
  KLik lik;
  // outputs
  double* scores;     // n_hyp x n_noise
  double* scores_mirror;  // optional second copy (mapped page-locked host memory)
  // fused score all-gather over NVLink: every score is also stored into
  // score_peers[r][(score_peer_offset + h) * n_noise + e] for each rank r
  // (peer-mapped symmetric buffers), so no separate collective is needed
  double* score_peers[8];
  int n_score_peers;
  long long score_peer_offset;
  long long score_peer_cap;  // elements per peer array; stores at or beyond are skipped
  uint8_t* status;    // n_hyp (1 = empty render)
  float* out_depth;   // n_hyp x W x H  (render mode)
  int32_t* out_ids;   // n_hyp x W x H  (render mode, draw index or -1)
  unsigned long long* out_keys;  // n_hyp x W x H raw (depth bits, draw) keys (base build)
  // fixed scene rendered once (compose_render, inference.cpp:102-109)
  const unsigned long long* base_keys;  // W x H keys, background depth 1e30; null = none
  int base_valid;                       // valid pixels of the base image
  const float* sbase;                   // n_slots x W x H window sums of the base image
  const double* cheb;                   // n_noise x kCheb coefficients of G(log |y|)
  double cheb_lo, cheb_hi;              // G's domain: [0, log(W*H)]
  // per-CTA global scratch (used only when the on-chip buffers overflow)
  unsigned long long* zscratch;  // gridDim x zstride keys
  long long zstride;             // (W + 4w) * (H + 4w): padded full-image region
  double* vscratch;              // gridDim x 3*nv
  int vcap;                      // vertices cached in shared memory
  int zcap;                      // z-buffer pixels in shared memory
  // optional: CTA 0 stores rng_init at rng_dst when the kernel starts (the
  // stage reduction launched after it then draws from that state, without
  // a separate host-to-device copy of 40 bytes)
  unsigned long long* rng_dst;
  unsigned long long rng_init[5];
  int obs_stage;  // stage the observation region into shared memory (bulk copy)
  int q1_small;  // tile-class bound for big projected faces (render_score.cuh hc.q1)
  int q1_ratio;  // region px per 100 triangles above which faces count as big
};

struct KStageResult {
  unsigned long long argmax;
  unsigned long long sample;
  double max_score;
  double logsumexp;
  double total;        // sum exp(x - max)
  double sample_logp;  // x[sample] - logsumexp
  unsigned int all_zero;
  unsigned int n_nonfinite;
  unsigned int sample_fallback;  // sequential CDF rescan was needed
  unsigned int pad;
};

// signal-pad barrier of a sharded stage (exchange.cu)
struct KBarrier {
  unsigned long long* sig[8];  // rank r's signal pad, mapped on this device
  int n_ranks, rank;
  unsigned long long epoch;
};

// fp64 image likelihood (exact_score.cu): one chunk of <= kMaxNoise noise
// entries with <= kMaxSlots distinct sigmas, window < 0 = full likelihood
struct KExactLik {
  int n_noise, n_slots, window;
  int slot_of[kMaxNoise];
  double inv2s2[kMaxSlots];  // 1 / (2 sigma^2) in the form's own rounding order
  double one_minus_p[kMaxNoise], norm3[kMaxNoise], floor_term[kMaxNoise], prefactor[kMaxNoise];
};

struct KExactArgs {
  const float4* obs;  // W x H observation cache (x, y, z, valid); z is the raw depth
  const float* rend;  // n x W x H rendered depth (sentinel = (float)far)
  int W, H;
  double fx, fy, cx, cy;
  float far_f;
  long long n;
  double* scores;  // scores[h * ld + col0 + e]
  int ld, col0;
  uint8_t* status;  // 1 = empty render (may be null)
  double* pts;      // full form: per-CTA rendered cloud, 3 x W x H doubles per CTA
  KExactLik lik;
};

}  // namespace b3d200
