/*
 * b3d_oracle.h -- CPU ORACLE for the pose-enumeration hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * (Bayes3D C++ reference, /root/reference/proj) arithmetic for the hot path:
 * pose math, voxel mesh construction, the software z-buffer rasterizer, the
 * windowed mixture likelihood and the score/normalize/sample/argmax stage.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it -- and only as the checker, never as the thing measured or shipped.
 * The product path (libb3d_b200.so) never links or calls this library.
 *
 * Pinning: the restatement is checked against the reference's own known-answer
 * tests and test oracles (tests/test_oracle_*.py restate test_renderer.cpp,
 * test_likelihood.cpp, test_geometry.cpp, test_scene_graph.cpp with the same
 * parameters and tolerances) and, for the RNG, bit-for-bit against the
 * reference's own rng.cpp compiled from /root/reference (oracle/_ref, golden
 * vectors in tests/golden/).  Eigen (un-vendored, unpinned version) is absent,
 * so Eigen's expression evaluation order is restated explicitly below; it is
 * unpinned at the ulp level.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, mirroring the
 * reference's RelWithDebInfo no-FMA x86-64 build, proj/CMakeLists.txt:8-10).
 *
 * Extensions beyond the reference: per-pixel draw index
 * (=> instance id + triangle id) with the reference's strict-less tie rule,
 * and op counters for the roofline.
 */
#ifndef B3D_ORACLE_H
#define B3D_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as b3d_intrinsics (proj/include/b3d/b3d.h:45-49). */
typedef struct orc_intrinsics {
  double fx, fy, cx, cy;
  uint32_t width, height;
  double near_m, far_m;
} orc_intrinsics;

/* Same layout as b3d_pose (b3d.h:52-55): unit quaternion (w,x,y,z) + t. */
typedef struct orc_pose {
  double qw, qx, qy, qz;
  double tx, ty, tz;
} orc_pose;

typedef struct orc_noise {
  double p_outlier;
  double sigma_noise;
} orc_noise;

/* A mesh placed in the world (renderer.hpp:11-14). */
typedef struct orc_instance {
  const double* vertices;    /* n_vertices x 3, model frame */
  const uint32_t* triangles; /* n_triangles x 3 */
  uint64_t n_vertices, n_triangles;
  orc_pose model_to_world;
} orc_instance;

/* Algorithmic op counters. */
typedef struct orc_counters {
  uint64_t vertices;     /* N_v  vertices transformed            */
  uint64_t triangles;    /* T    screen triangles after clipping  */
  uint64_t bbox_px;      /* C_px bbox pixels tested               */
  uint64_t fragments;    /* F    pixels passing coverage          */
  uint64_t rend_valid;   /* R    rendered valid pixels            */
  uint64_t obs_valid;    /* M    observed valid pixels            */
  uint64_t pairs;        /* P    valid window pairs               */
} orc_counters;

/* ---- RNG: xoshiro256** seeded by splitmix64 (rng.hpp:8-42, rng.cpp) ----
 * state[0] = seed, state[1..4] = s[0..3]. */
void orc_rng_seed(uint64_t seed, uint64_t state[5]);
void orc_rng_split(const uint64_t state[5], uint64_t k0, uint64_t k1, uint64_t k2,
                   uint64_t out[5]);
uint64_t orc_rng_next_u64(uint64_t state[5]);
double orc_rng_uniform(uint64_t state[5]);
uint64_t orc_rng_uniform_int(uint64_t state[5], uint64_t n);
double orc_rng_normal(uint64_t state[5]);

/* ---- pose math (geometry.cpp:11-31, Eigen formulas restated) ---- */
void orc_compose(const orc_pose* a, const orc_pose* b, orc_pose* out);
void orc_inverse(const orc_pose* p, orc_pose* out);
void orc_rotation_matrix(const orc_pose* p, double r[9]); /* row-major */
void orc_quat_rotate(const orc_pose* p, const double v[3], double out[3]);
void orc_from_axis_angle(const double axis[3], double angle, orc_pose* out);
void orc_camera_pose_from_spherical(double distance, double azimuth, double altitude,
                                    orc_pose* out);
/* contact_to_pose (scene_graph.cpp:97-121); table extents (w,h), object
 * model-frame AABB.  Returns 0 on success, 1 if params are out of range. */
int orc_contact_to_pose(double table_w, double table_h, const double aabb_min[3],
                        const double aabb_max[3], int face, double dx, double dy,
                        double dtheta, orc_pose* out);
void orc_rotated_bounds(const double aabb_min[3], const double aabb_max[3], int face,
                        double lo[3], double hi[3]);

/* ---- meshes (geometry.cpp:142-177, scene_graph.cpp:37-58) ----
 * voxels: n x 3 int32 in stored order (must be sorted+unique for the
 * reference invariant).  vertices cap >= 8n*3, triangles cap >= 12n*3. */
int orc_voxel_to_mesh(const int32_t* voxels, size_t n, double resolution,
                      const double origin[3], double* vertices, uint32_t* triangles,
                      size_t* n_vertices, size_t* n_triangles);
void orc_box_mesh(const double lo[3], const double hi[3], double vertices[24],
                  uint32_t triangles[36]);

/* ---- renderer (renderer.cpp:61-189) ----
 * depth: W*H floats (initialised by the caller, e.g. to (float)far);
 * draw_index: W*H int32 or NULL (initialised to -1 by the caller);
 * draw_base: draw index of this mesh's triangle 0. */
void orc_raster_mesh(float* depth, int32_t* draw_index, const orc_intrinsics* k,
                     const double* vertices, uint64_t n_vertices,
                     const uint32_t* triangles, uint64_t n_triangles,
                     const orc_pose* model_to_camera, uint32_t draw_base,
                     orc_counters* counters);
/* render_instances (renderer.cpp:164-174): fills depth with (float)far and
 * draw_index with -1, then rasterizes each instance in order with
 * model_to_camera = compose(inverse(camera), model_to_world). */
void orc_render_instances(const orc_intrinsics* k, const orc_pose* camera,
                          const orc_instance* instances, size_t n_instances,
                          float* depth, int32_t* draw_index, orc_counters* counters);

/* ---- likelihood (likelihood.cpp:14-35,106-233) ---- */
double orc_visible_volume(const orc_intrinsics* k);
int orc_default_window(uint32_t width);
/* windowed_log_likelihood_multi.  prefactor: 0 = printed, 1 = uniform.
 * Returns 0 ok, 1 invalid argument (incl. empty render, which the reference
 * throws for at likelihood.cpp:159-160). */
int orc_windowed_loglik_multi(const float* observed, const float* rendered,
                              const orc_intrinsics* k, const orc_noise* noise,
                              size_t n_noise, double volume, double sigma_max,
                              int window, int prefactor, double* out,
                              orc_counters* counters);
/* depth_to_cloud (geometry.cpp:54-70): non-sentinel pixels row-major,
 * ((u-cx)z/fx, (v-cy)z/fy, z).  out: capacity W*H*3 doubles. */
void orc_depth_to_cloud(const float* depth, const orc_intrinsics* k, double* out, size_t* n);
/* sample_observation (likelihood.cpp:44-80) with the reference's Rng stream;
 * out: W*H fp32 depths.  Returns 1 on invalid noise / all-sentinel render. */
int orc_sample_observation(const float* rendered, const orc_intrinsics* k, double p_outlier,
                           double sigma, uint64_t st[5], float* out);
/* full_log_likelihood over explicit point clouds (likelihood.cpp:82-104).
 * Returns 1 for an empty rendered cloud / invalid noise. */
int orc_full_loglik_points(const double* obs, size_t n_obs, const double* rend,
                           size_t n_rend, const orc_noise* noise, double volume,
                           double sigma_max, int prefactor, double* out);
/* full_log_likelihood over the two depth images' clouds (likelihood.cpp:82-104). */
int orc_full_loglik(const float* observed, const float* rendered,
                    const orc_intrinsics* k, const orc_noise* noise, double volume,
                    double sigma_max, int prefactor, double* out);

/* ---- batched score (score_cells inner loop, inference.cpp:102-109,290-313) ----
 * For each hypothesis i: copy the base render (base_depth/base_index, may be
 * NULL => empty scene), rasterize the object mesh at
 * compose(inverse(camera), poses[i]) with draw_base, score against observed.
 * scores: n x n_noise.  status[i] = 0 ok / 1 empty render (score -inf).
 * threads: parallel_for semantics (parallel.hpp:19-54), 0 = hardware. */
int orc_score_poses(const orc_intrinsics* k, const orc_pose* camera,
                    const float* observed, const float* base_depth,
                    const double* vertices, uint64_t n_vertices,
                    const uint32_t* triangles, uint64_t n_triangles,
                    const orc_pose* poses, size_t n, const orc_noise* noise,
                    size_t n_noise, double sigma_max, int window, int prefactor,
                    double* scores, uint8_t* status, int threads,
                    orc_counters* counters);

/* ---- stage reductions (inference.cpp:16-23,315-353; tracking.cpp:132-134) ---- */
double orc_logsumexp(const double* xs, size_t n);
/* score_cells normalisation: returns all_zero flag. */
int orc_normalize(const double* log_targets, size_t n, double* probs);
size_t orc_sample_categorical(const double* probs, size_t n, uint64_t state[5]);
size_t orc_argmax(const double* xs, size_t n);

/* ---- pose grid (BASELINE 6-DoF grid; no reference -- see DESIGN.md) ----
 * lattice (tracking.cpp:27-37) per axis around center.t, rotation
 * q = normalized(center.q * dq[r]) (Eigen quaternion product). mode 0:
 * product, index = ((ix*ny+iy)*nz+iz)*n_rot + r; mode 1: zip, index i uses
 * translation i and rotation i (n = nx*ny*nz = n_rot). */
typedef struct orc_pose_grid {
  orc_pose center;
  double extent[3];
  uint32_t count[3];
  const double* rotations; /* n_rot x 4 (w,x,y,z) */
  uint32_t n_rot;
  uint32_t mode;
} orc_pose_grid;
uint64_t orc_grid_size(const orc_pose_grid* g);
void orc_grid_pose(const orc_pose_grid* g, uint64_t index, orc_pose* out);
double orc_lattice(double center, double extent, int n, int i);

#ifdef __cplusplus
}
#endif
#endif
