/*
 * b3d_b200.h -- C ABI of the B200-native pose-enumeration hot path.
 *
 * Drop-in boundary for the reference's C API (proj/include/b3d/b3d.h): same
 * conventions -- opaque handles created by *_create and released by the
 * matching *_destroy (b3d.h:4-7), every fallible call returns b3d_status
 * (b3d.h:26-32) and leaves a message in the thread-local b3d_last_error()
 * (b3d_capi.cpp:22,118), no exception crosses the ABI (guarded(),
 * b3d_capi.cpp:33-48), caller-owned output buffers (b3d.h:130-131).
 *
 * Part 1 keeps the reference's on-path entry points with their exact
 * signatures and semantics (GPU-backed).  Part 2 adds the batched entry
 * points the reference's internal seams correspond to:
 * render-many (render_batch, renderer.hpp:42-43), score-many
 * (score_cells / windowed_log_likelihood_multi, inference.hpp:111-113,
 * likelihood.hpp:65-69) and the enumerate/reduce/sample stage
 * (coarse_to_fine_propose / sample_categorical, inference.hpp:136-138,
 * inference.cpp:345-353).
 *
 * Memory: every pointer argument of part 2 may be a host pointer or a CUDA
 * device pointer (detected with cudaPointerGetAttributes).  A call whose
 * pointers are all device pointers is asynchronous on the context's stream;
 * otherwise the call copies through the stream and returns when the results
 * are in the caller's buffers.  Inputs in page-locked (pinned) host memory
 * are read in stream order: such a buffer must stay unchanged until the next
 * call that returns results to the host (or b3d_gpu_synchronize).
 */
#ifndef B3D_B200_H
#define B3D_B200_H

#include <stddef.h>
#include <stdint.h>

#define B3D_API __attribute__((visibility("default")))

#ifdef __cplusplus
extern "C" {
#endif

/* ===================== part 1: reference-compatible ===================== */

/* b3d.h:26-32 */
typedef enum b3d_status {
  B3D_OK = 0,
  B3D_ERROR = 1,
  B3D_ERROR_CONFIG = 2,
  B3D_ERROR_IO = 3,
  B3D_ERROR_NUMERIC = 4
} b3d_status;

/* b3d.h:45-49 */
typedef struct b3d_intrinsics {
  double fx, fy, cx, cy;
  uint32_t width, height;
  double near_m, far_m;
} b3d_intrinsics;

/* b3d.h:52-55: unit quaternion (w, x, y, z) plus translation, meters. */
typedef struct b3d_pose {
  double qw, qx, qy, qz;
  double tx, ty, tz;
} b3d_pose;

/* b3d.h:34,37 */
B3D_API const char* b3d_version(void);
B3D_API const char* b3d_last_error(void);

/* b3d.h:39,59-68 (SDPT on disk: "SDPT" | u32 w | u32 h | f32[w*h]) */
typedef struct b3d_depth_image b3d_depth_image;
B3D_API b3d_status b3d_depth_image_create(uint32_t width, uint32_t height,
                                          const float* depth, b3d_depth_image** out);
B3D_API b3d_status b3d_depth_image_load(const char* path, b3d_depth_image** out);
B3D_API b3d_status b3d_depth_image_save(const b3d_depth_image* img, const char* path);
B3D_API uint32_t b3d_depth_image_width(const b3d_depth_image* img);
B3D_API uint32_t b3d_depth_image_height(const b3d_depth_image* img);
B3D_API const float* b3d_depth_image_data(const b3d_depth_image* img);
B3D_API void b3d_depth_image_destroy(b3d_depth_image* img);

/* b3d.h:110-115 -- windowed depth likelihood; window < 0 selects the
 * untruncated form.  Same semantics as the reference (b3d_capi.cpp:276-295),
 * including B3D_ERROR for an all-sentinel rendered image; runs on GPU 0. */
B3D_API b3d_status b3d_log_likelihood(const b3d_depth_image* observed,
                                      const b3d_depth_image* rendered,
                                      const b3d_intrinsics* k, double p_outlier,
                                      double sigma_noise, double sigma_max,
                                      int window, double* out);

/* ---- object models, libraries, scenes (b3d.h:40-43,72-101) ---- */
typedef struct b3d_object_model b3d_object_model;
typedef struct b3d_library b3d_library;
typedef struct b3d_scene b3d_scene;
typedef struct b3d_particles b3d_particles;

/* SVOX on disk ("SVOX" | f32 res | f32 origin[3] | u32 n | i32[3n]);
 * ObjectModel::from_grid: voxel_to_mesh in stored voxel order + mesh_bounds. */
B3D_API b3d_status b3d_model_load(const char* path, int id, b3d_object_model** out);
B3D_API b3d_status b3d_model_save(const b3d_object_model* model, const char* path);
B3D_API b3d_status b3d_model_bbox(const b3d_object_model* model, double extents[3]);
B3D_API b3d_status b3d_model_resolution(const b3d_object_model* model, double* out);
B3D_API b3d_status b3d_model_voxel_count(const b3d_object_model* model, size_t* out);
B3D_API void b3d_model_destroy(b3d_object_model* model);
/* In-memory model (extension): n voxels (i,j,k) in stored order. */
B3D_API b3d_status b3d_model_from_voxels(const int32_t* voxels, size_t n, double resolution,
                                         const double origin[3], int id,
                                         b3d_object_model** out);
/* The model's mesh (extension; views owned by the model). */
B3D_API b3d_status b3d_model_mesh(const b3d_object_model* model, const double** vertices,
                                  uint64_t* n_vertices, const uint32_t** triangles,
                                  uint64_t* n_triangles);

/* Manifest JSON {"models": [{"id", "path"}]} with paths relative to it. */
B3D_API b3d_status b3d_library_open(const char* manifest_path, b3d_library** out);
/* In-memory library (extension): copies of models[0..n), object id = index. */
B3D_API b3d_status b3d_library_create(const b3d_object_model* const* models, size_t n,
                                      b3d_library** out);
B3D_API size_t b3d_library_size(const b3d_library* lib);
B3D_API void b3d_library_destroy(b3d_library* lib);

/* Scene JSON: {"table": {"width", "height"[, "thickness"]}, "children":
 * [{"object_id", "face", "dx", "dy", "dtheta"}]} (b3d.h:92-98). */
B3D_API b3d_status b3d_scene_from_json(const char* json, const b3d_library* lib,
                                       b3d_scene** out);
B3D_API b3d_status b3d_scene_to_json(const b3d_scene* scene, char** out_json);
B3D_API void b3d_scene_destroy(b3d_scene* scene);
B3D_API void b3d_string_free(char* s);

/* b3d.h:107-108 -- render_depth of the scene at `camera` (camera-to-world),
 * on the device: table, then children in order (draw order = ids). */
B3D_API b3d_status b3d_render(const b3d_scene* scene, const b3d_pose* camera,
                              const b3d_intrinsics* k, b3d_depth_image** out);

/* b3d.h:121-141 -- run_smc over the library with the `infer` config schema
 * (intrinsics required; table, sigma_max, window >= 0, schedule
 * (<= 4 refine stages), noise_grid, particles, resample_threshold,
 * n_objects, threads accepted), every render+score on the device. */
B3D_API b3d_status b3d_infer(const b3d_depth_image* observed, const b3d_pose* camera,
                             const b3d_library* lib, const char* config_json, uint64_t seed,
                             b3d_particles** out);
B3D_API size_t b3d_particles_count(const b3d_particles* p);
B3D_API b3d_status b3d_particles_log_evidence(const b3d_particles* p, double* out);
/* One JSON object per line: children, noise, log_weight. */
B3D_API b3d_status b3d_particles_to_jsonl(const b3d_particles* p, char** out);
B3D_API b3d_status b3d_particles_type_marginal(const b3d_particles* p, double* probs,
                                               size_t capacity);
B3D_API b3d_status b3d_particles_map_pose(const b3d_particles* p, size_t index,
                                          b3d_pose* out);
B3D_API void b3d_particles_destroy(b3d_particles* p);

/* ===================== part 2: batched GPU entry points ================= */

typedef struct b3d_gpu_context b3d_gpu_context;

/* NoiseParams (likelihood.hpp:10-13) */
typedef struct b3d_noise {
  double p_outlier;
  double sigma_noise;
} b3d_noise;

enum { B3D_PREFACTOR_PRINTED = 0, B3D_PREFACTOR_UNIFORM = 1 };
enum { B3D_GRID_PRODUCT = 0, B3D_GRID_ZIP = 1 };
/* noise entries / distinct sigmas per fused launch; calls with more are split
 * into several launches (no limit on the call) */
enum { B3D_MAX_NOISE = 12, B3D_MAX_SIGMAS = 4 };

/* 6-DoF hypothesis grid generated on the device.  Translation lattice per
 * axis: center.t - extent + 2*extent*i/(n-1) (tracking.cpp:34-35); rotation
 * q = normalized(center.q * dq[r]) for a table of unit quaternions dq
 * (w,x,y,z).  PRODUCT: index = ((ix*ny + iy)*nz + iz)*n_rot + r.  ZIP:
 * index i pairs translation i with rotation i (nx*ny*nz == n_rot). */
typedef struct b3d_pose_grid {
  b3d_pose center;
  double extent[3];
  uint32_t count[3];
  const double* rotations; /* n_rot x 4 */
  uint32_t n_rot;
  uint32_t mode;
} b3d_pose_grid;

/* One stage's reduction: argmax (first index of the strict max), max,
 * logsumexp, sum exp(x-max), and one categorical draw (u < running CDF,
 * inference.cpp:345-353) with the stream's next uniform(). */
typedef struct b3d_stage_result {
  uint64_t argmax;
  uint64_t sample;
  double max_score;
  double logsumexp;
  double total;
  double sample_logp;
  uint32_t all_zero;
  uint32_t n_nonfinite;
  uint32_t sample_fallback;
  uint32_t reserved;
} b3d_stage_result;

/* Context: device, stream, uploaded meshes, observation, likelihood config. */
B3D_API b3d_status b3d_gpu_context_create(int device, b3d_gpu_context** out);
B3D_API void b3d_gpu_context_destroy(b3d_gpu_context* ctx);
/* Use an external cudaStream_t (NULL = the context's own stream).  The own
 * stream is a blocking stream: it is ordered with work on the legacy default
 * stream (e.g. torch's default stream), so device inputs produced there are
 * complete before a call reads them, and events recorded there bracket it. */
B3D_API b3d_status b3d_gpu_set_stream(b3d_gpu_context* ctx, void* cuda_stream);
B3D_API b3d_status b3d_gpu_synchronize(b3d_gpu_context* ctx);

/* Intrinsics plus camera-to-world pose (NULL = identity). */
B3D_API b3d_status b3d_gpu_set_camera(b3d_gpu_context* ctx, const b3d_intrinsics* k,
                                      const b3d_pose* camera);
/* TriangleMesh (geometry.hpp:84-89): vertices n_vertices x 3 (fp64, model
 * frame), triangles n_triangles x 3 (u32).  Triangle order = draw order. */
B3D_API b3d_status b3d_gpu_upload_mesh(b3d_gpu_context* ctx, const double* vertices,
                                       uint64_t n_vertices, const uint32_t* triangles,
                                       uint64_t n_triangles, int32_t* out_mesh_id);
/* Fused score all-gather for one-process-per-GPU runs:
 * score_poses / score_grid / score_grid_range / enumerate_grid launches of
 * this context also store score (h, e) into peer_ptrs[r][(offset + h) *
 * n_noise + e] for r < n_peers -- device addresses of each rank's copy of the
 * global score array, mapped on this device (e.g. symmetric memory over
 * NVLink) -- when that element index is below `capacity` (elements per
 * array).  The caller makes the ranks meet (b3d_gpu_shard_barrier) before
 * reading, and must not let a rank write an array a peer may still be
 * reading (alternate two arrays: see b3d_gpu_enumerate_shard).  n_peers = 0
 * turns it off.  Other score paths (contact cells, camera mode, chains) never
 * store to peers. */
B3D_API b3d_status b3d_gpu_set_score_peers(b3d_gpu_context* ctx, const uint64_t* peer_ptrs,
                                           uint32_t n_peers, uint64_t offset,
                                           uint64_t capacity);
/* Device barrier of the ranks of a sharded stage: rank `rank` stores `epoch`
 * into slot `rank` of every rank's signal pad (signal_ptrs[r]: n_ranks u64,
 * mapped on this device, zero-initialised once) with a system-scope release
 * after a system fence, then waits until every slot of its own pad holds at
 * least `epoch` (acquire).  Epochs must grow from call to call.  Stream
 * ordered on the context stream; a rank that never arrives makes the call
 * fail after 20 s instead of hanging the device. */
B3D_API b3d_status b3d_gpu_shard_barrier(b3d_gpu_context* ctx, const uint64_t* signal_ptrs,
                                         uint32_t n_ranks, uint32_t rank, uint64_t epoch);
/* Diagnostics: the exchange protocol (stores into every rank's array half,
 * signal-pad barrier, reads of the own half) for n_ranks ranks emulated as the
 * blocks of one cooperative launch on this device, `rounds` epochs, one rank
 * per epoch holding its reads hold_ns apart.  *errors = reads that saw a value
 * other than the epoch's (0 double-buffered; single-buffered shows the race
 * the double buffer removes). */
B3D_API b3d_status b3d_gpu_test_exchange_emulation(b3d_gpu_context* ctx, uint32_t n_ranks,
                                                   uint32_t rounds, int32_t double_buffered,
                                                   uint64_t hold_ns, uint32_t* errors);
/* Back-face culling in score-many (default on).  Applies only to meshes the
 * upload found closed (every directed edge matched by its reverse) and only
 * to hypotheses with no vertex in front of z = near: a back face of a closed
 * solid never holds the nearest depth of a pixel, so the
 * scores are unchanged.  Render-many (depth/ids) never culls. */
B3D_API b3d_status b3d_gpu_set_culling(b3d_gpu_context* ctx, int enable);
/* +1 / -1: closed mesh, outward / inward wound; 0: not closed (no culling).
 * The host-only form runs the same test on caller memory. */
B3D_API b3d_status b3d_mesh_cull_sign(const double* vertices, uint64_t n_vertices,
                                      const uint32_t* triangles, uint64_t n_triangles,
                                      int32_t* out);
B3D_API b3d_status b3d_gpu_mesh_cull_sign(const b3d_gpu_context* ctx, int32_t mesh_id,
                                          int32_t* out);
/* Observed depth image (W x H fp32, sentinel = (float)far). */
B3D_API b3d_status b3d_gpu_set_observation(b3d_gpu_context* ctx, const float* depth);
/* Likelihood settings (likelihood.hpp:65-69), any number of noise entries.
 * Score-many (object mode) is the score_cells seam, observation_loglik_cached_multi
 * (inference.cpp:40-83): an entry outside the noise support (p_outlier not in
 * [0,1], sigma_noise <= 0 or > sigma_max) scores -inf, window < 0 is the
 * untruncated likelihood.  The camera paths are windowed_log_likelihood_multi
 * itself (tracking.cpp:98-101): such entries and window < 0 are errors there,
 * sigma_noise > sigma_max is scored.  window < 0 or p_outlier < 1e-6 run on the
 * fp64 image path (render, then exact_score.cu) so -inf and tiny-floor terms
 * are the reference's. */
B3D_API b3d_status b3d_gpu_set_likelihood(b3d_gpu_context* ctx, const b3d_noise* noise,
                                          uint32_t n_noise, double sigma_max, int window,
                                          int prefactor);

/* score-many: scores[i*n_noise + e] = windowed log-likelihood of the
 * observation given the render of mesh at poses[i] (model-to-world).
 * status[i] = 1 marks an empty render (score -inf; the reference throws). */
B3D_API b3d_status b3d_gpu_score_poses(b3d_gpu_context* ctx, int32_t mesh_id,
                                       const b3d_pose* poses, uint64_t n, double* scores,
                                       uint8_t* status);
B3D_API b3d_status b3d_gpu_score_grid(b3d_gpu_context* ctx, int32_t mesh_id,
                                      const b3d_pose_grid* grid, double* scores,
                                      uint8_t* status);
/* render-many: depth n x W x H (fp32, sentinel = far) and optional
 * draw_index n x W x H (int32, triangle index in mesh order, -1 = none). */
B3D_API b3d_status b3d_gpu_render_poses(b3d_gpu_context* ctx, int32_t mesh_id,
                                        const b3d_pose* poses, uint64_t n, float* depth,
                                        int32_t* draw_index);
/* Stage reduction over scores[i*stride + col], i < n.  rng_state (5 x u64:
 * seed, s0..s3 of the reference Rng) is advanced by one uniform() when not
 * NULL; NULL skips the draw.  probs (optional, n) receives the normalised
 * CellScores (inference.cpp:315-330). */
B3D_API b3d_status b3d_gpu_stage_reduce(b3d_gpu_context* ctx, const double* scores,
                                        uint64_t n, uint32_t stride, uint32_t col,
                                        uint64_t* rng_state, b3d_stage_result* out,
                                        double* probs);

/* Fixed scene content rendered once per context and composited under every
 * hypothesis (render_partial / compose_render, inference.cpp:102-109,172-184):
 * instances in draw order (table first, then base children).  Triangle draw
 * indices run across the instances; hypotheses' triangles follow them.
 * n = 0 removes the base scene. */
B3D_API b3d_status b3d_gpu_set_base_scene(b3d_gpu_context* ctx, const int32_t* mesh_ids,
                                          const b3d_pose* model_to_world, uint32_t n);

/* Table-contact hypotheses of one (object, face): the cell centres of an
 * n_dx x n_dy x n_dtheta partition of the support (stage0_cells,
 * inference.cpp:208-238), posed by contact_to_pose (scene_graph.cpp:97-121)
 * on a table with its top at z = 0 of the world frame (ObjectModel::table).
 * index = (ix * n_dy + iy) * n_dtheta + it. */
typedef struct b3d_contact_grid {
  double table_w, table_h;
  double aabb_min[3], aabb_max[3]; /* object model-frame AABB (mesh_bounds) */
  int32_t face;                    /* 1..6 */
  uint32_t count[3];               /* n_dx, n_dy, n_dtheta */
} b3d_contact_grid;

B3D_API b3d_status b3d_gpu_score_contact_grid(b3d_gpu_context* ctx, int32_t mesh_id,
                                              const b3d_contact_grid* grid, double* scores,
                                              uint8_t* status);
/* Host poses (model-to-world) of a contact grid, n_dx * n_dy * n_dtheta of them. */
B3D_API b3d_status b3d_contact_grid_poses(const b3d_contact_grid* grid, b3d_pose* out);

/* subdivide_cell (inference.cpp:240-259): the n_dx x n_dy x n_dtheta children
 * of a parent contact cell, child (ix, iy, it) spanning
 * [lo + (hi - lo) ix / n, lo + (hi - lo) (ix + 1) / n) per dimension; each is
 * scored at its centre (cell_center_child, inference.cpp:126-137).  The
 * contact grid above is the stage-0 parent [0, table - footprint] x [0, 2 pi). */
typedef struct b3d_contact_cells {
  b3d_contact_grid grid; /* table, object bounds, face, child counts */
  double dx_lo, dx_hi, dy_lo, dy_hi, dtheta_lo, dtheta_hi;
} b3d_contact_cells;
B3D_API b3d_status b3d_gpu_score_contact_cells(b3d_gpu_context* ctx, int32_t mesh_id,
                                               const b3d_contact_cells* cells, double* scores,
                                               uint8_t* status);
B3D_API b3d_status b3d_contact_cells_poses(const b3d_contact_cells* cells, b3d_pose* out);

/* One stage of a device-resident enumeration schedule: a pose grid around
 * the previous stage's chosen pose (the caller's centre for stage 0), its
 * likelihood settings (sigma_max and prefactor come from the context), and
 * how the next centre is chosen: B3D_SELECT_SAMPLE draws from the stage's
 * categorical posterior (coarse_to_fine_propose, inference.cpp:357-396),
 * B3D_SELECT_ARGMAX keeps the MAP pose (track_camera, tracking.cpp:132-138). */
enum { B3D_SELECT_SAMPLE = 0, B3D_SELECT_ARGMAX = 1 };
typedef struct b3d_stage_spec {
  double extent[3];
  uint32_t count[3];
  const double* rotations; /* n_rot x 4 (w,x,y,z), host or device */
  uint32_t n_rot;
  uint32_t mode;
  b3d_noise noise;
  int32_t window;
  uint32_t select;
} b3d_stage_spec;

/* Runs n_stages enumerate -> score -> reduce -> select stages back to back
 * on the context's stream with no host round trip between stages.
 * rng_state (5 x u64, advanced by one uniform() per SAMPLE stage), results
 * (n_stages) and centers (n_stages + 1; centers[0] = *center) are caller
 * buffers, host or device. */
B3D_API b3d_status b3d_gpu_coarse_to_fine(b3d_gpu_context* ctx, int32_t mesh_id,
                                          const b3d_pose* center,
                                          const b3d_stage_spec* stages, uint32_t n_stages,
                                          uint64_t* rng_state, b3d_stage_result* results,
                                          b3d_pose* centers);

/* n_samples categorical draws from the posterior softmax(scores) with
 * consecutive uniform() values of rng_state (each draw has
 * sample_categorical semantics, inference.cpp:345-353); also fills *out
 * like b3d_gpu_stage_reduce (argmax, logsumexp; its `sample` = the first
 * draw). */
B3D_API b3d_status b3d_gpu_sample_many(b3d_gpu_context* ctx, const double* scores, uint64_t n,
                                       uint32_t stride, uint32_t col, uint64_t* rng_state,
                                       uint32_t n_samples, uint64_t* samples,
                                       b3d_stage_result* out);

/* One enumeration stage through the host boundary in a single call:
 * score-many of poses (model-to-world) + the stage reduction of noise entry 0
 * (argmax, logsumexp, one draw when rng_state != NULL); optional scores
 * (n x n_noise).  One synchronisation per call. */
B3D_API b3d_status b3d_gpu_enumerate_poses(b3d_gpu_context* ctx, int32_t mesh_id,
                                           const b3d_pose* poses, uint64_t n,
                                           uint64_t* rng_state, b3d_stage_result* out,
                                           double* scores);
/* One frame of the hot loop (score_cells after ObservationCache::build,
 * inference.cpp:261-353): b3d_gpu_set_observation(depth) followed by
 * b3d_gpu_enumerate_poses in one call (one boundary crossing). */
B3D_API b3d_status b3d_gpu_enumerate_observed(b3d_gpu_context* ctx, int32_t mesh_id,
                                              const float* depth, const b3d_pose* poses,
                                              uint64_t n, uint64_t* rng_state,
                                              b3d_stage_result* out, double* scores);

/* One stage of a hypothesis-sharded enumeration in one call.
 * Each rank's global score array (scores[r], peer-mapped) holds 2 x n_total
 * x n_noise doubles: exchange `epoch` uses half (epoch & 1), so a rank never
 * writes the half a slower peer may still be reducing (the barrier of
 * exchange e+1 orders every rank's reduction of e before anyone's writes of
 * e+2).  The call: b3d_gpu_set_observation(depth) when depth != NULL; score
 * the n_local hypotheses (poses; or grid rows [offset, offset + n_local) of a
 * global grid of n_total rows, rows [0, n_local) of a per-rank grid of any
 * other size) with every score also stored into every rank's array at row
 * offset + i (the all-gather fused into the score kernel); the signal-pad
 * barrier; the stage reduction (argmax, logsumexp, one draw with rng_state)
 * of this rank's complete array.  Every rank computes the same result,
 * bitwise, for any rank count.  out / rng_state may be host (one read-back)
 * or device memory. */
typedef struct b3d_shard_exchange {
  uint32_t n_ranks; /* <= 8 */
  uint32_t rank;
  uint64_t offset;  /* this rank's first global hypothesis */
  uint64_t n_total; /* global hypotheses */
  uint64_t scores[8];  /* rank r's global score array (2 x n_total x n_noise) */
  uint64_t signals[8]; /* rank r's signal pad (n_ranks u64) */
  uint64_t epoch;      /* > the previous exchange's */
} b3d_shard_exchange;
B3D_API b3d_status b3d_gpu_enumerate_shard(b3d_gpu_context* ctx, int32_t mesh_id,
                                           const float* depth, const b3d_pose* poses,
                                           const b3d_pose_grid* grid, uint64_t n_local,
                                           const b3d_shard_exchange* ex, uint64_t* rng_state,
                                           b3d_stage_result* out);

/* score-many over a device pose grid followed by the stage reduction of
 * scores[:, 0] (argmax, logsumexp, one draw with rng_state if non-NULL) in
 * one call.  All buffers device memory; asynchronous on the context stream. */
B3D_API b3d_status b3d_gpu_enumerate_grid(b3d_gpu_context* ctx, int32_t mesh_id,
                                          const b3d_pose_grid* grid, uint64_t* rng_state,
                                          b3d_stage_result* out, double* scores);

/* Score hypotheses [first, first + n) of a device pose grid (one rank's
 * shard of a large enumeration); scores[i] is hypothesis
 * first + i. */
B3D_API b3d_status b3d_gpu_score_grid_range(b3d_gpu_context* ctx, int32_t mesh_id,
                                            const b3d_pose_grid* grid, uint64_t first,
                                            uint64_t n, double* scores, uint8_t* status);

/* ---- camera mode: a scene of mesh instances under camera hypotheses ----
 * render_instances (renderer.cpp:153-189) of any number of instances in draw
 * order (draw indices continue across instances); model_to_world[i] is used
 * verbatim, as scene_instances (inference.cpp:172-184) produces it.  Up to
 * B3D_MAX_INSTANCES instances render and score in one fused launch; larger
 * scenes render per group of B3D_MAX_INSTANCES, merged per pixel (the same
 * depth and ids), and score through the fp64 image likelihood. */
enum { B3D_MAX_INSTANCES = 16 };
B3D_API b3d_status b3d_gpu_set_camera_scene(b3d_gpu_context* ctx, const int32_t* mesh_ids,
                                            const b3d_pose* model_to_world, uint32_t n);
/* render-many / score-many over camera-to-world poses cameras[0..n) (host or
 * device memory, used verbatim like track_camera's Pose values). */
B3D_API b3d_status b3d_gpu_render_cameras(b3d_gpu_context* ctx, const b3d_pose* cameras,
                                          uint64_t n, float* depth, int32_t* draw_index);
B3D_API b3d_status b3d_gpu_score_cameras(b3d_gpu_context* ctx, const b3d_pose* cameras,
                                         uint64_t n, double* scores, uint8_t* status);

/* TrackSearch (tracking.hpp:25-34). */
typedef struct b3d_track_search {
  double pos_extent;   /* +- m on distance */
  double angle_extent; /* +- rad on azimuth / altitude */
  int32_t points_per_dim;
  int32_t refine_stages;
  double refine_factor;
  int32_t beam_width;
  int32_t reserved;
} b3d_track_search;

/* track_camera (tracking.cpp:59-172) over the camera scene: frames are
 * n_frames depth images (W x H fp32 each, host or device); every lattice
 * stage is scored on the device.  Likelihood: the context's settings (one
 * noise entry).  out_poses[n_frames] (frame 0 = initial), optional
 * out_frame_ms[n_frames] (per-frame wall time, the reference's close_frame).
 * camera_pose_from_spherical / camera_pose_to_spherical run on the host
 * with the reference's libm calls (generative.cpp:35-85). */
B3D_API b3d_status b3d_gpu_track_camera(b3d_gpu_context* ctx, const float* frames,
                                        uint32_t n_frames, const b3d_pose* initial,
                                        const b3d_track_search* search, b3d_pose* out_poses,
                                        double* out_frame_ms);
/* make_box_mesh (scene_graph.cpp:37-58): 8 vertices, 12 triangles. */
B3D_API b3d_status b3d_box_mesh(const double lo[3], const double hi[3], double vertices[24],
                                uint32_t triangles[36]);
/* contact_to_pose (scene_graph.cpp:97-121) with the table's extents given
 * directly; B3D_ERROR for out-of-range contact parameters. */
B3D_API b3d_status b3d_contact_to_pose(double table_w, double table_h, const double aabb_min[3],
                                       const double aabb_max[3], int32_t face, double dx,
                                       double dy, double dtheta, b3d_pose* out);
/* rotated_bounds (scene_graph.cpp:73-89): AABB of the object with `face` down. */
B3D_API b3d_status b3d_rotated_bounds(const double aabb_min[3], const double aabb_max[3],
                                      int32_t face, double lo[3], double hi[3]);
/* generative.cpp:35-59 / 61-85 on the host (exposed for tests and callers). */
B3D_API b3d_status b3d_camera_pose_from_spherical(double distance, double azimuth,
                                                  double altitude, b3d_pose* out);
B3D_API int b3d_camera_pose_to_spherical(const b3d_pose* pose, double tol, double* distance,
                                         double* azimuth, double* altitude);

/* ---- sequential Monte Carlo over scene graphs (run_smc, inference.cpp:398-520) ----
 * Library object: an uploaded mesh and its model-frame AABB (mesh_bounds). */
typedef struct b3d_smc_object {
  int32_t mesh_id;
  int32_t reserved;
  double aabb_min[3], aabb_max[3];
} b3d_smc_object;
/* ScheduleStage (inference.hpp:22-28) */
typedef struct b3d_schedule_stage {
  uint32_t n_dx, n_dy, n_dtheta;
} b3d_schedule_stage;
/* InferenceContext pieces (inference.hpp:58-72): table (top plane at z = 0,
 * rendered first, identity pose), schedule, noise grid, model settings. */
typedef struct b3d_smc_config {
  double table_w, table_h;
  int32_t table_mesh;
  uint32_t n_refine; /* any number of refine stages (Schedule::refine) */
  b3d_schedule_stage stage0;
  const b3d_schedule_stage* refine; /* n_refine entries */
  const b3d_noise* noise_grid;
  uint32_t n_noise_grid; /* any size; entries must lie in the noise support */
  uint32_t n_objects;    /* objects placed, >= 1 (inference.cpp:495) */
  uint32_t n_particles;
  double resample_threshold;
  double sigma_max;
  int32_t window; /* < 0: untruncated likelihood (ModelConfig::windowed = false) */
  int32_t prefactor;
  uint64_t* renders; /* optional out: hypotheses rendered+scored on the device
                        (distinct evaluations; particles sharing a base scene,
                        object, noise entry and cell share them) */
} b3d_smc_config;
typedef struct b3d_smc_child {
  int32_t object_id, face;
  double dx, dy, dtheta; /* ContactParams */
} b3d_smc_child;
typedef struct b3d_smc_particle {
  b3d_smc_child* children; /* caller storage for cfg->n_objects entries */
  int32_t n_children, noise_index;
  double log_target, log_weight;
} b3d_smc_particle;
/* run_smc: smc_init, smc_extend per further object, ESS-triggered systematic
 * resampling, log-evidence; the reference's Rng streams (rng.split(1, i),
 * rng.split(arity + 1, i), rng.split(0x5e5a, 0).split(stage)).  Every
 * render+score runs on the device (stage 0 per (object, face) with the whole
 * noise grid, refinement batched across particles).  Uses the context's
 * camera and observation; replaces its likelihood settings and base scene. */
B3D_API b3d_status b3d_gpu_run_smc(b3d_gpu_context* ctx, const b3d_smc_object* library,
                                   uint32_t n_library, const b3d_smc_config* cfg, uint64_t seed,
                                   b3d_smc_particle* particles, double* log_evidence);

/* Reference Rng seeding (rng.cpp:20-28), for building rng_state. */
B3D_API void b3d_rng_seed(uint64_t seed, uint64_t state[5]);
B3D_API void b3d_rng_split(const uint64_t state[5], uint64_t k0, uint64_t k1, uint64_t k2,
                           uint64_t out[5]);

/* voxel_to_mesh on the device (8f.4, for large grids): the same vertices,
 * vertex numbering and triangle order as b3d_voxel_to_mesh / the reference's
 * voxel_to_mesh (geometry.cpp:142-177), built with hash sets and prefix scans
 * instead of the sequential first-seen walk.  voxels: host or device int32
 * n x 3 with coordinates in [-2^20+1, 2^20-2]; vertices / triangles: host or
 * device, capacity 8n x 3 doubles / 12n x 3 uint32.  Synchronous. */
B3D_API b3d_status b3d_gpu_voxel_to_mesh(b3d_gpu_context* ctx, const int32_t* voxels, uint64_t n,
                                         double resolution, const double origin[3],
                                         double* vertices, uint32_t* triangles,
                                         uint64_t* n_vertices, uint64_t* n_triangles);

/* sample_observation (likelihood.cpp:44-80; replaces the reference's
 * b3d::sample_observation, likelihood.hpp:34-35): a synthetic observed depth
 * image from a rendered one -- |cloud| draws, each an outlier uniform in the
 * viewing frustum with probability p_outlier, else a rendered point drawn with
 * replacement plus N(0, sigma) per axis, reprojected (lround) and kept as the
 * nearest fp32 depth.  Bitwise the reference's on the same Rng state, which
 * is advanced in place.  Host code: one sequential Rng stream.
 * Errors: invalid noise (sigma <= 0, p outside [0,1]) or an all-sentinel
 * render -> B3D_ERROR (the reference throws ErrorCode::invalid). */
B3D_API b3d_status b3d_sample_observation(const b3d_intrinsics* k, const float* rendered,
                                          const b3d_noise* noise, uint64_t rng_state[5],
                                          float* out);
/* n frames at once as generate_orbit_sequence draws them
 * (tracking.cpp:199-202): frame i uses rng_state.split(split_key, i)
 * (0x0f in the reference); frames run on all host threads.  rendered / out:
 * n x H x W fp32.  rng_state is not advanced. */
B3D_API b3d_status b3d_sample_observations(const b3d_intrinsics* k, const float* rendered,
                                           uint64_t n, const b3d_noise* noise,
                                           const uint64_t rng_state[5], uint64_t split_key,
                                           float* out);

/* voxel_to_mesh (geometry.cpp:142-177) on the host: exterior faces of the
 * occupied voxels in stored order.  Capacities: vertices >= 24*n doubles,
 * triangles >= 36*n u32. */
B3D_API b3d_status b3d_voxel_to_mesh(const int32_t* voxels, uint64_t n, double resolution,
                                     const double origin[3], double* vertices,
                                     uint32_t* triangles, uint64_t* n_vertices,
                                     uint64_t* n_triangles);

#ifdef __cplusplus
}
#endif
#endif /* B3D_B200_H */
