// ref_bridge.cpp -- ORACLE TEST INFRASTRUCTURE, not product code.
//
// extern "C" entry points into the reference's OWN C++ implementation
// (/root/reference/proj/src/core/*.cpp compiled unmodified against
// oracle/ref_shim/, see oracle/Makefile `ref`), for the internal seams that
// b3d.h does not export: raster_mesh / render_instances, the windowed and full
// likelihoods, score_cells / coarse_to_fine_propose, track_camera,
// sample_observation, voxel_to_mesh and the pose helpers.  The reference's
// public C ABI (b3d_render, b3d_log_likelihood, b3d_infer, ...) is linked into
// the same library and called directly.
//
// Used only by tests/ and tests/golden/make_ref_golden.py to produce golden
// fixtures; nothing in the product links or loads it.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "core/error.hpp"
#include "core/geometry.hpp"
#include "core/inference.hpp"
#include "core/likelihood.hpp"
#include "core/parallel.hpp"
#include "core/renderer.hpp"
#include "core/rng.hpp"
#include "core/scene_graph.hpp"
#include "core/tracking.hpp"

#define REFB_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const b3d::Error& e) {
    g_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

// same layout as b3d_intrinsics (b3d.h:45-49)
struct RefIntr {
  double fx, fy, cx, cy;
  uint32_t width, height;
  double near_m, far_m;
};

b3d::CameraIntrinsics intr(const RefIntr* k) {
  b3d::CameraIntrinsics o;
  o.fx = k->fx;
  o.fy = k->fy;
  o.cx = k->cx;
  o.cy = k->cy;
  o.width = k->width;
  o.height = k->height;
  o.near = k->near_m;
  o.far = k->far_m;
  return o;
}

// pose as 7 doubles (qw, qx, qy, qz, tx, ty, tz), b3d_pose order
b3d::Pose pose_in(const double* p) {
  b3d::Pose o;
  o.rotation = b3d::Quat(p[0], p[1], p[2], p[3]);
  o.translation = b3d::Vec3(p[4], p[5], p[6]);
  return o;
}

void pose_out(const b3d::Pose& p, double* o) {
  o[0] = p.rotation.w();
  o[1] = p.rotation.x();
  o[2] = p.rotation.y();
  o[3] = p.rotation.z();
  o[4] = p.translation.x();
  o[5] = p.translation.y();
  o[6] = p.translation.z();
}

b3d::TriangleMesh mesh_in(const double* verts, uint64_t nv, const uint32_t* tris, uint64_t nt) {
  b3d::TriangleMesh m;
  m.vertices.reserve(nv);
  for (uint64_t i = 0; i < nv; ++i)
    m.vertices.emplace_back(verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]);
  m.triangles.reserve(nt);
  for (uint64_t i = 0; i < nt; ++i) m.triangles.push_back({tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]});
  return m;
}

b3d::DepthImage image_in(const float* d, uint32_t w, uint32_t h) {
  b3d::DepthImage img;
  img.width = w;
  img.height = h;
  img.depth.assign(d, d + static_cast<size_t>(w) * h);
  return img;
}

b3d::VoxelGrid grid_in(const int32_t* vox, uint64_t n, double res, const double* origin) {
  b3d::VoxelGrid g;
  g.resolution = res;
  g.origin = b3d::Vec3(origin[0], origin[1], origin[2]);
  for (uint64_t i = 0; i < n; ++i) g.occupied.emplace_back(vox[3 * i], vox[3 * i + 1], vox[3 * i + 2]);
  return g;
}

std::vector<b3d::NoiseParams> noise_in(int n, const double* p, const double* sigma) {
  std::vector<b3d::NoiseParams> v(n);
  for (int i = 0; i < n; ++i) v[i] = {p[i], sigma[i]};
  return v;
}

}  // namespace

REFB_API const char* refb_last_error(void) { return g_error.c_str(); }

// ---- pose math (geometry.cpp:11-31, scene_graph.cpp:60-121, generative.cpp:35-59)
REFB_API int refb_compose(const double* a, const double* b, double* out) {
  return guarded([&] { pose_out(b3d::compose(pose_in(a), pose_in(b)), out); });
}
REFB_API int refb_inverse(const double* a, double* out) {
  return guarded([&] { pose_out(b3d::inverse(pose_in(a)), out); });
}
REFB_API int refb_rotation_matrix(const double* a, double* out9) {
  return guarded([&] {
    const b3d::Mat3 m = pose_in(a).rotation_matrix();
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) out9[3 * r + c] = m(r, c);
  });
}
REFB_API int refb_from_axis_angle(const double* axis, double angle, double* out) {
  return guarded([&] {
    pose_out(b3d::Pose::from_axis_angle(b3d::Vec3(axis[0], axis[1], axis[2]), angle), out);
  });
}
REFB_API int refb_camera_pose_from_spherical(double d, double az, double alt, double* out) {
  return guarded([&] { pose_out(b3d::camera_pose_from_spherical(d, az, alt), out); });
}
REFB_API int refb_camera_pose_to_spherical(const double* pose, double tol, double* out3, int* ok) {
  return guarded([&] {
    *ok = b3d::camera_pose_to_spherical(pose_in(pose), out3[0], out3[1], out3[2], tol) ? 1 : 0;
  });
}
// object given by its voxel grid (ObjectModel::from_grid), table by extents
REFB_API int refb_contact_to_pose(double table_w, double table_h, const int32_t* vox, uint64_t n,
                                  double res, const double* origin, int face, double dx, double dy,
                                  double dtheta, double* out) {
  return guarded([&] {
    const b3d::ObjectModel table = b3d::ObjectModel::table(table_w, table_h);
    const b3d::ObjectModel obj = b3d::ObjectModel::from_grid(0, grid_in(vox, n, res, origin));
    pose_out(b3d::contact_to_pose(table, obj, face, {dx, dy, dtheta}), out);
  });
}

// ---- meshes (geometry.cpp:142-177, scene_graph.cpp:26-58)
REFB_API int refb_voxel_to_mesh(const int32_t* vox, uint64_t n, double res, const double* origin,
                                double* verts, uint64_t vcap, uint32_t* tris, uint64_t tcap,
                                uint64_t* nv, uint64_t* nt) {
  return guarded([&] {
    const b3d::TriangleMesh m = b3d::voxel_to_mesh(grid_in(vox, n, res, origin));
    *nv = m.vertices.size();
    *nt = m.triangles.size();
    b3d::require(m.vertices.size() <= vcap && m.triangles.size() <= tcap, b3d::ErrorCode::invalid,
                 "refb_voxel_to_mesh: capacity");
    for (size_t i = 0; i < m.vertices.size(); ++i)
      for (int c = 0; c < 3; ++c) verts[3 * i + c] = m.vertices[i][c];
    for (size_t i = 0; i < m.triangles.size(); ++i)
      for (int c = 0; c < 3; ++c) tris[3 * i + c] = m.triangles[i][c];
  });
}

// ---- renderer (renderer.cpp:112-189)
// Instances in draw order, each a mesh + model_to_world pose; `camera` is
// camera_to_world.  render_instances: fp32(far) background, inverse(camera)
// composed with each instance.
REFB_API int refb_render_instances(const RefIntr* k, int n_inst, const double* const* verts,
                                   const uint64_t* nv, const uint32_t* const* tris,
                                   const uint64_t* nt, const double* poses, const double* camera,
                                   float* out) {
  return guarded([&] {
    std::vector<b3d::TriangleMesh> meshes;
    meshes.reserve(n_inst);
    std::vector<b3d::MeshInstance> inst;
    for (int i = 0; i < n_inst; ++i) meshes.push_back(mesh_in(verts[i], nv[i], tris[i], nt[i]));
    for (int i = 0; i < n_inst; ++i) inst.push_back({&meshes[i], pose_in(poses + 7 * i)});
    const b3d::DepthImage img = b3d::render_instances(inst, pose_in(camera), intr(k));
    std::memcpy(out, img.depth.data(), img.depth.size() * sizeof(float));
  });
}

// ---- likelihood (likelihood.cpp:106-233)
REFB_API int refb_windowed_multi(const RefIntr* k, const float* obs, const float* rend, int n_noise,
                                 const double* p, const double* sigma, double sigma_max,
                                 int window, int prefactor, double* out) {
  return guarded([&] {
    const b3d::CameraIntrinsics kk = intr(k);
    const b3d::ObservationCache cache =
        b3d::ObservationCache::build(image_in(obs, k->width, k->height), kk);
    const std::vector<double> r = b3d::windowed_log_likelihood_multi(
        cache, image_in(rend, k->width, k->height), kk, noise_in(n_noise, p, sigma),
        b3d::visible_volume(kk), sigma_max, window,
        prefactor ? b3d::SigmaPrefactor::uniform : b3d::SigmaPrefactor::printed);
    for (int i = 0; i < n_noise; ++i) out[i] = r[i];
  });
}

REFB_API int refb_full_loglik(const RefIntr* k, const float* obs, const float* rend, double p,
                              double sigma, double sigma_max, int prefactor, double* out) {
  return guarded([&] {
    const b3d::CameraIntrinsics kk = intr(k);
    *out = b3d::full_log_likelihood(
        b3d::depth_to_cloud(image_in(obs, k->width, k->height), kk),
        b3d::depth_to_cloud(image_in(rend, k->width, k->height), kk), {p, sigma},
        b3d::visible_volume(kk), sigma_max,
        prefactor ? b3d::SigmaPrefactor::uniform : b3d::SigmaPrefactor::printed);
  });
}

// Score many poses of one object composited over a fixed base scene: the
// base instances are rendered once (render_instances, renderer.cpp:174-184)
// and each hypothesis rasterizes the object into a copy of it with
// compose(inverse(camera), pose) -- compose_render, inference.cpp:102-109 --
// then windowed_log_likelihood_multi: the body of score_cells' parallel loop
// (inference.cpp:290-313).  n_base = 0 and an identity camera give the
// BASELINE single-object 6-DoF grids.  An empty render throws in the
// reference (likelihood.cpp:159-160); here that hypothesis gets status 1 and
// -inf so the batch continues.  window < 0: full_log_likelihood
// (inference.cpp:51-56, -inf for an empty render).
REFB_API int refb_score_poses(const RefIntr* k, const float* obs, const double* camera, int n_base,
                              const double* const* base_verts, const uint64_t* base_nv,
                              const uint32_t* const* base_tris, const uint64_t* base_nt,
                              const double* base_poses, const double* verts, uint64_t nv,
                              const uint32_t* tris, uint64_t nt, int n, const double* poses,
                              int n_noise, const double* p, const double* sigma, double sigma_max,
                              int window, int prefactor, int threads, double* out, int* status) {
  return guarded([&] {
    const b3d::CameraIntrinsics kk = intr(k);
    const b3d::DepthImage obs_img = image_in(obs, k->width, k->height);
    const b3d::ObservationCache cache = b3d::ObservationCache::build(obs_img, kk);
    const b3d::PointCloud obs_cloud = b3d::depth_to_cloud(obs_img, kk);
    std::vector<b3d::TriangleMesh> base_meshes;
    base_meshes.reserve(n_base);
    std::vector<b3d::MeshInstance> base_inst;
    for (int i = 0; i < n_base; ++i)
      base_meshes.push_back(mesh_in(base_verts[i], base_nv[i], base_tris[i], base_nt[i]));
    for (int i = 0; i < n_base; ++i) base_inst.push_back({&base_meshes[i], pose_in(base_poses + 7 * i)});
    const b3d::Pose cam = pose_in(camera);
    const b3d::DepthImage base = b3d::render_instances(base_inst, cam, kk);
    const b3d::Pose world_to_camera = b3d::inverse(cam);
    const b3d::TriangleMesh mesh = mesh_in(verts, nv, tris, nt);
    const std::vector<b3d::NoiseParams> noise = noise_in(n_noise, p, sigma);
    const b3d::SceneVolume vol = b3d::visible_volume(kk);
    const b3d::SigmaPrefactor pf = prefactor ? b3d::SigmaPrefactor::uniform : b3d::SigmaPrefactor::printed;
    b3d::parallel_for(static_cast<size_t>(n), threads, [&](size_t h) {
      b3d::DepthImage img = base;
      b3d::raster_mesh(img, kk, mesh, b3d::compose(world_to_camera, pose_in(poses + 7 * h)));
      status[h] = 0;
      if (window < 0) {  // observation_loglik_cached: an empty render scores -inf
        const b3d::PointCloud rc = b3d::depth_to_cloud(img, kk);
        status[h] = rc.points.empty() ? 1 : 0;  // flagged like the windowed path
        for (int e = 0; e < n_noise; ++e)
          out[h * n_noise + e] = rc.points.empty()
              ? -INFINITY
              : b3d::full_log_likelihood(obs_cloud, rc, noise[e], vol, sigma_max, pf);
        return;
      }
      try {
        const std::vector<double> r =
            b3d::windowed_log_likelihood_multi(cache, img, kk, noise, vol, sigma_max, window, pf);
        for (int e = 0; e < n_noise; ++e) out[h * n_noise + e] = r[e];
      } catch (const b3d::Error&) {
        for (int e = 0; e < n_noise; ++e) out[h * n_noise + e] = -INFINITY;
        status[h] = 1;
      }
    });
  });
}

// ---- observation sampler (likelihood.cpp:44-80); stream = Rng(seed).split(k0, k1, k2)
REFB_API int refb_sample_observation(const RefIntr* k, const float* rend, double p, double sigma,
                                     uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2,
                                     float* out) {
  return guarded([&] {
    b3d::Rng rng = b3d::Rng(seed).split(k0, k1, k2);
    const b3d::DepthImage img = b3d::sample_observation(image_in(rend, k->width, k->height),
                                                        intr(k), {p, sigma}, rng);
    std::memcpy(out, img.depth.data(), img.depth.size() * sizeof(float));
  });
}

// ---- scene-graph inference stage (inference.cpp:139-396)
// A library of voxel objects (concatenated voxels, per-object counts, one
// resolution and origin per object), a table, the observation and model
// settings.  Returns stage-0 cells + score_cells probabilities, and one
// coarse_to_fine_propose from Rng(seed) over the shared stage-0 table.
struct RefSmcSpec {
  int n_objects;
  const int32_t* voxels;
  const uint64_t* counts;
  const double* resolutions;
  const double* origins;  // 3 per object
  double table_w, table_h;
  double sigma_max;
  int window;  // < 0: full likelihood
  int stage0[3];
  int n_refine;
  const int* refine;  // 3 per refine stage
  int n_noise;
  const double* noise_p;
  const double* noise_sigma;
  int threads;
};

namespace {

struct SmcWorld {
  b3d::Library library;
  std::shared_ptr<const b3d::ObjectModel> table;
  b3d::InferenceContext ctx;
};

std::unique_ptr<SmcWorld> make_world(const RefIntr* k, const float* obs, const double* camera,
                                     const RefSmcSpec* s) {
  auto w = std::make_unique<SmcWorld>();
  const int32_t* vp = s->voxels;
  for (int o = 0; o < s->n_objects; ++o) {
    w->library.push_back(std::make_shared<b3d::ObjectModel>(b3d::ObjectModel::from_grid(
        o, grid_in(vp, s->counts[o], s->resolutions[o], s->origins + 3 * o))));
    vp += 3 * s->counts[o];
  }
  w->table = std::make_shared<b3d::ObjectModel>(b3d::ObjectModel::table(s->table_w, s->table_h));
  b3d::ModelConfig model;
  model.intrinsics = intr(k);
  model.sigma_max = s->sigma_max;
  model.windowed = s->window >= 0;
  model.window = s->window < 0 ? 0 : s->window;
  b3d::Schedule sched;
  sched.stage0 = {s->stage0[0], s->stage0[1], s->stage0[2]};
  sched.refine.clear();
  for (int i = 0; i < s->n_refine; ++i)
    sched.refine.push_back({s->refine[3 * i], s->refine[3 * i + 1], s->refine[3 * i + 2]});
  b3d::NoiseGrid grid;
  grid.entries = noise_in(s->n_noise, s->noise_p, s->noise_sigma);
  w->ctx = b3d::make_inference_context(image_in(obs, k->width, k->height), pose_in(camera),
                                       w->library, w->table, model, sched, grid, {}, s->threads);
  return w;
}

}  // namespace

// Model-to-world poses of the stage-0 cell centres of one (object, face):
// stage0_cells (inference.cpp:208-238) filtered to that branch and noise
// entry 0, then cell_center_child + contact_to_pose (inference.cpp:126-137,
// scene_graph.cpp:97-121).  The cfg3 contact grid is exactly this set.
REFB_API int refb_stage0_cell_poses(const RefIntr* k, const float* obs, const RefSmcSpec* s,
                                    int object, int face, uint64_t cap, uint64_t* n_out,
                                    double* poses) {
  return guarded([&] {
    const double ident[7] = {1, 0, 0, 0, 0, 0, 0};
    auto w = make_world(k, obs, ident, s);
    const std::vector<b3d::Cell> cells = b3d::stage0_cells(w->ctx);
    uint64_t n = 0;
    for (const b3d::Cell& c : cells) {
      if (c.object_id != object || c.face != face || c.noise_index != 0) continue;
      b3d::require(n < cap, b3d::ErrorCode::invalid, "refb_stage0_cell_poses: capacity");
      const b3d::SceneChild ch = b3d::cell_center_child(c, w->library);
      pose_out(b3d::contact_to_pose(*w->table, *ch.object, ch.face, ch.contact), poses + 7 * n);
      ++n;
    }
    *n_out = n;
  });
}

// cells_out: per cell (object, face, noise_index) ints and (dx.lo, dx.hi, dy.lo,
// dy.hi, dth.lo, dth.hi) doubles; scores_out: normalised probabilities.
REFB_API int refb_stage0(const RefIntr* k, const float* obs, const double* camera,
                         const RefSmcSpec* s, uint64_t cap, uint64_t* n_cells, int32_t* cell_ints,
                         double* cell_iv, double* scores, int* all_zero) {
  return guarded([&] {
    auto w = make_world(k, obs, camera, s);
    const b3d::Stage0Table t = b3d::build_stage0(w->ctx, {});
    *n_cells = t.cells.size();
    b3d::require(t.cells.size() <= cap, b3d::ErrorCode::invalid, "refb_stage0: capacity");
    for (size_t i = 0; i < t.cells.size(); ++i) {
      const b3d::Cell& c = t.cells[i];
      cell_ints[3 * i] = c.object_id;
      cell_ints[3 * i + 1] = c.face;
      cell_ints[3 * i + 2] = c.noise_index;
      const double iv[6] = {c.dx.lo, c.dx.hi, c.dy.lo, c.dy.hi, c.dtheta.lo, c.dtheta.hi};
      std::memcpy(cell_iv + 6 * i, iv, sizeof iv);
      scores[i] = t.scored.scores[i];
    }
    *all_zero = t.scored.all_zero ? 1 : 0;
  });
}

// One coarse_to_fine_propose per stream Rng(seed).split(1, i), i < n_props
// (smc_init's streams, inference.cpp:407-410): path (n_stages ints), leaf
// (object, face, noise), child contact (dx, dy, dtheta), log_q.
REFB_API int refb_propose(const RefIntr* k, const float* obs, const double* camera,
                          const RefSmcSpec* s, uint64_t seed, int n_props, int32_t* paths,
                          int32_t* leaf, double* contact, double* log_q) {
  return guarded([&] {
    auto w = make_world(k, obs, camera, s);
    const b3d::Stage0Table t = b3d::build_stage0(w->ctx, {});
    const int n_stages = 1 + s->n_refine;
    const b3d::Rng root(seed);
    for (int i = 0; i < n_props; ++i) {
      b3d::Rng stream = root.split(1, static_cast<uint64_t>(i));
      const b3d::Proposal p = b3d::coarse_to_fine_propose(w->ctx, {}, stream, &t);
      for (int j = 0; j < n_stages; ++j) paths[i * n_stages + j] = p.path[j];
      leaf[3 * i] = p.leaf.object_id;
      leaf[3 * i + 1] = p.leaf.face;
      leaf[3 * i + 2] = p.noise_index;
      contact[3 * i] = p.child.contact.dx;
      contact[3 * i + 1] = p.child.contact.dy;
      contact[3 * i + 2] = p.child.contact.dtheta;
      log_q[i] = p.log_q;
    }
  });
}

// run_smc with the world above (inference.cpp:493-520): per particle the
// children (object, face, dx, dy, dtheta), noise index, log_weight,
// log_target; plus log_evidence.
REFB_API int refb_run_smc(const RefIntr* k, const float* obs, const double* camera,
                          const RefSmcSpec* s, int n_objects, int n_particles, double threshold,
                          uint64_t seed, int32_t* child_ints, double* child_contact,
                          int32_t* noise_index, double* log_weight, double* log_target,
                          double* log_evidence) {
  return guarded([&] {
    auto w = make_world(k, obs, camera, s);
    const b3d::SmcResult r = b3d::run_smc(w->ctx, n_objects, n_particles, threshold, b3d::Rng(seed));
    for (size_t i = 0; i < r.particles.size(); ++i) {
      const b3d::Particle& p = r.particles[i];
      for (int c = 0; c < n_objects; ++c) {
        const b3d::SceneChild& ch = p.children[c];
        child_ints[(i * n_objects + c) * 2] = ch.object->id;
        child_ints[(i * n_objects + c) * 2 + 1] = ch.face;
        child_contact[(i * n_objects + c) * 3] = ch.contact.dx;
        child_contact[(i * n_objects + c) * 3 + 1] = ch.contact.dy;
        child_contact[(i * n_objects + c) * 3 + 2] = ch.contact.dtheta;
      }
      noise_index[i] = p.noise_index;
      log_weight[i] = p.log_weight;
      log_target[i] = p.log_target;
    }
    *log_evidence = r.log_evidence;
  });
}

// ---- camera tracking (tracking.cpp:59-172)
// Scene = table (w x h) + one object resting face 1 at the table centre, as
// generate_orbit_sequence builds it (tracking.cpp:174-193).  frames: n_frames
// images; initial camera pose; out: n_frames poses.
struct RefTrackSpec {
  double table_w, table_h;
  double sigma_max;
  int window;
  double p_outlier, sigma;
  double pos_extent, angle_extent;
  int points_per_dim, refine_stages;
  double refine_factor;
  int beam_width;
  int threads;
};

REFB_API int refb_track_camera(const RefIntr* k, const int32_t* vox, uint64_t n, double res,
                               const double* origin, const RefTrackSpec* s, int n_frames,
                               const float* frames, const double* initial, double* out_poses) {
  return guarded([&] {
    b3d::SceneGraph scene;
    scene.table = std::make_shared<b3d::ObjectModel>(b3d::ObjectModel::table(s->table_w, s->table_h));
    b3d::SceneChild child;
    child.object = std::make_shared<b3d::ObjectModel>(
        b3d::ObjectModel::from_grid(0, grid_in(vox, n, res, origin)));
    child.face = 1;
    const Eigen::Vector2d fp = b3d::footprint(*child.object, 1);
    child.contact.dx = (s->table_w - fp.x()) / 2;
    child.contact.dy = (s->table_h - fp.y()) / 2;
    child.contact.dtheta = 0;
    scene.children.push_back(child);
    b3d::ModelConfig model;
    model.intrinsics = intr(k);
    model.sigma_max = s->sigma_max;
    model.window = s->window;
    b3d::TrackSearch search;
    search.pos_extent = s->pos_extent;
    search.angle_extent = s->angle_extent;
    search.points_per_dim = s->points_per_dim;
    search.refine_stages = s->refine_stages;
    search.refine_factor = s->refine_factor;
    search.beam_width = s->beam_width;
    std::vector<b3d::DepthImage> fr;
    const size_t px = static_cast<size_t>(k->width) * k->height;
    for (int f = 0; f < n_frames; ++f) fr.push_back(image_in(frames + f * px, k->width, k->height));
    const b3d::TrackState st = b3d::track_camera(fr, scene, model, pose_in(initial), search,
                                                 {s->p_outlier, s->sigma}, s->threads);
    for (size_t f = 0; f < st.poses.size(); ++f) pose_out(st.poses[f], out_poses + 7 * f);
  });
}

// generate_orbit_sequence (tracking.cpp:174-206): frames + ground-truth poses.
REFB_API int refb_orbit_sequence(const RefIntr* k, const int32_t* vox, uint64_t n, double res,
                                 const double* origin, int n_frames, double distance,
                                 double altitude, double azimuth_start, double sweep,
                                 double table_w, double table_h, double p_outlier, double sigma,
                                 uint64_t seed, float* frames, double* poses) {
  return guarded([&] {
    b3d::ModelConfig model;
    model.intrinsics = intr(k);
    b3d::OrbitParams orbit;
    orbit.distance = distance;
    orbit.altitude = altitude;
    orbit.azimuth_start = azimuth_start;
    orbit.sweep = sweep;
    orbit.table_width = table_w;
    orbit.table_height = table_h;
    b3d::Rng rng(seed);
    const b3d::OrbitSequence seq = b3d::generate_orbit_sequence(
        std::make_shared<b3d::ObjectModel>(b3d::ObjectModel::from_grid(0, grid_in(vox, n, res, origin))),
        model, n_frames, orbit, {p_outlier, sigma}, rng);
    const size_t px = static_cast<size_t>(k->width) * k->height;
    for (int f = 0; f < n_frames; ++f) {
      std::memcpy(frames + f * px, seq.frames[f].depth.data(), px * sizeof(float));
      pose_out(seq.camera_poses[f], poses + 7 * f);
    }
  });
}
