// smc.cpp -- run_smc (inference.cpp:398-520) over the device scoring seams.
//
// The sequential Monte Carlo loop of the reference -- stage-0 cells over
// (object, face, dx, dy, dtheta, noise), coarse-to-fine refinement per
// particle, uniform leaf draws, scene_target_logpdf, systematic resampling --
// runs on the host exactly as the reference orders its Rng draws and fp64
// normalisations, while every render+score is a batched device call through
// this library's own C ABI:
//   * stage 0: one contact-cells launch per (object, face) with all noise
//     entries, over the particle's partial scene as the base image
//     (score_cells, inference.cpp:261-331; shared by all particles in
//     smc_init, per particle in smc_extend as the reference does);
//   * refine stages: the children of every particle's current cell, batched
//     across particles that share (object, noise) and base scene into one
//     explicit-pose launch (smc_init), else one launch per particle;
//   * the final scene_target_logpdf of each particle, batched the same way.
// Scores carry the fp32-term likelihood (<= 1e-4 relative of the reference,
// DESIGN.md 5.1); everything else is the reference's arithmetic.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <exception>
#include <mutex>
#include <thread>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "b3d_b200.h"

// b3d_capi.cpp: the library's thread-local error message
void b3d200_set_last_error(const char* msg);

namespace {

constexpr double kTwoPi = 6.283185307179586476925287;
constexpr double kNegInf = -std::numeric_limits<double>::infinity();

struct Fail : std::runtime_error {
  b3d_status st;
  Fail(b3d_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

void ok(b3d_status s) {
  if (s != B3D_OK) throw Fail(s, b3d_last_error());
}
void need(bool c, b3d_status s, const char* m) {
  if (!c) throw Fail(s, m);
}

// The per-particle host work (cell subdivision, child poses, priors,
// normalisation, draws from each particle's own stream) runs on all host
// threads, as the reference's parallel_for does (parallel.hpp:19-54); the
// result does not depend on the thread count.
template <class F>
void parallel_for(size_t n, F&& f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nth = std::min<size_t>(hw, (n + 31) / 32);
  if (nth <= 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::exception_ptr err;
  std::mutex mu;
  auto work = [&] {
    try {
      for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      if (!err) err = std::current_exception();
      next = n;
    }
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nth; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// rng.cpp: xoshiro256** seeded by splitmix64, split via mix()
struct Rng {
  uint64_t st[5];  // seed, s0..s3 (b3d_rng_seed layout)
  explicit Rng(uint64_t seed) { b3d_rng_seed(seed, st); }
  Rng split(uint64_t k0, uint64_t k1 = 0, uint64_t k2 = 0) const {
    Rng r(0);
    b3d_rng_split(st, k0, k1, k2, r.st);
    return r;
  }
  uint64_t next() {
    uint64_t* s = st + 1;
    auto rotl = [](uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

struct Interval {
  double lo, hi;
  double width() const { return hi - lo; }
  double center() const { return 0.5 * (lo + hi); }
};

struct Cell {  // inference.hpp:41-49
  int object_id = 0, face = 1;
  Interval dx{}, dy{}, dtheta{};
  int noise_index = -1;
  double volume() const { return dx.width() * dy.width() * dtheta.width(); }
};

struct Child {
  int object_id, face;
  double dx, dy, dtheta;
};

struct Particle {
  std::vector<Child> children;
  int noise_index = 0;
  double log_target = 0, log_weight = 0;
};

struct Smc {
  b3d_gpu_context* g;
  const b3d_smc_object* lib;
  uint32_t n_lib;
  const b3d_smc_config& cfg;
  std::vector<b3d_noise> grid;

  // footprint(obj, face) (scene_graph.cpp:91-95): x, y extents of the
  // face-down AABB; the stage-0 parent's upper ends are table - footprint
  void footprint(int obj, int face, double& fx, double& fy) const {
    double lo[3], hi[3];
    rotated(obj, face, lo, hi);
    fx = hi[0] - lo[0];
    fy = hi[1] - lo[1];
  }
  void rotated(int obj, int face, double lo[3], double hi[3]) const {
    ok(b3d_rotated_bounds(lib[obj].aabb_min, lib[obj].aabb_max, face, lo, hi));
  }
  b3d_contact_grid contact(int obj, int face) const {
    b3d_contact_grid cg{};
    cg.table_w = cfg.table_w;
    cg.table_h = cfg.table_h;
    for (int a = 0; a < 3; ++a) {
      cg.aabb_min[a] = lib[obj].aabb_min[a];
      cg.aabb_max[a] = lib[obj].aabb_max[a];
    }
    cg.face = face;
    return cg;
  }

  // child_prior_logpdf (inference.cpp:26-38)
  double child_prior(const Child& c) const {
    double fx, fy;
    footprint(c.object_id, c.face, fx, fy);
    const double dx_range = cfg.table_w - fx, dy_range = cfg.table_h - fy;
    if (dx_range <= 0 || dy_range <= 0) return kNegInf;
    if (c.dx < 0 || c.dx > dx_range || c.dy < 0 || c.dy > dy_range || c.dtheta < 0 ||
        c.dtheta >= kTwoPi)
      return kNegInf;
    return -std::log(static_cast<double>(n_lib)) - std::log(6.0) - std::log(dx_range) -
           std::log(dy_range) - std::log(kTwoPi);
  }
  // prior_sum (inference.cpp:85-94)
  double prior_sum(const std::vector<Child>& cs) const {
    double total = 0;
    for (const Child& c : cs) {
      const double lp = child_prior(c);
      if (!std::isfinite(lp)) return kNegInf;
      total += lp;
    }
    return total;
  }
  b3d_pose child_pose(const Child& c) const {
    b3d_pose p;
    ok(b3d_contact_to_pose(cfg.table_w, cfg.table_h, lib[c.object_id].aabb_min,
                           lib[c.object_id].aabb_max, c.face, c.dx, c.dy, c.dtheta, &p));
    return p;
  }
  // render_partial (inference.cpp:172-184) as the base image: table, then
  // the partial scene's children in order
  void set_base(const std::vector<Child>& partial) {
    std::vector<int32_t> ids{cfg.table_mesh};
    std::vector<b3d_pose> poses{b3d_pose{1, 0, 0, 0, 0, 0, 0}};
    for (const Child& c : partial) {
      ids.push_back(lib[c.object_id].mesh_id);
      poses.push_back(child_pose(c));
    }
    ok(b3d_gpu_set_base_scene(g, ids.data(), poses.data(), (uint32_t)ids.size()));
  }
  void set_noise(const b3d_noise* nz, uint32_t n) {
    ok(b3d_gpu_set_likelihood(g, nz, n, cfg.sigma_max, cfg.window, cfg.prefactor));
  }

  // score_cells normalisation (inference.cpp:315-330)
  static std::vector<double> normalise(const std::vector<double>& lt, bool& all_zero) {
    std::vector<double> s(lt.size(), 0.0);
    double max_log = kNegInf;
    for (double x : lt) max_log = std::max(max_log, x);
    all_zero = !std::isfinite(max_log);
    if (all_zero) {
      std::fill(s.begin(), s.end(), 1.0 / lt.size());
      return s;
    }
    double total = 0;
    for (size_t i = 0; i < lt.size(); ++i) {
      s[i] = std::exp(lt[i] - max_log);
      total += s[i];
    }
    for (double& x : s) x /= total;
    return s;
  }
  // sample_categorical (inference.cpp:345-353)
  static size_t sample(const std::vector<double>& probs, Rng& rng) {
    const double u = rng.uniform();
    double acc = 0;
    for (size_t i = 0; i < probs.size(); ++i) {
      acc += probs[i];
      if (u < acc) return i;
    }
    return probs.size() - 1;
  }

  // build_stage0 (inference.cpp:332-340) over `partial`: cells in the
  // reference's order (object, face, ix, iy, it, noise) and their scores
  struct Stage0 {
    std::vector<Cell> cells;
    std::vector<double> scores;
    bool all_zero = false;
  };
  Stage0 build_stage0(const std::vector<Child>& partial) {
    Stage0 t;
    const b3d_schedule_stage& s = cfg.stage0;
    const double base_prior = prior_sum(partial);
    set_base(partial);
    set_noise(grid.data(), (uint32_t)grid.size());
    const size_t nn = grid.size();
    std::vector<double> lt;
    for (uint32_t obj = 0; obj < n_lib; ++obj)
      for (int face = 1; face <= 6; ++face) {
        double fx, fy;
        footprint(obj, face, fx, fy);
        const double dx_range = cfg.table_w - fx, dy_range = cfg.table_h - fy;
        if (dx_range <= 0 || dy_range <= 0) continue;  // empty support branch
        const size_t first = t.cells.size();
        for (uint32_t ix = 0; ix < s.n_dx; ++ix)
          for (uint32_t iy = 0; iy < s.n_dy; ++iy)
            for (uint32_t it = 0; it < s.n_dtheta; ++it) {
              Cell c;
              c.object_id = (int)obj;
              c.face = face;
              c.dx = {dx_range * ix / s.n_dx, dx_range * (ix + 1) / s.n_dx};
              c.dy = {dy_range * iy / s.n_dy, dy_range * (iy + 1) / s.n_dy};
              c.dtheta = {kTwoPi * it / s.n_dtheta, kTwoPi * (it + 1) / s.n_dtheta};
              for (size_t e = 0; e < nn; ++e) {
                c.noise_index = (int)e;
                t.cells.push_back(c);
              }
            }
        // one device launch for the whole (object, face) group, all noise
        b3d_contact_grid cg = contact(obj, face);
        cg.count[0] = s.n_dx;
        cg.count[1] = s.n_dy;
        cg.count[2] = s.n_dtheta;
        const size_t nc = (size_t)s.n_dx * s.n_dy * s.n_dtheta;
        std::vector<double> lik(nc * nn);
        std::vector<uint8_t> st(nc);
        ok(b3d_gpu_score_contact_grid(g, lib[obj].mesh_id, &cg, lik.data(), st.data()));
        for (size_t k = 0; k < nc * nn; ++k) {
          const Cell& c = t.cells[first + k];
          const Child cc{c.object_id, c.face, c.dx.center(), c.dy.center(), c.dtheta.center()};
          const double cp = child_prior(cc);
          const double l = st[k / nn] ? kNegInf : lik[k];
          lt.push_back(std::isfinite(base_prior) && std::isfinite(cp) && std::isfinite(l)
                           ? base_prior + cp + l
                           : kNegInf);
        }
      }
    need(!t.cells.empty(), B3D_ERROR_NUMERIC,
         "stage 0: empty proposal support (no object fits the table)");
    t.scores = normalise(lt, t.all_zero);
    return t;
  }

  // subdivide_cell (inference.cpp:240-259)
  static std::vector<Cell> subdivide(const Cell& cell, const b3d_schedule_stage& st) {
    std::vector<Cell> out;
    for (uint32_t ix = 0; ix < st.n_dx; ++ix)
      for (uint32_t iy = 0; iy < st.n_dy; ++iy)
        for (uint32_t it = 0; it < st.n_dtheta; ++it) {
          Cell c = cell;
          c.dx = {cell.dx.lo + cell.dx.width() * ix / st.n_dx,
                  cell.dx.lo + cell.dx.width() * (ix + 1) / st.n_dx};
          c.dy = {cell.dy.lo + cell.dy.width() * iy / st.n_dy,
                  cell.dy.lo + cell.dy.width() * (iy + 1) / st.n_dy};
          c.dtheta = {cell.dtheta.lo + cell.dtheta.width() * it / st.n_dtheta,
                      cell.dtheta.lo + cell.dtheta.width() * (it + 1) / st.n_dtheta};
          out.push_back(c);
        }
    return out;
  }

  // Scores of explicit hypotheses (object mesh, noise entry) over the current
  // base scene: one device launch.
  std::vector<double> score_poses(int obj, int noise_index, const std::vector<b3d_pose>& poses) {
    set_noise(&grid[noise_index], 1);
    std::vector<double> s(poses.size());
    std::vector<uint8_t> st(poses.size());
    ok(b3d_gpu_score_poses(g, lib[obj].mesh_id, poses.data(), poses.size(), s.data(),
                           st.data()));
    for (size_t i = 0; i < s.size(); ++i)
      if (st[i]) s[i] = kNegInf;
    return s;
  }

  struct Prop {  // coarse_to_fine_propose state of one particle
    Cell current;
    double log_q = 0;
    Child child{};
  };

  // coarse_to_fine_propose (inference.cpp:357-396) for a batch of particles
  // (stream[i], partial[i]); stage0 shared (smc_init) or per particle.
  std::vector<Prop> propose(std::vector<Rng>& stream,
                            const std::vector<std::vector<Child>>& partial,
                            const Stage0* shared) {
    const size_t P = stream.size();
    std::vector<Prop> props(P);
    auto pick0 = [&](size_t i, const Stage0* s0) {
      const size_t k = sample(s0->scores, stream[i]);
      props[i].log_q = std::log(s0->scores[k]);
      props[i].current = s0->cells[k];
    };
    if (shared) {
      parallel_for(P, [&](size_t i) { pick0(i, shared); });
    } else {
      for (size_t i = 0; i < P; ++i) {  // a device stage 0 per particle
        const Stage0 local = build_stage0(partial[i]);
        pick0(i, &local);
      }
    }
    for (uint32_t r = 0; r < cfg.n_refine; ++r) {
      const b3d_schedule_stage& st = cfg.refine[r];
      std::vector<std::vector<Cell>> cells(P);
      parallel_for(P, [&](size_t i) { cells[i] = subdivide(props[i].current, st); });
      if (cells[0].size() == 1) {
        for (size_t i = 0; i < P; ++i) props[i].current = cells[i][0];
        continue;
      }
      // log targets of every particle's children (score_cells with the
      // particle's noise: the cells inherit noise_index)
      std::vector<std::vector<double>> lt(P);
      auto fill = [&](const std::vector<size_t>& members) {
        std::vector<size_t> offs(members.size() + 1, 0);
        for (size_t m = 0; m < members.size(); ++m)
          offs[m + 1] = offs[m] + cells[members[m]].size();
        std::vector<b3d_pose> poses(offs.back());
        parallel_for(members.size(), [&](size_t m) {
          const size_t i = members[m];
          b3d_contact_cells cc{};
          cc.grid = contact(props[i].current.object_id, props[i].current.face);
          cc.grid.count[0] = st.n_dx;
          cc.grid.count[1] = st.n_dy;
          cc.grid.count[2] = st.n_dtheta;
          const Cell& cur = props[i].current;
          cc.dx_lo = cur.dx.lo;
          cc.dx_hi = cur.dx.hi;
          cc.dy_lo = cur.dy.lo;
          cc.dy_hi = cur.dy.hi;
          cc.dtheta_lo = cur.dtheta.lo;
          cc.dtheta_hi = cur.dtheta.hi;
          ok(b3d_contact_cells_poses(&cc, poses.data() + offs[m]));
        });
        const Cell& lead = props[members[0]].current;
        const std::vector<double> lik = score_poses(lead.object_id, lead.noise_index, poses);
        parallel_for(members.size(), [&](size_t m) {
          const size_t i = members[m];
          const double base_prior = prior_sum(partial[i]);
          size_t k = offs[m];
          lt[i].reserve(cells[i].size());
          for (const Cell& c : cells[i]) {
            const Child cc{c.object_id, c.face, c.dx.center(), c.dy.center(), c.dtheta.center()};
            const double cp = child_prior(cc);
            const double l = lik[k++];
            lt[i].push_back(std::isfinite(base_prior) && std::isfinite(cp) && std::isfinite(l)
                                ? base_prior + cp + l
                                : kNegInf);
          }
        });
      };
      if (shared) {  // one base scene: batch by (object, noise entry)
        set_base(partial[0]);
        std::map<std::pair<int, int>, std::vector<size_t>> groups;
        for (size_t i = 0; i < P; ++i)
          groups[{props[i].current.object_id, props[i].current.noise_index}].push_back(i);
        for (const auto& kv : groups) fill(kv.second);
      } else {
        for (size_t i = 0; i < P; ++i) {
          set_base(partial[i]);
          fill({i});
        }
      }
      parallel_for(P, [&](size_t i) {
        bool az;
        const std::vector<double> sc = normalise(lt[i], az);
        const size_t pick = sample(sc, stream[i]);
        props[i].log_q += std::log(sc[pick]);
        props[i].current = cells[i][pick];
      });
    }
    for (size_t i = 0; i < P; ++i) {
      Prop& pr = props[i];
      const Cell& c = pr.current;
      pr.child.object_id = c.object_id;
      pr.child.face = c.face;
      pr.child.dx = stream[i].uniform(c.dx.lo, c.dx.hi);
      pr.child.dy = stream[i].uniform(c.dy.lo, c.dy.hi);
      pr.child.dtheta = stream[i].uniform(c.dtheta.lo, c.dtheta.hi);
      pr.log_q += -std::log(c.volume());
    }
    return props;
  }

  // scene_target_logpdf (inference.cpp:186-196) of each particle's scene
  // (partial + its new child) with its noise; same batching as propose
  std::vector<double> targets(const std::vector<std::vector<Child>>& partial,
                              const std::vector<Prop>& props, bool shared_base) {
    const size_t P = props.size();
    std::vector<double> out(P, kNegInf);
    auto fill = [&](const std::vector<size_t>& members) {
      std::vector<b3d_pose> poses(members.size());
      parallel_for(members.size(), [&](size_t m) { poses[m] = child_pose(props[members[m]].child); });
      const std::vector<double> lik =
          score_poses(props[members[0]].child.object_id, props[members[0]].current.noise_index,
                      poses);
      for (size_t k = 0; k < members.size(); ++k) {
        const size_t i = members[k];
        std::vector<Child> all = partial[i];
        all.push_back(props[i].child);
        const double prior = prior_sum(all);
        out[i] = (std::isfinite(prior) && std::isfinite(lik[k])) ? prior + lik[k] : kNegInf;
      }
    };
    if (shared_base) {
      set_base(partial[0]);
      std::map<std::pair<int, int>, std::vector<size_t>> groups;
      for (size_t i = 0; i < P; ++i)
        groups[{props[i].child.object_id, props[i].current.noise_index}].push_back(i);
      for (const auto& kv : groups) fill(kv.second);
    } else {
      for (size_t i = 0; i < P; ++i) {
        set_base(partial[i]);
        fill({i});
      }
    }
    return out;
  }

  static double logsumexp(const std::vector<double>& xs) {  // inference.cpp:16-23
    double m = kNegInf;
    for (double x : xs) m = std::max(m, x);
    if (!std::isfinite(m)) return kNegInf;
    double acc = 0;
    for (double x : xs) acc += std::exp(x - m);
    return m + std::log(acc);
  }
  static std::vector<double> weights(const std::vector<Particle>& ps) {  // 443-455
    std::vector<double> lw;
    for (const Particle& p : ps) lw.push_back(p.log_weight);
    const double lse = logsumexp(lw);
    need(std::isfinite(lse), B3D_ERROR_NUMERIC, "particle weights are all zero");
    std::vector<double> w(ps.size());
    for (size_t i = 0; i < ps.size(); ++i) w[i] = std::exp(lw[i] - lse);
    return w;
  }
  static double ess(const std::vector<Particle>& ps) {  // 457-463
    double sum_sq = 0;
    for (double wi : weights(ps)) sum_sq += wi * wi;
    return 1.0 / sum_sq;
  }
  static std::vector<Particle> resample(const std::vector<Particle>& ps, Rng& rng) {  // 465-491
    const std::vector<double> w = weights(ps);
    std::vector<double> lw;
    for (const Particle& p : ps) lw.push_back(p.log_weight);
    const double log_total = logsumexp(lw);
    const size_t n = ps.size();
    const double u = rng.uniform();
    std::vector<Particle> out;
    double cumulative = 0;
    size_t src = 0;
    for (size_t i = 0; i < n; ++i) {
      const double position = (static_cast<double>(i) + u) / static_cast<double>(n);
      while (src + 1 < n && cumulative + w[src] <= position) {
        cumulative += w[src];
        ++src;
      }
      out.push_back(ps[src]);
    }
    const double reset = log_total - std::log(static_cast<double>(n));
    for (Particle& p : out) p.log_weight = reset;
    return out;
  }

  // run_smc (inference.cpp:493-520)
  std::vector<Particle> run(uint64_t seed, double& log_evidence) {
    const Rng rng(seed);
    const size_t P = cfg.n_particles;
    std::vector<Particle> ps(P);
    {  // smc_init (inference.cpp:398-420)
      const Stage0 s0 = build_stage0({});
      need(!s0.all_zero, B3D_ERROR_NUMERIC, "smc_init: all-zero scores at stage 0");
      std::vector<Rng> streams;
      for (size_t i = 0; i < P; ++i) streams.push_back(rng.split(1, i));
      const std::vector<std::vector<Child>> partial(P);
      const std::vector<Prop> props = propose(streams, partial, &s0);
      const std::vector<double> lt = targets(partial, props, true);
      for (size_t i = 0; i < P; ++i) {
        ps[i].children = {props[i].child};
        ps[i].noise_index = props[i].current.noise_index;
        ps[i].log_target = lt[i];
        ps[i].log_weight = lt[i] - props[i].log_q;
      }
    }
    const Rng resample_stream = rng.split(0x5e5a, 0);
    auto maybe_resample = [&](int stage) {
      if (ess(ps) < cfg.resample_threshold * P) {
        Rng stage_stream = resample_stream.split(static_cast<uint64_t>(stage));
        ps = resample(ps, stage_stream);
      }
    };
    maybe_resample(1);
    for (uint32_t k = 2; k <= cfg.n_objects; ++k) {  // smc_extend (inference.cpp:422-441)
      const uint64_t stage_key = ps.front().children.size() + 1;
      std::vector<Rng> streams;
      std::vector<std::vector<Child>> partial;
      for (size_t i = 0; i < P; ++i) {
        streams.push_back(rng.split(stage_key, i));
        partial.push_back(ps[i].children);
      }
      const std::vector<Prop> props = propose(streams, partial, nullptr);
      const std::vector<double> lt = targets(partial, props, false);
      for (size_t i = 0; i < P; ++i) {
        const double prev = ps[i].log_target;
        ps[i].children.push_back(props[i].child);
        ps[i].noise_index = props[i].current.noise_index;
        ps[i].log_target = lt[i];
        ps[i].log_weight += lt[i] - prev - props[i].log_q;
      }
      maybe_resample((int)k);
    }
    std::vector<double> lw;
    for (const Particle& p : ps) lw.push_back(p.log_weight);
    log_evidence = logsumexp(lw) - std::log(static_cast<double>(P));
    return ps;
  }
};

}  // namespace

extern "C" b3d_status b3d_gpu_run_smc(b3d_gpu_context* ctx, const b3d_smc_object* library,
                                      uint32_t n_library, const b3d_smc_config* cfg,
                                      uint64_t seed, b3d_smc_particle* particles,
                                      double* log_evidence) {
  try {
    need(ctx && library && cfg && particles && log_evidence, B3D_ERROR, "bad arguments");
    need(n_library >= 1, B3D_ERROR, "inference: empty library");
    need(cfg->n_noise_grid >= 1 && cfg->noise_grid, B3D_ERROR, "inference: empty noise grid");
    need(cfg->n_objects >= 1, B3D_ERROR, "run_smc: n_objects must be >= 1");
    need(cfg->n_particles >= 1, B3D_ERROR, "smc_init: need at least one particle");
    for (uint32_t i = 0; i < cfg->n_particles; ++i)
      need(particles[i].children != nullptr, B3D_ERROR, "bad arguments");
    need(cfg->n_refine == 0 || cfg->refine, B3D_ERROR, "bad arguments");
    auto valid = [](const b3d_schedule_stage& s) {
      return s.n_dx >= 1 && s.n_dy >= 1 && s.n_dtheta >= 1;
    };
    need(valid(cfg->stage0), B3D_ERROR, "schedule stage: subdivision counts must be >= 1");
    for (uint32_t r = 0; r < cfg->n_refine; ++r)
      need(valid(cfg->refine[r]), B3D_ERROR, "schedule stage: subdivision counts must be >= 1");
    for (uint32_t e = 0; e < cfg->n_noise_grid; ++e) {
      const b3d_noise& np = cfg->noise_grid[e];
      need(np.p_outlier >= 0 && np.p_outlier <= 1 && np.sigma_noise > 0 &&
               np.sigma_noise <= cfg->sigma_max,
           B3D_ERROR, "noise grid entry outside support");
    }
    Smc smc{ctx, library, n_library, *cfg, {}};
    smc.grid.assign(cfg->noise_grid, cfg->noise_grid + cfg->n_noise_grid);
    double le = 0;
    const std::vector<Particle> ps = smc.run(seed, le);
    for (size_t i = 0; i < ps.size(); ++i) {
      b3d_smc_particle& o = particles[i];
      o.n_children = (int32_t)ps[i].children.size();
      for (size_t c = 0; c < ps[i].children.size(); ++c) {
        const Child& ch = ps[i].children[c];
        o.children[c] = b3d_smc_child{ch.object_id, ch.face, ch.dx, ch.dy, ch.dtheta};
      }
      o.noise_index = ps[i].noise_index;
      o.log_target = ps[i].log_target;
      o.log_weight = ps[i].log_weight;
    }
    *log_evidence = le;
    return B3D_OK;
  } catch (const Fail& f) {
    b3d200_set_last_error(f.what());
    return f.st;
  } catch (const std::exception& e) {
    b3d200_set_last_error(e.what());
    return B3D_ERROR;
  }
}
