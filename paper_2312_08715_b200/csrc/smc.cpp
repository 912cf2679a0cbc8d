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
//     smc_init, per distinct partial scene in smc_extend);
//   * refine stages: the children of every distinct current cell, batched
//     across particles that share (object, noise) and base scene into one
//     explicit-pose launch; particles on the same cell share its scores and
//     normalisation (see "Memoised evaluation" below);
//   * the final scene_target_logpdf of each particle, batched the same way.
// Scores carry the fp32-term likelihood (<= 1e-4 relative of the reference,
// DESIGN.md 5.1); everything else is the reference's arithmetic.
#include <algorithm>
#include <sched.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
// normalisation, draws from each particle's own stream) runs on the host
// threads this process may use, as the reference's parallel_for does
// (parallel.hpp:19-54); the result does not depend on the thread count.
// Workers persist across calls (a call costs a wake-up, not a spawn).
class Pool {
 public:
  static Pool& get() {
    // never destroyed: the workers block on a condition variable until the
    // process ends (no join at exit, none attempted in a forked child)
    static Pool* p = new Pool;
    return *p;
  }
  // a forked child has none of the workers: it runs serially
  size_t threads() const { return getpid() == pid_ ? workers_.size() + 1 : 1; }
  static bool& in_pool() {  // a parallel_for inside a job runs serially
    thread_local bool f = false;
    return f;
  }
  void run(size_t n, const std::function<void(size_t)>& f) {
    std::unique_lock<std::mutex> lk(run_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      n_ = n;
      next_ = 0;
      err_ = nullptr;
      busy_ = workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return busy_ == 0; });
    job_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }

 private:
  Pool() : pid_(getpid()) {
    size_t hw = std::max(1u, std::thread::hardware_concurrency());
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof set, &set) == 0) hw = std::max(1, CPU_COUNT(&set));
    for (size_t t = 1; t < std::min<size_t>(hw, 64); ++t)
      workers_.emplace_back([this] { loop(); }).detach();
  }
  void work() {
    in_pool() = true;
    try {
      for (size_t i; (i = next_.fetch_add(1)) < n_;) (*job_)(i);
    } catch (...) {
      std::lock_guard<std::mutex> g(mu_);
      if (!err_) err_ = std::current_exception();
      next_ = n_;
    }
    in_pool() = false;
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
      }
      work();
      std::lock_guard<std::mutex> g(mu_);
      if (--busy_ == 0) done_.notify_one();
    }
  }
  const pid_t pid_;
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t)>* job_ = nullptr;
  size_t n_ = 0, busy_ = 0;
  std::atomic<size_t> next_{0};
  std::exception_ptr err_;
  uint64_t gen_ = 0;
};

template <class F>
void parallel_for(size_t n, F&& f) {
  if (n < 64 || Pool::get().threads() == 1 || Pool::in_pool()) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  // chunks of >= 16 items per atomic claim
  const size_t chunk = std::max<size_t>(16, n / (8 * Pool::get().threads()));
  const size_t nc = (n + chunk - 1) / chunk;
  const std::function<void(size_t)> body = [&](size_t c) {
    const size_t e = std::min(n, (c + 1) * chunk);
    for (size_t i = c * chunk; i < e; ++i) f(i);
  };
  Pool::get().run(nc, body);
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
  uint64_t renders = 0;  // device render+score evaluations

  // footprint(obj, face) (scene_graph.cpp:91-95): x, y extents of the
  // face-down AABB; the stage-0 parent's upper ends are table - footprint.
  // Tabulated once per (object, face 1..6) by init().
  std::vector<double> fp_tab, prior_tab;
  void init() {
    fp_tab.assign((size_t)n_lib * 12, 0.0);
    prior_tab.assign((size_t)n_lib * 6, kNegInf);
    for (uint32_t o = 0; o < n_lib; ++o)
      for (int f = 1; f <= 6; ++f) {
        double lo[3], hi[3];
        rotated((int)o, f, lo, hi);
        const size_t j = o * 6 + (f - 1);
        fp_tab[2 * j] = hi[0] - lo[0];
        fp_tab[2 * j + 1] = hi[1] - lo[1];
        // child_prior's in-support value (the same expression, evaluated once)
        const double dx_range = cfg.table_w - fp_tab[2 * j],
                     dy_range = cfg.table_h - fp_tab[2 * j + 1];
        if (dx_range > 0 && dy_range > 0)
          prior_tab[j] = -std::log(static_cast<double>(n_lib)) - std::log(6.0) -
                         std::log(dx_range) - std::log(dy_range) - std::log(kTwoPi);
      }
  }
  void footprint(int obj, int face, double& fx, double& fy) const {
    if (face >= 1 && face <= 6 && (size_t)obj < n_lib) {
      fx = fp_tab[((size_t)obj * 6 + (face - 1)) * 2];
      fy = fp_tab[((size_t)obj * 6 + (face - 1)) * 2 + 1];
      return;
    }
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
    if (c.face >= 1 && c.face <= 6 && (size_t)c.object_id < n_lib)
      return prior_tab[(size_t)c.object_id * 6 + (c.face - 1)];
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
  bool base_valid = false;
  std::string base_key;  // partial_key of the context's current base scene
  void set_base(const std::vector<Child>& partial) {
    const std::string key = partial_key(partial);
    if (base_valid && key == base_key) return;  // already the context's base image
    std::vector<int32_t> ids{cfg.table_mesh};
    std::vector<b3d_pose> poses{b3d_pose{1, 0, 0, 0, 0, 0, 0}};
    for (const Child& c : partial) {
      ids.push_back(lib[c.object_id].mesh_id);
      poses.push_back(child_pose(c));
    }
    base_valid = false;
    ok(b3d_gpu_set_base_scene(g, ids.data(), poses.data(), (uint32_t)ids.size()));
    base_key = key;
    base_valid = true;
  }
  // an empty render: the windowed likelihood throws (likelihood.cpp:159-160)
  // and with it the whole inference; the untruncated one scores it -inf
  // (observation_loglik_cached, inference.cpp:52-54)
  void empty_render() const {
    if (cfg.window >= 0) throw Fail(B3D_ERROR, "windowed likelihood: empty rendered cloud");
  }
  void set_noise(const b3d_noise* nz, uint32_t n) {
    ok(b3d_gpu_set_likelihood(g, nz, n, cfg.sigma_max, cfg.window, cfg.prefactor));
  }

  // score_cells normalisation (inference.cpp:315-330)
  static void normalise_into(const double* lt, size_t n, std::vector<double>& s,
                             bool& all_zero) {
    if (s.size() < n) s.resize(n);
    double max_log = kNegInf;
    for (size_t i = 0; i < n; ++i) max_log = std::max(max_log, lt[i]);
    all_zero = !std::isfinite(max_log);
    if (all_zero) {
      std::fill(s.begin(), s.begin() + n, 1.0 / n);
      return;
    }
    // the exps in parallel, their total in index order (the same bits)
    parallel_for((n + 255) / 256, [&](size_t b) {
      const size_t e = std::min(n, (b + 1) * 256);
      for (size_t i = b * 256; i < e; ++i) s[i] = std::exp(lt[i] - max_log);
    });
    double total = 0;
    for (size_t i = 0; i < n; ++i) total += s[i];
    for (size_t i = 0; i < n; ++i) s[i] /= total;
  }
  static std::vector<double> normalise(const std::vector<double>& lt, bool& all_zero) {
    std::vector<double> s;
    normalise_into(lt.data(), lt.size(), s, all_zero);
    s.resize(lt.size());
    return s;
  }
  // sample_categorical (inference.cpp:345-353)
  // The same draw against a precomputed running sum: cdf[i] is the value of
  // the loop's `acc` after probs[i] (the same additions in the same order),
  // non-decreasing, so the loop's first i with u < acc is an upper_bound.
  static size_t sample_cdf(const double* cdf, size_t n, Rng& rng) {
    const double u = rng.uniform();
    const size_t i = std::upper_bound(cdf, cdf + n, u) - cdf;
    return i < n ? i : n - 1;
  }
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
  // The cells are implicit -- per (object, face) block its first index and
  // support, cell k decoded on demand -- and the score buffers persist
  // across calls (stage 0 of smc_extend runs once per distinct partial scene).
  struct Stage0 {
    struct Block {
      size_t first;
      int obj, face;
      double dx_range, dy_range;
    };
    std::vector<Block> blocks;
    size_t n = 0, nn = 1;
    b3d_schedule_stage s{};
    std::vector<double> lt, scores, cdf;
    bool all_zero = false;
    // stage0_cells (inference.cpp:208-238): order (object, face, ix, iy,
    // it, noise), the reference's interval arithmetic
    Cell cell(size_t k) const {
      size_t b = blocks.size() - 1;
      while (blocks[b].first > k) --b;
      const Block& bl = blocks[b];
      const size_t local = k - bl.first, ci = local / nn;
      const uint32_t it = (uint32_t)(ci % s.n_dtheta);
      const uint32_t iy = (uint32_t)((ci / s.n_dtheta) % s.n_dy);
      const uint32_t ix = (uint32_t)(ci / ((size_t)s.n_dtheta * s.n_dy));
      Cell c;
      c.object_id = bl.obj;
      c.face = bl.face;
      c.dx = {bl.dx_range * ix / s.n_dx, bl.dx_range * (ix + 1) / s.n_dx};
      c.dy = {bl.dy_range * iy / s.n_dy, bl.dy_range * (iy + 1) / s.n_dy};
      c.dtheta = {kTwoPi * it / s.n_dtheta, kTwoPi * (it + 1) / s.n_dtheta};
      c.noise_index = (int)(local % nn);
      return c;
    }
  };
  Stage0 s0_buf;
  std::vector<b3d_pose> s0_poses;
  std::vector<double> s0_lik;
  std::vector<uint8_t> s0_st;
  const Stage0& build_stage0(const std::vector<Child>& partial) {
    Stage0& t = s0_buf;
    const b3d_schedule_stage& s = cfg.stage0;
    t.s = s;
    t.blocks.clear();
    const double base_prior = prior_sum(partial);
    set_base(partial);
    set_noise(grid.data(), (uint32_t)grid.size());
    const size_t nn = grid.size();
    t.nn = nn;
    const size_t nc = (size_t)s.n_dx * s.n_dy * s.n_dtheta;
    size_t total = 0;
    for (uint32_t obj = 0; obj < n_lib; ++obj) {
      // one device launch per object: every face's cells, all noise entries
      const size_t first = total;
      size_t np = 0;
      for (int face = 1; face <= 6; ++face) {
        double fx, fy;
        footprint(obj, face, fx, fy);
        const double dx_range = cfg.table_w - fx, dy_range = cfg.table_h - fy;
        if (dx_range <= 0 || dy_range <= 0) continue;  // empty support branch
        t.blocks.push_back({total, (int)obj, face, dx_range, dy_range});
        total += nc * nn;
        // the stage-0 parent [0, table - footprint] x [0, 2 pi) subdivided:
        // the block's cells posed at their centres (the device contact
        // grid's poses)
        b3d_contact_cells cc{};
        cc.grid = contact(obj, face);
        cc.grid.count[0] = s.n_dx;
        cc.grid.count[1] = s.n_dy;
        cc.grid.count[2] = s.n_dtheta;
        cc.dx_hi = dx_range;
        cc.dy_hi = dy_range;
        cc.dtheta_hi = kTwoPi;
        if (s0_poses.size() < np + nc) s0_poses.resize(np + nc);
        ok(b3d_contact_cells_poses(&cc, s0_poses.data() + np));
        np += nc;
      }
      if (np == 0) continue;
      if (s0_lik.size() < np * nn) s0_lik.resize(np * nn);
      if (s0_st.size() < np) s0_st.resize(np);
      prof("s0 host");
      ok(b3d_gpu_score_poses(g, lib[obj].mesh_id, s0_poses.data(), np, s0_lik.data(),
                             s0_st.data()));
      prof("s0 device");
      renders += np;
      for (size_t j = 0; j < np; ++j)
        if (s0_st[j]) empty_render();
      if (t.lt.size() < total) t.lt.resize(total);
      parallel_for(np, [&](size_t j) {
        for (size_t e = 0; e < nn; ++e) {
          const size_t k = j * nn + e;
          const Cell c = t.cell(first + k);
          const Child cc{c.object_id, c.face, c.dx.center(), c.dy.center(), c.dtheta.center()};
          const double cp = child_prior(cc);
          const double l = s0_st[j] ? kNegInf : s0_lik[k];
          t.lt[first + k] = std::isfinite(base_prior) && std::isfinite(cp) && std::isfinite(l)
                                ? base_prior + cp + l
                                : kNegInf;
        }
      });
    }
    need(total > 0, B3D_ERROR_NUMERIC,
         "stage 0: empty proposal support (no object fits the table)");
    t.n = total;
    normalise_into(t.lt.data(), total, t.scores, t.all_zero);
    if (t.cdf.size() < total) t.cdf.resize(total);
    double acc = 0;  // sample_categorical's running sum (see sample_cdf)
    for (size_t i = 0; i < total; ++i) t.cdf[i] = acc += t.scores[i];
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
    renders += poses.size();
    ok(b3d_gpu_score_poses(g, lib[obj].mesh_id, poses.data(), poses.size(), s.data(),
                           st.data()));
    for (size_t i = 0; i < s.size(); ++i)
      if (st[i]) {
        empty_render();
        s[i] = kNegInf;
      }
    return s;
  }

  struct Prop {  // coarse_to_fine_propose state of one particle
    Cell current;
    double log_q = 0;
    Child child{};
  };

  // Memoised evaluation.  A stage's log targets are a pure function of the
  // base scene (the partial children), the object, the noise entry and the
  // cell, and so are its normalised scores: particles that share them (many
  // draw the same stage-0 cell; resampled particles are copies) share one
  // device launch slot and one normalisation, and only their draws -- each
  // from the particle's own stream -- stay per particle.  Identical values
  // to evaluating every particle separately (the kernel's score of a pose
  // does not depend on the rest of its batch).  Keys are the fields' bytes.
  template <class T>
  static void put(std::string& k, const T& v) {
    k.append(reinterpret_cast<const char*>(&v), sizeof v);
  }
  static std::string partial_key(const std::vector<Child>& cs) {
    std::string k;
    for (const Child& c : cs) {
      put(k, c.object_id);
      put(k, c.face);
      put(k, c.dx);
      put(k, c.dy);
      put(k, c.dtheta);
    }
    return k;
  }
  static std::string cell_key(const Cell& c) {
    std::string k;
    put(k, c.object_id);
    put(k, c.face);
    put(k, c.noise_index);
    for (const Interval* iv : {&c.dx, &c.dy, &c.dtheta}) {
      put(k, iv->lo);
      put(k, iv->hi);
    }
    return k;
  }
  // distinct values of key(i) for i in members, in first-member order:
  // returns the representatives and sets of[m] = representative slot of
  // members[m]
  template <class K>
  static std::vector<size_t> distinct(const std::vector<size_t>& members, K&& key,
                                      std::vector<size_t>& of) {
    std::map<std::string, size_t> idx;
    std::vector<size_t> rep;
    of.resize(members.size());
    for (size_t m = 0; m < members.size(); ++m) {
      const auto ins = idx.emplace(key(members[m]), rep.size());
      if (ins.second) rep.push_back(members[m]);
      of[m] = ins.first->second;
    }
    return rep;
  }
  // particles grouped by identical partial scene (= base image)
  static std::vector<std::vector<size_t>> by_partial(
      const std::vector<std::vector<Child>>& partial) {
    std::vector<size_t> all(partial.size()), of;
    for (size_t i = 0; i < all.size(); ++i) all[i] = i;
    const std::vector<size_t> rep =
        distinct(all, [&](size_t i) { return partial_key(partial[i]); }, of);
    std::vector<std::vector<size_t>> groups(rep.size());
    for (size_t i = 0; i < all.size(); ++i) groups[of[i]].push_back(i);
    return groups;
  }

  // coarse_to_fine_propose (inference.cpp:357-396) for a batch of particles
  // (stream[i], partial[i]); stage0 shared (smc_init) or per distinct partial
  // scene (smc_extend).
  std::vector<Prop> propose(std::vector<Rng>& stream,
                            const std::vector<std::vector<Child>>& partial,
                            const Stage0* shared) {
    const size_t P = stream.size();
    std::vector<Prop> props(P);
    auto pick0 = [&](size_t i, const Stage0* s0) {
      const size_t k = sample_cdf(s0->cdf.data(), s0->n, stream[i]);
      props[i].log_q = std::log(s0->scores[k]);
      props[i].current = s0->cell(k);
    };
    const std::vector<std::vector<size_t>> bases = by_partial(partial);
    if (shared) {
      parallel_for(P, [&](size_t i) { pick0(i, shared); });
    } else {
      for (const std::vector<size_t>& grp : bases) {  // a device stage 0 per partial scene
        const Stage0& local = build_stage0(partial[grp[0]]);
        parallel_for(grp.size(), [&](size_t m) { pick0(grp[m], &local); });
      }
    }
    for (uint32_t r = 0; r < cfg.n_refine; ++r) {
      const b3d_schedule_stage& st = cfg.refine[r];
      if ((size_t)st.n_dx * st.n_dy * st.n_dtheta == 1) {
        parallel_for(P, [&](size_t i) { props[i].current = subdivide(props[i].current, st)[0]; });
        continue;
      }
      for (const std::vector<size_t>& grp : bases) {
        // the group's distinct current cells: children, log targets and
        // normalised scores once each (score_cells with the particle's noise:
        // the cells inherit noise_index)
        std::vector<size_t> of;
        const std::vector<size_t> rep =
            distinct(grp, [&](size_t i) { return cell_key(props[i].current); }, of);
        const size_t U = rep.size();
        std::vector<std::vector<Cell>> cells(U);
        std::vector<std::vector<double>> sc(U);
        parallel_for(U, [&](size_t u) { cells[u] = subdivide(props[rep[u]].current, st); });
        const double base_prior = prior_sum(partial[grp[0]]);
        set_base(partial[grp[0]]);
        std::map<std::pair<int, int>, std::vector<size_t>> batches;  // (object, noise)
        for (size_t u = 0; u < U; ++u)
          batches[{props[rep[u]].current.object_id, props[rep[u]].current.noise_index}]
              .push_back(u);
        for (const auto& kv : batches) {
          const std::vector<size_t>& us = kv.second;
          std::vector<size_t> offs(us.size() + 1, 0);
          for (size_t m = 0; m < us.size(); ++m) offs[m + 1] = offs[m] + cells[us[m]].size();
          std::vector<b3d_pose> poses(offs.back());
          parallel_for(us.size(), [&](size_t m) {
            const Cell& cur = props[rep[us[m]]].current;
            b3d_contact_cells cc{};
            cc.grid = contact(cur.object_id, cur.face);
            cc.grid.count[0] = st.n_dx;
            cc.grid.count[1] = st.n_dy;
            cc.grid.count[2] = st.n_dtheta;
            cc.dx_lo = cur.dx.lo;
            cc.dx_hi = cur.dx.hi;
            cc.dy_lo = cur.dy.lo;
            cc.dy_hi = cur.dy.hi;
            cc.dtheta_lo = cur.dtheta.lo;
            cc.dtheta_hi = cur.dtheta.hi;
            ok(b3d_contact_cells_poses(&cc, poses.data() + offs[m]));
          });
          const std::vector<double> lik = score_poses(kv.first.first, kv.first.second, poses);
          parallel_for(us.size(), [&](size_t m) {
            const size_t u = us[m];
            std::vector<double> lt;
            lt.reserve(cells[u].size());
            size_t k = offs[m];
            for (const Cell& c : cells[u]) {
              const Child cc{c.object_id, c.face, c.dx.center(), c.dy.center(),
                             c.dtheta.center()};
              const double cp = child_prior(cc);
              const double l = lik[k++];
              lt.push_back(std::isfinite(base_prior) && std::isfinite(cp) && std::isfinite(l)
                               ? base_prior + cp + l
                               : kNegInf);
            }
            bool az;
            sc[u] = normalise(lt, az);
          });
        }
        parallel_for(grp.size(), [&](size_t m) {
          const size_t i = grp[m], u = of[m];
          const size_t pick = sample(sc[u], stream[i]);
          props[i].log_q += std::log(sc[u][pick]);
          props[i].current = cells[u][pick];
        });
      }
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
  // (partial + its new child) with its noise: per partial scene one launch
  // per (object, noise) over the distinct children
  std::vector<double> targets(const std::vector<std::vector<Child>>& partial,
                              const std::vector<Prop>& props) {
    const size_t P = props.size();
    std::vector<double> out(P, kNegInf);
    for (const std::vector<size_t>& grp : by_partial(partial)) {
      std::vector<size_t> of;
      const std::vector<size_t> rep = distinct(
          grp,
          [&](size_t i) {
            std::string k = partial_key({props[i].child});
            put(k, props[i].current.noise_index);
            return k;
          },
          of);
      set_base(partial[grp[0]]);
      std::map<std::pair<int, int>, std::vector<size_t>> batches;  // (object, noise)
      for (size_t u = 0; u < rep.size(); ++u)
        batches[{props[rep[u]].child.object_id, props[rep[u]].current.noise_index}].push_back(u);
      std::vector<double> lik(rep.size());
      for (const auto& kv : batches) {
        std::vector<b3d_pose> poses(kv.second.size());
        parallel_for(poses.size(),
                     [&](size_t m) { poses[m] = child_pose(props[rep[kv.second[m]]].child); });
        const std::vector<double> l = score_poses(kv.first.first, kv.first.second, poses);
        for (size_t m = 0; m < poses.size(); ++m) lik[kv.second[m]] = l[m];
      }
      parallel_for(grp.size(), [&](size_t m) {
        const size_t i = grp[m];
        std::vector<Child> all = partial[i];
        all.push_back(props[i].child);
        const double prior = prior_sum(all);
        const double l = lik[of[m]];
        out[i] = (std::isfinite(prior) && std::isfinite(l)) ? prior + l : kNegInf;
      });
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
  // B3D_SMC_PROFILE=1: wall time of each phase on stderr (diagnostics)
  std::chrono::steady_clock::time_point t_prev = std::chrono::steady_clock::now();
  const bool profiling = std::getenv("B3D_SMC_PROFILE") != nullptr;
  void prof(const char* what) {
    if (!profiling) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "smc %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_prev).count());
    t_prev = now;
  }

  std::vector<Particle> run(uint64_t seed, double& log_evidence) {
    const Rng rng(seed);
    const size_t P = cfg.n_particles;
    std::vector<Particle> ps(P);
    {  // smc_init (inference.cpp:398-420)
      prof("start");
      const Stage0& s0 = build_stage0({});
      prof("stage0");
      need(!s0.all_zero, B3D_ERROR_NUMERIC, "smc_init: all-zero scores at stage 0");
      std::vector<Rng> streams;
      for (size_t i = 0; i < P; ++i) streams.push_back(rng.split(1, i));
      const std::vector<std::vector<Child>> partial(P);
      const std::vector<Prop> props = propose(streams, partial, &s0);
      prof("propose");
      const std::vector<double> lt = targets(partial, props);
      prof("targets");
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
      const std::vector<double> lt = targets(partial, props);
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
    smc.init();
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
    if (cfg->renders) *cfg->renders = smc.renders;
    return B3D_OK;
  } catch (const Fail& f) {
    b3d200_set_last_error(f.what());
    return f.st;
  } catch (const std::exception& e) {
    b3d200_set_last_error(e.what());
    return B3D_ERROR;
  }
}
