// capi_handles.cpp -- the reference's handle-based C API (b3d.h: object
// models, libraries, scenes, b3d_render, b3d_infer and the particle
// accessors, SDPT / SVOX files) on top of this library's batched GPU entry
// points.  Same signatures, status codes, thread-local error messages and
// JSON schemas as proj/src/capi/b3d_capi.cpp:124-456; every render and score
// runs on the device through a per-thread GPU context (device
// $B3D_DEVICE, default 0).
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <tuple>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "b3d_b200.h"
#include "json_mini.hpp"

void b3d200_set_last_error(const char* msg);  // b3d_capi.cpp
b3d_depth_image* b3d200_depth_image_new(uint32_t width, uint32_t height,
                                        std::vector<float>&& depth);
void b3d200_validate_intrinsics(const b3d_intrinsics& k);
void b3d200_render_scene_keys(b3d_gpu_context* ctx, const b3d_intrinsics* k,
                              const b3d_pose* camera, const int32_t* ids, const b3d_pose* poses,
                              uint32_t n, float* out);

namespace {

namespace J = b3d200::json;

struct Fail : std::runtime_error {
  b3d_status st;
  Fail(b3d_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};
void require(bool c, b3d_status s, const std::string& m) {
  if (!c) throw Fail(s, m);
}
void check(bool c, const char* m) { require(c, B3D_ERROR, m); }
void ok(b3d_status s) {
  if (s != B3D_OK) throw Fail(s, b3d_last_error());
}

template <typename F>
b3d_status guarded(F&& fn) {
  try {
    fn();
    return B3D_OK;
  } catch (const Fail& f) {
    b3d200_set_last_error(f.what());
    return f.st;
  } catch (const std::exception& e) {
    b3d200_set_last_error(e.what());
    return B3D_ERROR;
  }
}

uint64_t next_serial() {
  static std::atomic<uint64_t> s{1};
  return s++;
}

}  // namespace

// ObjectModel (scene_graph.hpp:15-27): voxel grid, mesh, model-frame AABB.
struct b3d_object_model {
  int id = 0;
  uint64_t serial = 0;
  double resolution = 0, origin[3] = {0, 0, 0};
  std::vector<int32_t> voxels;  // stored order (defines triangle order)
  std::vector<double> verts;
  std::vector<uint32_t> tris;
  double aabb_min[3], aabb_max[3];
};
struct b3d_library {
  std::vector<std::shared_ptr<const b3d_object_model>> models;
};
struct b3d_scene {
  double table_w = 0, table_h = 0, thickness = 0.01;
  struct Child {
    std::shared_ptr<const b3d_object_model> obj;
    int face;
    double dx, dy, dtheta;
  };
  std::vector<Child> children;
};
struct b3d_particles {
  std::vector<b3d_smc_particle> ps;
  std::vector<b3d_smc_child> kids;  // ps[i].children = kids + i * n_objects
  double log_evidence = 0;
  double table_w = 0, table_h = 0;
  std::vector<std::shared_ptr<const b3d_object_model>> lib;
  std::vector<b3d_noise> grid;
};

namespace {

std::shared_ptr<b3d_object_model> model_from_grid(int id, double res, const double origin[3],
                                                  std::vector<int32_t> vox) {
  // ObjectModel::from_grid (scene_graph.cpp:16-24): voxel_to_mesh + mesh_bounds
  require(!vox.empty(), B3D_ERROR, "object model: empty grid");
  auto m = std::make_shared<b3d_object_model>();
  m->id = id;
  m->serial = next_serial();
  m->resolution = res;
  for (int a = 0; a < 3; ++a) m->origin[a] = origin[a];
  const uint64_t n = vox.size() / 3;
  m->verts.resize(24 * n);
  m->tris.resize(36 * n);
  uint64_t nv = 0, nt = 0;
  ok(b3d_voxel_to_mesh(vox.data(), n, res, origin, m->verts.data(), m->tris.data(), &nv, &nt));
  m->verts.resize(3 * nv);
  m->tris.resize(3 * nt);
  m->voxels = std::move(vox);
  for (int a = 0; a < 3; ++a) m->aabb_min[a] = m->aabb_max[a] = m->verts[a];
  for (uint64_t i = 0; i < nv; ++i)
    for (int a = 0; a < 3; ++a) {
      m->aabb_min[a] = std::min(m->aabb_min[a], m->verts[3 * i + a]);
      m->aabb_max[a] = std::max(m->aabb_max[a], m->verts[3 * i + a]);
    }
  return m;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  require(in.good(), B3D_ERROR_IO, "cannot open: " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  require(in.good() || in.eof(), B3D_ERROR_IO, "read failed: " + path);
  return buf.str();
}

void write_file_atomic(const std::string& path, const std::string& contents) {  // io.cpp:61-80
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    require(out.good(), B3D_ERROR_IO, "cannot open for writing: " + tmp);
    out.write(contents.data(), static_cast<std::streamsize>(contents.size()));
    out.flush();
    if (!out.good()) {
      out.close();
      std::remove(tmp.c_str());
      throw Fail(B3D_ERROR_IO, "write failed: " + tmp);
    }
  }
  require(std::rename(tmp.c_str(), path.c_str()) == 0, B3D_ERROR_IO,
          "rename failed: " + tmp + " -> " + path);
}

struct ByteReader {  // io.cpp:29-57
  const std::string& d;
  std::string path;
  size_t pos = 0;
  template <typename T>
  T read() {
    require(pos + sizeof(T) <= d.size(), B3D_ERROR_IO, path + ": truncated file");
    T v;
    std::memcpy(&v, d.data() + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  void magic(const char* m) {
    require(pos + 4 <= d.size(), B3D_ERROR_IO, path + ": truncated file");
    require(std::memcmp(d.data() + pos, m, 4) == 0, B3D_ERROR_IO, path + ": bad magic bytes");
    pos += 4;
  }
};
template <typename T>
void put(std::string& out, T v) {
  out.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

std::shared_ptr<b3d_object_model> load_svox(const std::string& path, int id) {  // io.cpp:132-147
  const std::string data = read_file(path);
  ByteReader r{data, path};
  r.magic("SVOX");
  const double res = r.read<float>();
  double origin[3];
  for (double& o : origin) o = r.read<float>();
  const uint32_t count = r.read<uint32_t>();
  require(data.size() == 24 + (size_t)count * 12, B3D_ERROR_IO, path + ": size mismatch");
  std::vector<int32_t> vox(3 * (size_t)count);
  for (auto& v : vox) v = r.read<int32_t>();
  require(res > 0, B3D_ERROR_IO, path + ": non-positive resolution");
  return model_from_grid(id, res, origin, std::move(vox));
}

// nlohmann's number -> int / uint32_t conversions as the reference's build
// performs them (static_cast under gcc on x86-64): integers wrap modulo
// 2^32; a float truncates toward zero, out of range giving INT_MIN (int,
// cvttsd2si) or 0 (uint32_t, through the 64-bit conversion).
int json_int(const J::Value& x) {
  if (x.kind == J::Value::Bool) return x.b ? 1 : 0;  // nlohmann converts booleans too
  if (x.int_kind == 1) return (int)(uint32_t)(uint64_t)x.i;
  if (x.int_kind == 2) return (int)(uint32_t)x.u;
  return (x.num > -2147483649.0 && x.num < 2147483648.0) ? (int)x.num : INT_MIN;
}
uint32_t json_u32(const J::Value& x) {
  if (x.kind == J::Value::Bool) return x.b ? 1u : 0u;
  if (x.int_kind == 1) return (uint32_t)(uint64_t)x.i;
  if (x.int_kind == 2) return (uint32_t)x.u;
  return (x.num > -9223372036854775809.0 && x.num < 9223372036854775808.0)
             ? (uint32_t)(uint64_t)(int64_t)x.num
             : 0u;
}

// the JSON kinds nlohmann's get<int> / get<uint32_t> accept (its generic
// arithmetic from_json converts booleans too); get<double> goes through
// get_arithmetic_value, numbers only
bool is_arith(const J::Value& x) { return x.kind == J::Value::Number || x.kind == J::Value::Bool; }

// ConfigReader (config.cpp): strict object view, unknown keys are errors
struct Reader {
  const J::Value& v;
  std::string ctx;
  std::set<std::string> seen;
  Reader(const J::Value& j, std::string c) : v(j), ctx(std::move(c)) {
    require(j.is_object(), B3D_ERROR_CONFIG, ctx + ": expected a JSON object");
  }
  bool has(const std::string& k) const { return v.find(k) != nullptr; }
  const J::Value& raw(const std::string& k) {
    seen.insert(k);
    const J::Value* x = v.find(k);
    require(x != nullptr, B3D_ERROR_CONFIG, ctx + ": missing required key '" + k + "'");
    return *x;
  }
  double num(const std::string& k) {  // get<double>: numbers only
    const J::Value& x = raw(k);
    require(x.kind == J::Value::Number, B3D_ERROR_CONFIG,
            ctx + ": key '" + k + "' has the wrong type");
    return x.num;
  }
  double num_or(const std::string& k, double d) { return has(k) ? num(k) : (seen.insert(k), d); }
  // get<int> / get<uint32_t> (config.hpp:21-27, 50-56): any JSON number
  // converts (json_int / json_u32), anything else is the wrong type
  int integer(const std::string& k) {
    const J::Value& x = raw(k);
    require(is_arith(x), B3D_ERROR_CONFIG, ctx + ": key '" + k + "' has the wrong type");
    return json_int(x);
  }
  uint32_t u32(const std::string& k) {
    const J::Value& x = raw(k);
    require(is_arith(x), B3D_ERROR_CONFIG, ctx + ": key '" + k + "' has the wrong type");
    return json_u32(x);
  }
  int int_or(const std::string& k, int d) { return has(k) ? integer(k) : (seen.insert(k), d); }
  Reader object(const std::string& k) { return Reader(raw(k), ctx + "." + k); }
  void finish() const {
    for (const auto& kv : v.obj)
      require(seen.count(kv.first) > 0, B3D_ERROR_CONFIG,
              ctx + ": unknown key '" + kv.first + "'");
  }
};

J::Value parse_or(const char* text, b3d_status st, const char* msg) {
  try {
    return J::parse(text);
  } catch (const std::exception&) {
    throw Fail(st, msg);
  }
}

// from_c(b3d_pose) (b3d_capi.cpp:66-74): unit-norm check, then normalize
b3d_pose normalized_pose(const b3d_pose& p) {
  const double n2 = (p.qx * p.qx + p.qy * p.qy) + (p.qz * p.qz + p.qw * p.qw);
  require(std::abs(std::sqrt(n2) - 1.0) < 1e-6, B3D_ERROR,
          "pose rotation must be a unit quaternion");
  b3d_pose o = p;
  const double n = std::sqrt(n2);
  if (n2 > 0) {
    o.qw /= n;
    o.qx /= n;
    o.qy /= n;
    o.qz /= n;
  }
  return o;
}

// per-thread GPU context and the meshes uploaded to it (keyed by model
// serial, or table extents)
struct Gpu {
  b3d_gpu_context* ctx = nullptr;
  std::map<uint64_t, int32_t> meshes;
  std::map<std::tuple<double, double, double>, int32_t> tables;
  // what the context holds now (b3d_render reuses it call after call); any
  // other setter of the camera clears cam_key
  std::string cam_key, scene_key;
  ~Gpu() {
    if (ctx) b3d_gpu_context_destroy(ctx);
  }
  b3d_gpu_context* get() {
    if (!ctx) {
      const char* d = std::getenv("B3D_DEVICE");
      ok(b3d_gpu_context_create(d ? std::atoi(d) : 0, &ctx));
    }
    return ctx;
  }
  int32_t mesh(const b3d_object_model& m) {
    auto it = meshes.find(m.serial);
    if (it != meshes.end()) return it->second;
    int32_t id = -1;
    ok(b3d_gpu_upload_mesh(get(), m.verts.data(), m.verts.size() / 3, m.tris.data(),
                           m.tris.size() / 3, &id));
    return meshes[m.serial] = id;
  }
  template <class T>
  static std::string bytes(const T* p, size_t n) {
    return std::string(reinterpret_cast<const char*>(p), sizeof(T) * n);
  }
  void camera(const b3d_intrinsics* k) {  // intrinsics only (camera-mode renders)
    const std::string key = bytes(k, 1);
    if (key == cam_key) return;
    cam_key.clear();
    ok(b3d_gpu_set_camera(get(), k, nullptr));
    cam_key = key;
  }
  void camera_scene(const std::vector<int32_t>& ids, const std::vector<b3d_pose>& poses) {
    const std::string key = bytes(ids.data(), ids.size()) + bytes(poses.data(), poses.size());
    if (key == scene_key) return;
    scene_key.clear();
    ok(b3d_gpu_set_camera_scene(get(), ids.data(), poses.data(), (uint32_t)ids.size()));
    scene_key = key;
  }
  int32_t table(double w, double h, double thickness) {  // ObjectModel::table
    const auto key = std::make_tuple(w, h, thickness);
    auto it = tables.find(key);
    if (it != tables.end()) return it->second;
    const double lo[3] = {-w / 2, -h / 2, -thickness}, hi[3] = {w / 2, h / 2, 0.0};
    double v[24];
    uint32_t t[36];
    ok(b3d_box_mesh(lo, hi, v, t));
    int32_t id = -1;
    ok(b3d_gpu_upload_mesh(get(), v, 8, t, 12, &id));
    return tables[key] = id;
  }
};
thread_local Gpu g_gpu;

char* owned(const std::string& s) {
  char* out = new char[s.size() + 1];
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

}  // namespace

extern "C" {

b3d_status b3d_depth_image_load(const char* path, b3d_depth_image** out) {
  return guarded([&] {  // io.cpp:104-116
    check(path && out, "bad arguments");
    const std::string data = read_file(path);
    ByteReader r{data, path};
    r.magic("SDPT");
    const uint32_t w = r.read<uint32_t>(), h = r.read<uint32_t>();
    const size_t count = (size_t)w * h;
    require(data.size() == 12 + count * 4, B3D_ERROR_IO, std::string(path) + ": size mismatch");
    std::vector<float> d(count);
    for (float& z : d) z = r.read<float>();
    *out = b3d200_depth_image_new(w, h, std::move(d));
  });
}

b3d_status b3d_depth_image_save(const b3d_depth_image* img, const char* path) {
  return guarded([&] {  // io.cpp:91-102
    check(img && path, "bad arguments");
    const uint32_t w = b3d_depth_image_width(img), h = b3d_depth_image_height(img);
    const float* d = b3d_depth_image_data(img);
    std::string out;
    out.append("SDPT", 4);
    put<uint32_t>(out, w);
    put<uint32_t>(out, h);
    for (size_t i = 0; i < (size_t)w * h; ++i) put<float>(out, d[i]);
    write_file_atomic(path, out);
  });
}

b3d_status b3d_model_from_voxels(const int32_t* voxels, size_t n, double resolution,
                                 const double origin[3], int id, b3d_object_model** out) {
  return guarded([&] {
    check(voxels && origin && out, "bad arguments");
    require(resolution > 0, B3D_ERROR, "object model: non-positive resolution");
    auto m = model_from_grid(id, resolution, origin,
                             std::vector<int32_t>(voxels, voxels + 3 * n));
    *out = new b3d_object_model(*m);
  });
}

b3d_status b3d_model_load(const char* path, int id, b3d_object_model** out) {
  return guarded([&] {
    check(path && out, "bad arguments");
    *out = new b3d_object_model(*load_svox(path, id));
  });
}

b3d_status b3d_model_save(const b3d_object_model* model, const char* path) {
  return guarded([&] {  // io.cpp:118-130
    check(model && path, "bad arguments");
    std::string out;
    out.append("SVOX", 4);
    put<float>(out, (float)model->resolution);
    for (int i = 0; i < 3; ++i) put<float>(out, (float)model->origin[i]);
    put<uint32_t>(out, (uint32_t)(model->voxels.size() / 3));
    for (int32_t v : model->voxels) put<int32_t>(out, v);
    write_file_atomic(path, out);
  });
}

b3d_status b3d_model_bbox(const b3d_object_model* model, double extents[3]) {
  return guarded([&] {
    check(model && extents, "bad arguments");
    for (int a = 0; a < 3; ++a) extents[a] = model->aabb_max[a] - model->aabb_min[a];
  });
}

b3d_status b3d_model_resolution(const b3d_object_model* model, double* out) {
  return guarded([&] {
    check(model && out, "bad arguments");
    *out = model->resolution;
  });
}

b3d_status b3d_model_voxel_count(const b3d_object_model* model, size_t* out) {
  return guarded([&] {
    check(model && out, "bad arguments");
    *out = model->voxels.size() / 3;
  });
}

b3d_status b3d_model_mesh(const b3d_object_model* model, const double** vertices,
                          uint64_t* n_vertices, const uint32_t** triangles,
                          uint64_t* n_triangles) {
  return guarded([&] {
    check(model && vertices && n_vertices && triangles && n_triangles, "bad arguments");
    *vertices = model->verts.data();
    *n_vertices = model->verts.size() / 3;
    *triangles = model->tris.data();
    *n_triangles = model->tris.size() / 3;
  });
}

void b3d_model_destroy(b3d_object_model* model) { delete model; }

// The reference parses scene / manifest JSON with nlohmann::json and reports
// its exceptions verbatim (scene_graph.cpp:201-203, 219-221): the same text
// for the same defect -- at() on a missing key (out_of_range.403), get<T>() of
// the wrong type (type_error.302), at() on a non-object (type_error.304).
const char* nl_type_name(const J::Value& v) {
  switch (v.kind) {
    case J::Value::Null: return "null";
    case J::Value::Bool: return "boolean";
    case J::Value::Number: return "number";
    case J::Value::String: return "string";
    case J::Value::Array: return "array";
    default: return "object";
  }
}
struct NlError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
const J::Value& nl_at(const J::Value& o, const char* key) {
  if (!o.is_object())
    throw NlError(std::string("[json.exception.type_error.304] cannot use at() with ") +
                  nl_type_name(o));
  const J::Value* x = o.find(key);
  if (!x) throw NlError(std::string("[json.exception.out_of_range.403] key '") + key + "' not found");
  return *x;
}
double nl_number(const J::Value& v) {  // get<double>
  if (v.kind != J::Value::Number)
    throw NlError(std::string("[json.exception.type_error.302] type must be number, but is ") +
                  nl_type_name(v));
  return v.num;
}
// Json::get<int>() outside a ConfigReader (the schedule lambda,
// b3d_capi.cpp:344-349): a non-number is nlohmann's own type_error
int nl_get_int(const J::Value& v) {
  if (!is_arith(v))
    throw NlError(std::string("[json.exception.type_error.302] type must be number, but is ") +
                  nl_type_name(v));
  return json_int(v);
}
// range-for over a json value: array elements, object values, nothing for
// null, the value itself for a primitive
std::vector<const J::Value*> nl_elems(const J::Value& v) {
  std::vector<const J::Value*> out;
  if (v.kind == J::Value::Array)
    for (const J::Value& e : v.arr) out.push_back(&e);
  else if (v.kind == J::Value::Object)
    for (const auto& kv : v.obj) out.push_back(&kv.second);
  else if (v.kind != J::Value::Null)
    out.push_back(&v);
  return out;
}
const std::string& nl_string(const J::Value& v) {
  if (v.kind != J::Value::String)
    throw NlError(std::string("[json.exception.type_error.302] type must be string, but is ") +
                  nl_type_name(v));
  return v.str;
}

b3d_status b3d_library_open(const char* manifest_path, b3d_library** out) {
  return guarded([&] {  // load_library (scene_graph.cpp:206-234)
    check(out && manifest_path, "bad arguments");
    const std::string mp = manifest_path;
    const std::string text = read_file(mp);
    const J::Value j = parse_or(text.c_str(), B3D_ERROR_CONFIG,
                                (mp + ": invalid JSON").c_str());
    const J::Value* models = j.is_object() ? j.find("models") : nullptr;
    require(models && models->is_array(), B3D_ERROR_CONFIG,
            mp + ": manifest requires a 'models' array");
    const size_t slash = mp.find_last_of('/');
    const std::string base = slash == std::string::npos ? "" : mp.substr(0, slash + 1);
    auto lib = std::make_unique<b3d_library>();
    lib->models.resize(models->arr.size());
    for (const J::Value& m : models->arr) {
      int id = 0;
      std::string rel;
      try {  // mj.at("id").get<int>(), mj.at("path").get<std::string>()
        id = nl_get_int(nl_at(m, "id"));
        rel = nl_string(nl_at(m, "path"));
      } catch (const NlError& e) {
        throw Fail(B3D_ERROR_CONFIG, mp + ": bad model entry: " + e.what());
      }
      require(id >= 0 && (size_t)id < lib->models.size(), B3D_ERROR_CONFIG,
              mp + ": model ids must be dense 0-based");
      require(!lib->models[id], B3D_ERROR_CONFIG, mp + ": duplicate model id");
      lib->models[id] = load_svox(base + rel, id);
    }
    *out = lib.release();
  });
}

b3d_status b3d_library_create(const b3d_object_model* const* models, size_t n,
                              b3d_library** out) {
  return guarded([&] {
    check(models && out && n > 0, "bad arguments");
    auto lib = std::make_unique<b3d_library>();
    for (size_t i = 0; i < n; ++i) {
      check(models[i] != nullptr, "null model");
      lib->models.push_back(std::make_shared<b3d_object_model>(*models[i]));
    }
    *out = lib.release();
  });
}

size_t b3d_library_size(const b3d_library* lib) { return lib ? lib->models.size() : 0; }

void b3d_library_destroy(b3d_library* lib) { delete lib; }

b3d_status b3d_scene_from_json(const char* json, const b3d_library* lib, b3d_scene** out) {
  return guarded([&] {  // scene_from_json (scene_graph.cpp:182-204)
    check(json && lib && out, "bad arguments");
    const J::Value j = parse_or(json, B3D_ERROR_CONFIG, "invalid scene JSON");
    const J::Value* t = j.is_object() ? j.find("table") : nullptr;
    require(t != nullptr, B3D_ERROR_CONFIG, "scene JSON: missing 'table'");
    auto s = std::make_unique<b3d_scene>();
    try {  // the reference's order: thickness (value), then the table() arguments
           // right to left as its build (gcc) evaluates them, then children
      const J::Value* th = t->is_object() ? t->find("thickness") : nullptr;
      if (!t->is_object())
        throw NlError(std::string("[json.exception.type_error.306] cannot use value() with ") +
                      nl_type_name(*t));
      s->thickness = th ? nl_number(*th) : 0.01;
      s->table_h = nl_number(nl_at(*t, "height"));
      s->table_w = nl_number(nl_at(*t, "width"));
      require(s->table_w > 0 && s->table_h > 0 && s->thickness > 0, B3D_ERROR,
              "table: extents must be positive");
      if (const J::Value* ch = j.find("children")) {  // j.value("children", [])
        for (const J::Value* cp : nl_elems(*ch)) {
          const J::Value& c = *cp;
          const int id = nl_get_int(nl_at(c, "object_id"));
          require(id >= 0 && (size_t)id < lib->models.size(), B3D_ERROR_CONFIG,
                  "scene JSON: object_id out of library range");
          const int face = nl_get_int(nl_at(c, "face"));
          const double dx = nl_number(nl_at(c, "dx"));
          const double dy = nl_number(nl_at(c, "dy"));
          const double dth = nl_number(nl_at(c, "dtheta"));
          s->children.push_back({lib->models[id], face, dx, dy, dth});
        }
      }
    } catch (const NlError& e) {
      throw Fail(B3D_ERROR_CONFIG, std::string("bad scene JSON: ") + e.what());
    }
    *out = s.release();
  });
}

b3d_status b3d_scene_to_json(const b3d_scene* scene, char** out_json) {
  return guarded([&] {  // scene_to_json (scene_graph.cpp:170-180)
    check(scene && out_json, "bad arguments");
    const double w = scene->table_w / 2 - (-scene->table_w / 2);
    const double h = scene->table_h / 2 - (-scene->table_h / 2);
    const double z = 0.0 - (-scene->thickness);
    std::string s = "{\"children\":[";
    for (size_t i = 0; i < scene->children.size(); ++i) {
      const auto& c = scene->children[i];
      if (i) s += ",";
      s += "{\"dtheta\":" + J::num(c.dtheta) + ",\"dx\":" + J::num(c.dx) +
           ",\"dy\":" + J::num(c.dy) + ",\"face\":" + std::to_string(c.face) +
           ",\"object_id\":" + std::to_string(c.obj->id) + "}";
    }
    s += "],\"table\":{\"height\":" + J::num(h) + ",\"thickness\":" + J::num(z) +
         ",\"width\":" + J::num(w) + "}}";
    *out_json = owned(s);
  });
}

void b3d_scene_destroy(b3d_scene* scene) { delete scene; }

void b3d_string_free(char* s) { delete[] s; }

b3d_status b3d_render(const b3d_scene* scene, const b3d_pose* camera, const b3d_intrinsics* k,
                      b3d_depth_image** out) {
  return guarded([&] {  // render_depth (renderer.cpp:176-179) on the device
    check(scene && camera && k && out, "bad arguments");
    // render_depth(scene, from_c(*camera), from_c(*k)) (b3d_capi.cpp:271):
    // the reference's build (gcc) evaluates the arguments right to left --
    // intrinsics, then the camera -- and scene_instances' contacts
    // (renderer.cpp:153-162) come inside
    b3d200_validate_intrinsics(*k);
    const b3d_pose cam = normalized_pose(*camera);
    std::vector<b3d_pose> poses{b3d_pose{1, 0, 0, 0, 0, 0, 0}};
    for (const auto& c : scene->children) {
      b3d_pose p;
      ok(b3d_contact_to_pose(scene->table_w, scene->table_h, c.obj->aabb_min, c.obj->aabb_max,
                             c.face, c.dx, c.dy, c.dtheta, &p));
      poses.push_back(p);
    }
    b3d_gpu_context* g = g_gpu.get();
    std::vector<int32_t> ids{g_gpu.table(scene->table_w, scene->table_h, scene->thickness)};
    for (const auto& c : scene->children) ids.push_back(g_gpu.mesh(*c.obj));
    std::vector<float> depth((size_t)k->width * k->height);
    if (ids.size() <= B3D_MAX_INSTANCES) {  // camera mode: one launch
      g_gpu.camera(k);  // both kept from the previous call when unchanged
      g_gpu.camera_scene(ids, poses);
      ok(b3d_gpu_render_cameras(g, &cam, 1, depth.data(), nullptr));
    } else {  // any number of children: instance after instance
      g_gpu.cam_key.clear();  // sets the camera itself
      b3d200_render_scene_keys(g, k, &cam, ids.data(), poses.data(), (uint32_t)ids.size(),
                               depth.data());
    }
    ok(b3d_depth_image_create(k->width, k->height, depth.data(), out));
  });
}

b3d_status b3d_infer(const b3d_depth_image* observed, const b3d_pose* camera,
                     const b3d_library* lib, const char* config_json, uint64_t seed,
                     b3d_particles** out) {
  return guarded([&] {  // b3d_capi.cpp:297-379 with run_smc on the device
    check(observed && camera && lib && config_json && out, "bad arguments");
    const J::Value config =
        parse_or(config_json, B3D_ERROR_CONFIG, "invalid inference config JSON");
    Reader r(config, "b3d_infer config");
    r.int_or("threads", 0);
    b3d_intrinsics ik{};
    require(r.has("intrinsics"), B3D_ERROR_CONFIG, "b3d_infer: config requires 'intrinsics'");
    {
      Reader ir = r.object("intrinsics");
      ik.fx = ir.num("fx");
      ik.fy = ir.num("fy");
      ik.cx = ir.num("cx");
      ik.cy = ir.num("cy");
      ik.width = ir.u32("width");
      ik.height = ir.u32("height");
      ik.near_m = ir.num("near");
      ik.far_m = ir.num("far");
      ir.finish();
      b3d200_validate_intrinsics(ik);  // from_c (b3d_capi.cpp:54-65)
    }
    const double sigma_max = r.num_or("sigma_max", 0.1);
    const int window = r.int_or("window", 2);
    // window < 0: ModelConfig::windowed = false, the untruncated likelihood
    // (b3d_capi.cpp:328-330) -- scored on the device's fp64 image path
    double tw, th, thick;
    {
      Reader tr = r.object("table");
      // ObjectModel::table(get("width"), get("height"), get_or("thickness"))
      // (b3d_capi.cpp:335-337): the reference's build (gcc) evaluates the
      // arguments right to left, so a bad thickness is reported first
      thick = tr.num_or("thickness", 0.01);
      th = tr.num("height");
      tw = tr.num("width");
      // ObjectModel::table (scene_graph.cpp:26-28) runs before tr.finish()
      require(tw > 0 && th > 0 && thick > 0, B3D_ERROR, "table: extents must be positive");
      tr.finish();
    }
    b3d_smc_config cfg{};
    struct StageI {
      int n_dx, n_dy, n_dtheta;
    };
    StageI stage0{10, 10, 8};  // Schedule defaults (inference.hpp:30-31)
    std::vector<StageI> refine_i{{5, 5, 5}, {5, 5, 5}};
    if (r.has("schedule")) {
      Reader sr = r.object("schedule");
      auto stage = [](const J::Value& v) {
        require(v.is_array() && v.arr.size() == 3, B3D_ERROR_CONFIG,
                "schedule stages must be [n_dx, n_dy, n_dtheta]");
        return StageI{nl_get_int(v.arr[0]), nl_get_int(v.arr[1]), nl_get_int(v.arr[2])};
      };
      stage0 = stage(sr.raw("stage0"));
      refine_i.clear();
      for (const J::Value* v : nl_elems(sr.raw("refine"))) refine_i.push_back(stage(*v));
      sr.finish();
    }
    std::vector<b3d_noise> grid;  // default_noise_grid (inference.cpp:127-133)
    for (double p : {0.05, 0.3, 0.8})
      for (double frac : {0.25, 0.5, 1.0}) grid.push_back({p, frac * sigma_max});
    if (r.has("noise_grid")) {
      Reader gr = r.object("noise_grid");
      grid.clear();
      // b3d_capi.cpp:356-363 reads "sigma" inside the p_outlier loop: an
      // empty p_outlier leaves it unread (an unknown key at finish())
      for (const J::Value* p : nl_elems(gr.raw("p_outlier")))
        for (const J::Value* sv : nl_elems(gr.raw("sigma")))
          grid.push_back({nl_number(*p), nl_number(*sv)});
      gr.finish();
    }
    const int n_objects = r.int_or("n_objects", 1);
    const int n_particles = r.int_or("particles", 1000);
    cfg.resample_threshold = r.num_or("resample_threshold", 0.5);
    r.finish();
    // make_inference_context(observed, from_c(*camera), ...) (b3d_capi.cpp:368-370):
    // the camera is converted (unit quaternion check) as an argument, before
    // the context's own checks
    const b3d_pose cam = normalized_pose(*camera);
    // make_inference_context (inference.cpp:140-157), then run_smc / smc_init
    // (inference.cpp:495, 400): the reference's checks in its order, all
    // before any device work
    require(!lib->models.empty(), B3D_ERROR, "inference: empty library");
    require(!grid.empty(), B3D_ERROR, "inference: empty noise grid");
    auto valid = [](const StageI& st) { return st.n_dx >= 1 && st.n_dy >= 1 && st.n_dtheta >= 1; };
    require(valid(stage0), B3D_ERROR, "schedule stage: subdivision counts must be >= 1");
    for (const StageI& st : refine_i)
      require(valid(st), B3D_ERROR, "schedule stage: subdivision counts must be >= 1");
    for (const b3d_noise& np : grid)
      require(np.p_outlier >= 0 && np.p_outlier <= 1 && np.sigma_noise > 0 &&
                  np.sigma_noise <= sigma_max,
              B3D_ERROR, "noise grid entry outside support");
    require(b3d_depth_image_width(observed) == ik.width &&
                b3d_depth_image_height(observed) == ik.height,
            B3D_ERROR, "observation dimensions do not match intrinsics");
    require(n_objects >= 1, B3D_ERROR, "run_smc: n_objects must be >= 1");
    require(n_particles >= 1, B3D_ERROR, "smc_init: need at least one particle");
    cfg.stage0 = {(uint32_t)stage0.n_dx, (uint32_t)stage0.n_dy, (uint32_t)stage0.n_dtheta};
    std::vector<b3d_schedule_stage> refine;
    for (const StageI& st : refine_i)
      refine.push_back({(uint32_t)st.n_dx, (uint32_t)st.n_dy, (uint32_t)st.n_dtheta});
    cfg.n_objects = (uint32_t)n_objects;
    cfg.n_particles = (uint32_t)n_particles;
    b3d_gpu_context* g = g_gpu.get();
    g_gpu.cam_key.clear();
    ok(b3d_gpu_set_camera(g, &ik, &cam));
    ok(b3d_gpu_set_observation(g, b3d_depth_image_data(observed)));
    std::vector<b3d_smc_object> objs;
    for (const auto& m : lib->models) {
      b3d_smc_object o{};
      o.mesh_id = g_gpu.mesh(*m);
      for (int a = 0; a < 3; ++a) {
        o.aabb_min[a] = m->aabb_min[a];
        o.aabb_max[a] = m->aabb_max[a];
      }
      objs.push_back(o);
    }
    cfg.table_w = tw / 2 - (-tw / 2);  // ObjectModel::table extents
    cfg.table_h = th / 2 - (-th / 2);
    cfg.table_mesh = g_gpu.table(tw, th, thick);
    cfg.n_refine = (uint32_t)refine.size();
    cfg.refine = refine.data();
    cfg.noise_grid = grid.data();
    cfg.n_noise_grid = (uint32_t)grid.size();
    cfg.sigma_max = sigma_max;
    cfg.window = (int32_t)window;
    cfg.prefactor = B3D_PREFACTOR_PRINTED;  // ModelConfig default (generative.hpp:38)
    auto res = std::make_unique<b3d_particles>();
    res->ps.resize(cfg.n_particles ? cfg.n_particles : 1);
    res->kids.resize(res->ps.size() * std::max<size_t>(cfg.n_objects, 1));
    for (size_t i = 0; i < res->ps.size(); ++i)
      res->ps[i].children = res->kids.data() + i * std::max<size_t>(cfg.n_objects, 1);
    ok(b3d_gpu_run_smc(g, objs.data(), (uint32_t)objs.size(), &cfg, seed, res->ps.data(),
                       &res->log_evidence));
    res->table_w = cfg.table_w;
    res->table_h = cfg.table_h;
    res->lib = lib->models;
    res->grid = grid;
    *out = res.release();
  });
}

size_t b3d_particles_count(const b3d_particles* p) { return p ? p->ps.size() : 0; }

b3d_status b3d_particles_log_evidence(const b3d_particles* p, double* out) {
  return guarded([&] {
    check(p && out, "bad arguments");
    *out = p->log_evidence;
  });
}

b3d_status b3d_particles_to_jsonl(const b3d_particles* p, char** out) {
  return guarded([&] {  // b3d_capi.cpp:389-411 (keys sorted like nlohmann's dump)
    check(p && out, "bad arguments");
    std::string lines;
    for (const b3d_smc_particle& q : p->ps) {
      std::string s = "{\"children\":[";
      for (int c = 0; c < q.n_children; ++c) {
        const b3d_smc_child& ch = q.children[c];
        if (c) s += ",";
        s += "{\"dtheta\":" + J::num(ch.dtheta) + ",\"dx\":" + J::num(ch.dx) +
             ",\"dy\":" + J::num(ch.dy) + ",\"face\":" + std::to_string(ch.face) +
             ",\"object_id\":" + std::to_string(p->lib[ch.object_id]->id) + "}";
      }
      const b3d_noise& nz = p->grid[q.noise_index];
      s += "],\"log_weight\":" + J::num(q.log_weight) + ",\"noise\":{\"p_outlier\":" +
           J::num(nz.p_outlier) + ",\"sigma_noise\":" + J::num(nz.sigma_noise) + "}}\n";
      lines += s;
    }
    *out = owned(lines);
  });
}

b3d_status b3d_particles_type_marginal(const b3d_particles* p, double* probs, size_t capacity) {
  return guarded([&] {  // posterior_object_marginal (inference.cpp:522-537)
    check(p && probs, "bad arguments");
    check(capacity >= p->lib.size(), "marginal buffer too small");
    require(!p->ps.empty(), B3D_ERROR, "marginal: empty particle set");
    for (const b3d_smc_particle& q : p->ps)
      require(q.n_children == 1, B3D_ERROR, "marginal: expected one-object particles");
    double m = -INFINITY;  // normalized_weights (inference.cpp:443-455)
    for (const b3d_smc_particle& q : p->ps) m = std::max(m, q.log_weight);
    require(std::isfinite(m), B3D_ERROR_NUMERIC, "particle weights are all zero");
    double acc = 0;
    for (const b3d_smc_particle& q : p->ps) acc += std::exp(q.log_weight - m);
    const double lse = m + std::log(acc);
    std::vector<double> marginal(p->lib.size(), 0.0);
    for (const b3d_smc_particle& q : p->ps) {
      const int id = p->lib[q.children[0].object_id]->id;
      require(id >= 0 && (size_t)id < p->lib.size(), B3D_ERROR,
              "marginal: object id out of range");
      marginal[id] += std::exp(q.log_weight - lse);
    }
    std::copy(marginal.begin(), marginal.end(), probs);
  });
}

b3d_status b3d_particles_map_pose(const b3d_particles* p, size_t index, b3d_pose* out) {
  return guarded([&] {  // map_particle (inference.cpp:539-545) + contact_to_pose
    check(p && out, "bad arguments");
    require(!p->ps.empty(), B3D_ERROR, "map_particle: empty set");
    size_t best = 0;
    for (size_t i = 1; i < p->ps.size(); ++i)
      if (p->ps[i].log_target > p->ps[best].log_target) best = i;
    const b3d_smc_particle& q = p->ps[best];
    check(index < (size_t)q.n_children, "child index out of range");
    const b3d_smc_child& c = q.children[index];
    const b3d_object_model& m = *p->lib[c.object_id];
    ok(b3d_contact_to_pose(p->table_w, p->table_h, m.aabb_min, m.aabb_max, c.face, c.dx, c.dy,
                           c.dtheta, out));
  });
}

void b3d_particles_destroy(b3d_particles* p) { delete p; }

}  // extern "C"
