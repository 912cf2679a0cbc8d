/*
 * b3d_oracle.c -- CPU ORACLE (test infrastructure only; see b3d_oracle.h).
 *
 * A scalar fp64 restatement of the reference hot path.  Every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/src/core/).  Compiled with -O2 -ffp-contract=off so
 * no FMA contraction happens, like the reference's x86-64 -O2 build.
 *
 * Eigen expressions are restated with Eigen's scalar (non-SIMD) evaluation
 * order: 3-term sums reduce as a0 + (a1 + a2), 4-term sums as
 * (a0 + a1) + (a2 + a3), quaternion products with the generic formula.
 * Eigen is absent from this container, so this order is unpinned at the
 * ulp level; the CUDA product path follows the same order.
 */
#include "b3d_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static const double kTwoPi = 6.283185307179586476925287;

/* ------------------------------------------------------------------ RNG */
/* rng.hpp:8-13 */
static uint64_t splitmix64_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.cpp:13-16 */
static uint64_t rng_mix(uint64_t a, uint64_t b) {
  uint64_t state = a ^ (0x9e3779b97f4a7c15ull + (b << 6) + (b >> 2));
  return splitmix64_next(&state);
}

/* rng.cpp:20-23 */
void orc_rng_seed(uint64_t seed, uint64_t st[5]) {
  uint64_t s = seed;
  st[0] = seed;
  for (int i = 0; i < 4; ++i) st[1 + i] = splitmix64_next(&s);
}

/* rng.cpp:25-28 */
void orc_rng_split(const uint64_t st[5], uint64_t k0, uint64_t k1, uint64_t k2,
                   uint64_t out[5]) {
  orc_rng_seed(rng_mix(rng_mix(rng_mix(st[0], k0), k1), k2), out);
}

/* rng.cpp:30-40 */
uint64_t orc_rng_next_u64(uint64_t st[5]) {
  uint64_t* s = st + 1;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.cpp:42-44 */
double orc_rng_uniform(uint64_t st[5]) {
  return (double)(orc_rng_next_u64(st) >> 11) * 0x1.0p-53;
}

/* rng.cpp:48-57 */
uint64_t orc_rng_uniform_int(uint64_t st[5], uint64_t n) {
  if (n < 1) return 0;
  const uint64_t limit = n * (UINT64_MAX / n);
  uint64_t x;
  do {
    x = orc_rng_next_u64(st);
  } while (x >= limit);
  return x % n;
}

/* rng.cpp:59-64 */
double orc_rng_normal(uint64_t st[5]) {
  double u1 = orc_rng_uniform(st);
  double u2 = orc_rng_uniform(st);
  while (u1 <= 0.0) u1 = orc_rng_uniform(st);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}

/* ------------------------------------------------------------ pose math */
typedef struct quat {
  double w, x, y, z;
} quat;

/* Eigen QuaternionBase::normalized(): coeffs / sqrt(squaredNorm) with the
 * coefficients stored (x,y,z,w); scalar 4-term redux (x2+y2)+(z2+w2). */
static quat q_normalized(quat q) {
  const double n2 = (q.x * q.x + q.y * q.y) + (q.z * q.z + q.w * q.w);
  if (n2 > 0) {
    const double n = sqrt(n2);
    q.w /= n;
    q.x /= n;
    q.y /= n;
    q.z /= n;
  }
  return q;
}

/* Eigen generic quat_product. */
static quat q_mul(quat a, quat b) {
  quat r;
  r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  r.y = a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z;
  r.z = a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x;
  return r;
}

static void cross3(const double a[3], const double b[3], double out[3]) {
  out[0] = a[1] * b[2] - a[2] * b[1];
  out[1] = a[2] * b[0] - a[0] * b[2];
  out[2] = a[0] * b[1] - a[1] * b[0];
}

/* Eigen QuaternionBase::_transformVector: uv = q.vec x v; uv += uv;
 * return v + w*uv + q.vec x uv. */
static void q_rotate(quat q, const double v[3], double out[3]) {
  const double qv[3] = {q.x, q.y, q.z};
  double uv[3], c[3];
  cross3(qv, v, uv);
  uv[0] += uv[0];
  uv[1] += uv[1];
  uv[2] += uv[2];
  cross3(qv, uv, c);
  for (int i = 0; i < 3; ++i) out[i] = v[i] + q.w * uv[i] + c[i];
}

static quat pose_q(const orc_pose* p) {
  quat q = {p->qw, p->qx, p->qy, p->qz};
  return q;
}

void orc_quat_rotate(const orc_pose* p, const double v[3], double out[3]) {
  q_rotate(pose_q(p), v, out);
}

/* geometry.cpp:19-24: q = (a.q * b.q).normalized(); t = a.q * b.t + a.t */
void orc_compose(const orc_pose* a, const orc_pose* b, orc_pose* out) {
  const quat q = q_normalized(q_mul(pose_q(a), pose_q(b)));
  const double bt[3] = {b->tx, b->ty, b->tz};
  double r[3];
  q_rotate(pose_q(a), bt, r);
  orc_pose o;
  o.qw = q.w;
  o.qx = q.x;
  o.qy = q.y;
  o.qz = q.z;
  o.tx = r[0] + a->tx;
  o.ty = r[1] + a->ty;
  o.tz = r[2] + a->tz;
  *out = o;
}

/* geometry.cpp:26-31: q' = conj(q).normalized(); t' = -(q' * t) */
void orc_inverse(const orc_pose* p, orc_pose* out) {
  quat c = {p->qw, -p->qx, -p->qy, -p->qz};
  c = q_normalized(c);
  const double t[3] = {p->tx, p->ty, p->tz};
  double r[3];
  q_rotate(c, t, r);
  orc_pose o;
  o.qw = c.w;
  o.qx = c.x;
  o.qy = c.y;
  o.qz = c.z;
  o.tx = -r[0];
  o.ty = -r[1];
  o.tz = -r[2];
  *out = o;
}

/* Eigen QuaternionBase::toRotationMatrix (geometry.hpp:29). Row-major. */
void orc_rotation_matrix(const orc_pose* p, double m[9]) {
  const double tx = 2.0 * p->qx, ty = 2.0 * p->qy, tz = 2.0 * p->qz;
  const double twx = tx * p->qw, twy = ty * p->qw, twz = tz * p->qw;
  const double txx = tx * p->qx, txy = ty * p->qx, txz = tz * p->qx;
  const double tyy = ty * p->qy, tyz = tz * p->qy, tzz = tz * p->qz;
  m[0] = 1.0 - (tyy + tzz);
  m[1] = txy - twz;
  m[2] = txz + twy;
  m[3] = txy + twz;
  m[4] = 1.0 - (txx + tzz);
  m[5] = tyz - twx;
  m[6] = txz - twy;
  m[7] = tyz + twx;
  m[8] = 1.0 - (txx + tyy);
}

/* Eigen AngleAxis -> Quaternion; geometry.cpp:11-17 normalizes the axis. */
void orc_from_axis_angle(const double axis[3], double angle, orc_pose* out) {
  double a[3] = {axis[0], axis[1], axis[2]};
  const double n2 = a[0] * a[0] + (a[1] * a[1] + a[2] * a[2]);
  if (n2 > 0) {
    const double n = sqrt(n2);
    a[0] /= n;
    a[1] /= n;
    a[2] /= n;
  }
  const double ha = 0.5 * angle;
  const double s = sin(ha);
  out->qw = cos(ha);
  out->qx = s * a[0];
  out->qy = s * a[1];
  out->qz = s * a[2];
  out->tx = out->ty = out->tz = 0.0;
}

/* Eigen quaternionbase_assign_impl<Matrix3>: rotation matrix -> quaternion.
 * m row-major. */
static quat quat_from_matrix(const double m[9]) {
#define M(i, j) m[(i)*3 + (j)]
  quat q;
  double t = M(0, 0) + (M(1, 1) + M(2, 2));
  if (t > 0) {
    t = sqrt(t + 1.0);
    q.w = 0.5 * t;
    t = 0.5 / t;
    q.x = (M(2, 1) - M(1, 2)) * t;
    q.y = (M(0, 2) - M(2, 0)) * t;
    q.z = (M(1, 0) - M(0, 1)) * t;
  } else {
    int i = 0;
    if (M(1, 1) > M(0, 0)) i = 1;
    if (M(2, 2) > M(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    double c[3];
    t = sqrt(M(i, i) - M(j, j) - M(k, k) + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    q.w = (M(k, j) - M(j, k)) * t;
    c[j] = (M(j, i) + M(i, j)) * t;
    c[k] = (M(k, i) + M(i, k)) * t;
    q.x = c[0];
    q.y = c[1];
    q.z = c[2];
  }
#undef M
  return q;
}

/* generative.cpp:35-59 */
void orc_camera_pose_from_spherical(double distance, double azimuth, double altitude,
                                    orc_pose* out) {
  const double pos[3] = {distance * cos(altitude) * cos(azimuth),
                         distance * cos(altitude) * sin(azimuth),
                         distance * sin(altitude)};
  double fwd[3] = {-pos[0], -pos[1], -pos[2]};
  {
    const double n2 = fwd[0] * fwd[0] + (fwd[1] * fwd[1] + fwd[2] * fwd[2]);
    const double n = sqrt(n2);
    if (n2 > 0) {
      fwd[0] /= n;
      fwd[1] /= n;
      fwd[2] /= n;
    }
  }
  const double d = 0.0 * fwd[0] + (0.0 * fwd[1] + 1.0 * fwd[2]);
  double up[3] = {0.0 - d * fwd[0], 0.0 - d * fwd[1], 1.0 - d * fwd[2]};
  {
    const double n2 = up[0] * up[0] + (up[1] * up[1] + up[2] * up[2]);
    const double n = sqrt(n2);
    if (n2 > 0) {
      up[0] /= n;
      up[1] /= n;
      up[2] /= n;
    }
  }
  const double down[3] = {-up[0], -up[1], -up[2]};
  double right[3];
  cross3(down, fwd, right);
  const double m[9] = {right[0], down[0], fwd[0], right[1], down[1],
                       fwd[1],   right[2], down[2], fwd[2]};
  const quat q = q_normalized(quat_from_matrix(m));
  out->qw = q.w;
  out->qx = q.x;
  out->qy = q.y;
  out->qz = q.z;
  out->tx = pos[0];
  out->ty = pos[1];
  out->tz = pos[2];
}

/* scene_graph.cpp:60-71 */
static quat face_rotation(int face) {
  const double half_pi = kTwoPi / 4.0;
  static const double ux[3] = {1, 0, 0}, uy[3] = {0, 1, 0};
  orc_pose p;
  switch (face) {
    case 1: {
      quat q = {1, 0, 0, 0};
      return q;
    }
    case 2: orc_from_axis_angle(ux, 2 * half_pi, &p); break;
    case 3: orc_from_axis_angle(uy, -half_pi, &p); break;
    case 4: orc_from_axis_angle(uy, half_pi, &p); break;
    case 5: orc_from_axis_angle(ux, half_pi, &p); break;
    default: orc_from_axis_angle(ux, -half_pi, &p); break;
  }
  return pose_q(&p);
}

static void mat_vec(const double m[9], const double v[3], double out[3]) {
  for (int i = 0; i < 3; ++i)
    out[i] = m[i * 3 + 0] * v[0] + (m[i * 3 + 1] * v[1] + m[i * 3 + 2] * v[2]);
}

/* scene_graph.cpp:73-89 */
void orc_rotated_bounds(const double amin[3], const double amax[3], int face,
                        double lo[3], double hi[3]) {
  const quat q = face_rotation(face);
  orc_pose p = {q.w, q.x, q.y, q.z, 0, 0, 0};
  double m[9];
  orc_rotation_matrix(&p, m);
  for (int i = 0; i < 8; ++i) {
    const double c[3] = {i & 1 ? amax[0] : amin[0], i & 2 ? amax[1] : amin[1],
                         i & 4 ? amax[2] : amin[2]};
    double r[3];
    mat_vec(m, c, r);
    for (int a = 0; a < 3; ++a) {
      if (i == 0) {
        lo[a] = hi[a] = r[a];
      } else {
        lo[a] = r[a] < lo[a] ? r[a] : lo[a];  /* cwiseMin */
        hi[a] = r[a] > hi[a] ? r[a] : hi[a];  /* cwiseMax */
      }
    }
  }
}

/* scene_graph.cpp:97-121 */
int orc_contact_to_pose(double table_w, double table_h, const double amin[3],
                        const double amax[3], int face, double dx, double dy,
                        double dtheta, orc_pose* out) {
  if (face < 1 || face > 6) return 1;
  double lo[3], hi[3];
  orc_rotated_bounds(amin, amax, face, lo, hi);
  const double w = hi[0] - lo[0];
  const double h = hi[1] - lo[1];
  if (!(dx >= 0 && dx <= table_w - w && dy >= 0 && dy <= table_h - h && dtheta >= 0 &&
        dtheta < kTwoPi))
    return 1;
  const double corner[3] = {-table_w / 2, -table_h / 2, 0.0};
  const double bt[3] = {corner[0] + (dx - lo[0]), corner[1] + (dy - lo[1]),
                        corner[2] + -lo[2]};
  const double pivot[3] = {corner[0] + (dx + w / 2), corner[1] + (dy + h / 2),
                           corner[2] + 0.0};
  static const double uz[3] = {0, 0, 1};
  orc_pose sp;
  orc_from_axis_angle(uz, dtheta, &sp);
  const quat spin = pose_q(&sp);
  const quat q = q_normalized(q_mul(spin, face_rotation(face)));
  const double rel[3] = {bt[0] - pivot[0], bt[1] - pivot[1], bt[2] - pivot[2]};
  double r[3];
  q_rotate(spin, rel, r);
  out->qw = q.w;
  out->qx = q.x;
  out->qy = q.y;
  out->qz = q.z;
  out->tx = r[0] + pivot[0];
  out->ty = r[1] + pivot[1];
  out->tz = r[2] + pivot[2];
  return 0;
}

/* --------------------------------------------------------------- meshes */
/* geometry.cpp:128-138 */
static const int kFaceCorners[6][4][3] = {
    {{0, 0, 0}, {0, 0, 1}, {0, 1, 1}, {0, 1, 0}},
    {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}, {1, 0, 1}},
    {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}, {0, 0, 1}},
    {{0, 1, 0}, {0, 1, 1}, {1, 1, 1}, {1, 1, 0}},
    {{0, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 0, 0}},
    {{0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}},
};
static const int kFaceOffsets[6][3] = {{-1, 0, 0}, {1, 0, 0},  {0, -1, 0},
                                       {0, 1, 0},  {0, 0, -1}, {0, 0, 1}};

/* open-addressing hash of int3 keys -> u32 (the reference uses
 * unordered_map; only membership / first-insertion ids matter) */
typedef struct ihash {
  int32_t* keys;
  uint32_t* vals;
  uint8_t* used;
  size_t cap;
} ihash;

static size_t ihash_slot(const ihash* h, const int32_t k[3]) {
  uint64_t x = 1469598103934665603ull;
  for (int i = 0; i < 3; ++i) {
    x ^= (uint64_t)(uint32_t)k[i];
    x *= 1099511628211ull;
  }
  size_t s = (size_t)(x & (h->cap - 1));
  while (h->used[s] && (h->keys[3 * s] != k[0] || h->keys[3 * s + 1] != k[1] ||
                        h->keys[3 * s + 2] != k[2]))
    s = (s + 1) & (h->cap - 1);
  return s;
}

static int ihash_init(ihash* h, size_t n) {
  size_t cap = 16;
  while (cap < 4 * n) cap <<= 1;
  h->cap = cap;
  h->keys = (int32_t*)malloc(cap * 3 * sizeof(int32_t));
  h->vals = (uint32_t*)malloc(cap * sizeof(uint32_t));
  h->used = (uint8_t*)calloc(cap, 1);
  return h->keys && h->vals && h->used ? 0 : 1;
}

static void ihash_free(ihash* h) {
  free(h->keys);
  free(h->vals);
  free(h->used);
}

/* geometry.cpp:142-177 */
int orc_voxel_to_mesh(const int32_t* vox, size_t n, double res, const double origin[3],
                      double* vertices, uint32_t* triangles, size_t* n_vertices,
                      size_t* n_triangles) {
  if (n == 0) return 1;
  ihash occ, corners;
  if (ihash_init(&occ, n) || ihash_init(&corners, 8 * n)) return 1;
  for (size_t i = 0; i < n; ++i) {
    const size_t s = ihash_slot(&occ, vox + 3 * i);
    occ.used[s] = 1;
    memcpy(occ.keys + 3 * s, vox + 3 * i, 3 * sizeof(int32_t));
  }
  size_t nv = 0, nt = 0;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* v = vox + 3 * i;
    for (int face = 0; face < 6; ++face) {
      const int32_t nb[3] = {v[0] + kFaceOffsets[face][0], v[1] + kFaceOffsets[face][1],
                             v[2] + kFaceOffsets[face][2]};
      if (occ.used[ihash_slot(&occ, nb)]) continue;
      uint32_t quad[4];
      for (int c = 0; c < 4; ++c) {
        const int32_t cc[3] = {v[0] + kFaceCorners[face][c][0],
                               v[1] + kFaceCorners[face][c][1],
                               v[2] + kFaceCorners[face][c][2]};
        const size_t s = ihash_slot(&corners, cc);
        if (!corners.used[s]) {
          corners.used[s] = 1;
          memcpy(corners.keys + 3 * s, cc, 3 * sizeof(int32_t));
          corners.vals[s] = (uint32_t)nv;
          /* VoxelGrid::voxel_corner: origin + resolution * v.cast<double>() */
          for (int a = 0; a < 3; ++a) vertices[3 * nv + a] = origin[a] + res * (double)cc[a];
          ++nv;
        }
        quad[c] = corners.vals[s];
      }
      uint32_t* t = triangles + 3 * nt;
      t[0] = quad[0]; t[1] = quad[1]; t[2] = quad[2];
      t[3] = quad[0]; t[4] = quad[2]; t[5] = quad[3];
      nt += 2;
    }
  }
  ihash_free(&occ);
  ihash_free(&corners);
  *n_vertices = nv;
  *n_triangles = nt;
  return 0;
}

/* scene_graph.cpp:37-58 */
void orc_box_mesh(const double lo[3], const double hi[3], double v[24], uint32_t t[36]) {
  for (int i = 0; i < 8; ++i) {
    v[3 * i + 0] = (i & 1) ? hi[0] : lo[0];
    v[3 * i + 1] = (i & 2) ? hi[1] : lo[1];
    v[3 * i + 2] = (i & 4) ? hi[2] : lo[2];
  }
  static const uint32_t quads[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4},
                                       {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
  for (int f = 0; f < 6; ++f) {
    uint32_t* o = t + 6 * f;
    o[0] = quads[f][0]; o[1] = quads[f][1]; o[2] = quads[f][2];
    o[3] = quads[f][0]; o[4] = quads[f][2]; o[5] = quads[f][3];
  }
}

/* ------------------------------------------------------------- renderer */
typedef struct sv {
  double u, v, iz;
} sv;

/* renderer.cpp:18-21 */
static double edge_function(double ax, double ay, double bx, double by, double px,
                            double py) {
  return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

/* renderer.cpp:26-59 */
typedef struct edgefn {
  double ox, oy, cdx, cdy, sign, dx, dy;
} edgefn;

static edgefn make_edge(sv a, sv b) {
  const int canonical = a.u < b.u || (a.u == b.u && a.v < b.v);
  const sv lo = canonical ? a : b;
  const sv hi = canonical ? b : a;
  edgefn e;
  e.ox = lo.u;
  e.oy = lo.v;
  e.cdx = hi.u - lo.u;
  e.cdy = hi.v - lo.v;
  e.sign = canonical ? 1.0 : -1.0;
  e.dx = b.u - a.u;
  e.dy = b.v - a.v;
  return e;
}

static double edge_eval(const edgefn* e, double px, double py) {
  return e->sign * (e->cdx * (py - e->oy) - e->cdy * (px - e->ox));
}

static int edge_covers(const edgefn* e, double v) {
  if (v > 0) return 1;
  if (v < 0) return 0;
  return e->dy < 0 || (e->dy == 0 && e->dx > 0);
}

/* static_cast<int>(double) as compiled for x86-64 (cvttsd2si): values
 * outside the int range (and NaN) produce INT_MIN. */
static int to_int(double x) {
  if (!(x > -2147483649.0 && x < 2147483648.0)) return (int)0x80000000u;
  return (int)x;
}

static double min3(double a, double b, double c) {
  /* std::min({a,b,c}) */
  double m = a;
  if (b < m) m = b;
  if (c < m) m = c;
  return m;
}
static double max3(double a, double b, double c) {
  double m = a;
  if (m < b) m = b;
  if (m < c) m = c;
  return m;
}

/* renderer.cpp:61-103 (+ draw-index extension: ties keep the earlier draw) */
static void raster_screen_triangle(float* depth, int32_t* ids, const orc_intrinsics* k,
                                   sv a, sv b, sv c, int32_t draw, orc_counters* cnt) {
  double area2 = edge_function(a.u, a.v, b.u, b.v, c.u, c.v);
  if (area2 == 0) return;
  if (area2 < 0) {
    sv t = b;
    b = c;
    c = t;
    area2 = -area2;
  }
  int u_min = to_int(ceil(min3(a.u, b.u, c.u)));
  if (u_min < 0) u_min = 0;
  int u_max = to_int(floor(max3(a.u, b.u, c.u)));
  if (u_max > (int)k->width - 1) u_max = (int)k->width - 1;
  int v_min = to_int(ceil(min3(a.v, b.v, c.v)));
  if (v_min < 0) v_min = 0;
  int v_max = to_int(floor(max3(a.v, b.v, c.v)));
  if (v_max > (int)k->height - 1) v_max = (int)k->height - 1;
  if (u_min > u_max || v_min > v_max) return;

  const edgefn ab = make_edge(a, b);
  const edgefn bc = make_edge(b, c);
  const edgefn ca = make_edge(c, a);
  const double inv_area2 = 1.0 / area2;
  const float far_f = (float)k->far_m;
  const double near_z = k->near_m;

  for (int pv = v_min; pv <= v_max; ++pv) {
    float* row = depth + (size_t)pv * k->width;
    int32_t* idrow = ids ? ids + (size_t)pv * k->width : 0;
    for (int pu = u_min; pu <= u_max; ++pu) {
      if (cnt) cnt->bbox_px++;
      const double px = pu, py = pv;
      const double e_ab = edge_eval(&ab, px, py);
      const double e_bc = edge_eval(&bc, px, py);
      const double e_ca = edge_eval(&ca, px, py);
      if (!edge_covers(&ab, e_ab) || !edge_covers(&bc, e_bc) || !edge_covers(&ca, e_ca))
        continue;
      if (cnt) cnt->fragments++;
      const double inv_z = (e_bc * a.iz + e_ca * b.iz + e_ab * c.iz) * inv_area2;
      if (inv_z <= 0) continue;
      const double z = 1.0 / inv_z;
      if (z < near_z * (1.0 - 1e-12) || z > k->far_m) continue;
      const float zf = (float)z;
      if (zf < row[pu] && zf < far_f) {
        row[pu] = zf;
        if (idrow) idrow[pu] = draw;
      }
    }
  }
}

/* renderer.cpp:105-108 */
static sv project(const double p[3], const orc_intrinsics* k) {
  const double inv_z = 1.0 / p[2];
  sv s;
  s.u = k->fx * p[0] * inv_z + k->cx;
  s.v = k->fy * p[1] * inv_z + k->cy;
  s.iz = inv_z;
  return s;
}

/* renderer.cpp:112-151 */
void orc_raster_mesh(float* depth, int32_t* ids, const orc_intrinsics* k,
                     const double* verts, uint64_t nv, const uint32_t* tris, uint64_t nt,
                     const orc_pose* m2c, uint32_t draw_base, orc_counters* cnt) {
  double rot[9];
  orc_rotation_matrix(m2c, rot);
  const double t[3] = {m2c->tx, m2c->ty, m2c->tz};
  double* cam = (double*)malloc(sizeof(double) * 3 * (nv ? nv : 1));
  for (uint64_t i = 0; i < nv; ++i) {
    double r[3];
    mat_vec(rot, verts + 3 * i, r);
    cam[3 * i + 0] = r[0] + t[0];
    cam[3 * i + 1] = r[1] + t[1];
    cam[3 * i + 2] = r[2] + t[2];
  }
  if (cnt) cnt->vertices += nv;
  const double near = k->near_m;
  for (uint64_t ti = 0; ti < nt; ++ti) {
    const double* v[3] = {cam + 3 * tris[3 * ti], cam + 3 * tris[3 * ti + 1],
                          cam + 3 * tris[3 * ti + 2]};
    double poly[4][3];
    int n_poly = 0;
    for (int i = 0; i < 3; ++i) {
      const double* cur = v[i];
      const double* nxt = v[(i + 1) % 3];
      const int cur_in = cur[2] >= near;
      const int nxt_in = nxt[2] >= near;
      if (cur_in) {
        memcpy(poly[n_poly], cur, sizeof(double) * 3);
        ++n_poly;
      }
      if (cur_in != nxt_in) {
        const double s = (near - cur[2]) / (nxt[2] - cur[2]);
        /* Eigen: cur + s * (nxt - cur) */
        for (int a = 0; a < 3; ++a) poly[n_poly][a] = cur[a] + s * (nxt[a] - cur[a]);
        ++n_poly;
      }
    }
    if (n_poly < 3) continue;
    const int32_t draw = (int32_t)(draw_base + (uint32_t)ti);
    const sv s0 = project(poly[0], k);
    sv prev = project(poly[1], k);
    for (int i = 2; i < n_poly; ++i) {
      const sv cur = project(poly[i], k);
      if (cnt) cnt->triangles++;
      raster_screen_triangle(depth, ids, k, s0, prev, cur, draw, cnt);
      prev = cur;
    }
  }
  free(cam);
}

/* renderer.cpp:164-174 */
void orc_render_instances(const orc_intrinsics* k, const orc_pose* camera,
                          const orc_instance* inst, size_t n, float* depth, int32_t* ids,
                          orc_counters* cnt) {
  const size_t npx = (size_t)k->width * k->height;
  const float far_f = (float)k->far_m;
  for (size_t i = 0; i < npx; ++i) {
    depth[i] = far_f;
    if (ids) ids[i] = -1;
  }
  orc_pose w2c;
  orc_inverse(camera, &w2c);
  uint32_t draw_base = 0;
  for (size_t i = 0; i < n; ++i) {
    if (inst[i].n_triangles == 0) continue;
    orc_pose m2c;
    orc_compose(&w2c, &inst[i].model_to_world, &m2c);
    orc_raster_mesh(depth, ids, k, inst[i].vertices, inst[i].n_vertices,
                    inst[i].triangles, inst[i].n_triangles, &m2c, draw_base, cnt);
    draw_base += (uint32_t)inst[i].n_triangles;
  }
}

/* ----------------------------------------------------------- likelihood */
/* likelihood.cpp:30-35 */
double orc_visible_volume(const orc_intrinsics* k) {
  const double di = (k->far_m * k->far_m * k->far_m - k->near_m * k->near_m * k->near_m) / 3.0;
  return di * (k->width / k->fx) * (k->height / k->fy);
}

/* likelihood.cpp:231-233 */
int orc_default_window(uint32_t width) {
  const int w = (int)llround(2.0 * width / 100.0);
  return w > 1 ? w : 1;
}

/* likelihood.cpp:14-19 */
static double log_prefactor(const orc_noise* np, double sigma_max, int prefactor) {
  if (prefactor == 0) return log(np->sigma_noise / sigma_max);
  return -log(sigma_max);
}

static int noise_ok(const orc_noise* np, double sigma_max) {
  return sigma_max > 0 && np->sigma_noise > 0 && np->p_outlier >= 0 && np->p_outlier <= 1;
}

/* ObservationCache (likelihood.hpp:55-61) and ::build (likelihood.cpp:106-126) */
typedef struct obs_cache {
  int32_t* index;
  double* points;
  size_t n;
} obs_cache;

static void obs_cache_build(obs_cache* c, const float* obs, const orc_intrinsics* k) {
  const int w = (int)k->width, h = (int)k->height;
  const float sentinel = (float)k->far_m;
  const size_t npx = (size_t)w * h;
  c->index = (int32_t*)malloc(npx * sizeof(int32_t));
  c->points = (double*)malloc(npx * 3 * sizeof(double));
  c->n = 0;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const float z = obs[(size_t)v * w + u];
      c->index[(size_t)v * w + u] = -1;
      if (z >= sentinel) continue;
      c->index[(size_t)v * w + u] = (int32_t)c->n;
      const double zd = z;
      c->points[3 * c->n + 0] = (u - k->cx) * zd / k->fx;
      c->points[3 * c->n + 1] = (v - k->cy) * zd / k->fy;
      c->points[3 * c->n + 2] = zd;
      ++c->n;
    }
}

static void obs_cache_free(obs_cache* c) {
  free(c->index);
  free(c->points);
}

/* likelihood.cpp:128-220 */
static int windowed_loglik_cached(const obs_cache* oc, const float* rend,
                                  const orc_intrinsics* k, const orc_noise* noise,
                                  size_t n_noise, double volume, double sigma_max, int window,
                                  int prefactor, double* out, orc_counters* cnt) {
  if (window < 0 || !(volume > 0) || n_noise == 0) return 1;
  for (size_t e = 0; e < n_noise; ++e)
    if (!noise_ok(&noise[e], sigma_max)) return 1;
  const int w = (int)k->width, h = (int)k->height;
  const float sentinel = (float)k->far_m;
  const size_t npx = (size_t)w * h;
  const int32_t* oidx = oc->index;
  const double* opts = oc->points;
  const size_t n_obs = oc->n;

  /* backproject the rendered image once (144-158) */
  double* rp = (double*)malloc(npx * 3 * sizeof(double));
  uint8_t* rvalid = (uint8_t*)calloc(npx, 1);
  size_t rend_count = 0;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const float z = rend[(size_t)v * w + u];
      if (z >= sentinel) continue;
      const double zd = z;
      const size_t idx = (size_t)v * w + u;
      rp[3 * idx + 0] = (u - k->cx) * zd / k->fx;
      rp[3 * idx + 1] = (v - k->cy) * zd / k->fy;
      rp[3 * idx + 2] = zd;
      rvalid[idx] = 1;
      ++rend_count;
    }
  if (cnt) {
    cnt->rend_valid += rend_count;
    cnt->obs_valid += n_obs;
  }
  if (rend_count == 0) {
    free(rp); free(rvalid);
    return 1; /* "windowed likelihood: empty rendered cloud" */
  }

  /* 162-186 (any number of noise entries) */
  double* const nbuf = (double*)malloc(sizeof(double) * 5 * n_noise);
  size_t* const slot_of = (size_t*)malloc(sizeof(size_t) * n_noise);
  double *coef = nbuf, *floor_term = nbuf + n_noise, *slot_scale = nbuf + 2 * n_noise,
         *slot_sigma = nbuf + 3 * n_noise, *slot_sum = nbuf + 4 * n_noise;
  size_t n_slots = 0;
  for (size_t e = 0; e < n_noise; ++e) {
    const double sigma2 = noise[e].sigma_noise * noise[e].sigma_noise;
    coef[e] = (1.0 - noise[e].p_outlier) / rend_count * pow(kTwoPi * sigma2, -1.5);
    floor_term[e] = noise[e].p_outlier / volume;
    out[e] = log_prefactor(&noise[e], sigma_max, prefactor);
    size_t s = 0;
    while (s < n_slots && slot_sigma[s] != noise[e].sigma_noise) ++s;
    if (s == n_slots) slot_sigma[n_slots++] = noise[e].sigma_noise;
    slot_of[e] = s;
  }
  for (size_t s = 0; s < n_slots; ++s)
    slot_scale[s] = 1.0 / (2.0 * slot_sigma[s] * slot_sigma[s]);

  double dist2[4096];
  const int wd = 2 * window + 1;
  double* d2 = (size_t)wd * wd <= 4096 ? dist2 : (double*)malloc(sizeof(double) * wd * wd);
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      const int32_t oi = oidx[(size_t)v * w + u];
      if (oi < 0) continue;
      const double* o = opts + 3 * (size_t)oi;
      size_t nd = 0;
      const int v_lo = v - window > 0 ? v - window : 0;
      const int v_hi = v + window < h - 1 ? v + window : h - 1;
      const int u_lo = u - window > 0 ? u - window : 0;
      const int u_hi = u + window < w - 1 ? u + window : w - 1;
      for (int rv = v_lo; rv <= v_hi; ++rv) {
        const size_t row = (size_t)rv * w;
        for (int ru = u_lo; ru <= u_hi; ++ru) {
          if (!rvalid[row + ru]) continue;
          const double* r = rp + 3 * (row + ru);
          const double dx = o[0] - r[0], dy = o[1] - r[1], dz = o[2] - r[2];
          /* squaredNorm: scalar 3-term redux */
          d2[nd++] = dx * dx + (dy * dy + dz * dz);
        }
      }
      if (cnt) cnt->pairs += nd;
      for (size_t s = 0; s < n_slots; ++s) {
        double acc = 0.0;
        for (size_t i = 0; i < nd; ++i) acc += exp(-d2[i] * slot_scale[s]);
        slot_sum[s] = acc;
      }
      for (size_t e = 0; e < n_noise; ++e)
        out[e] += log(floor_term[e] + coef[e] * slot_sum[slot_of[e]]);
    }
  }
  if (d2 != dist2) free(d2);
  free(nbuf); free(slot_of);
  free(rp); free(rvalid);
  return 0;
}

int orc_windowed_loglik_multi(const float* obs, const float* rend, const orc_intrinsics* k,
                              const orc_noise* noise, size_t n_noise, double volume,
                              double sigma_max, int window, int prefactor, double* out,
                              orc_counters* cnt) {
  if (k->width == 0 || k->height == 0) return 1;
  obs_cache oc;
  obs_cache_build(&oc, obs, k);
  const int rc = windowed_loglik_cached(&oc, rend, k, noise, n_noise, volume, sigma_max,
                                        window, prefactor, out, cnt);
  obs_cache_free(&oc);
  return rc;
}

/* geometry.cpp:54-70 */
void orc_depth_to_cloud(const float* depth, const orc_intrinsics* k, double* out, size_t* n) {
  const float sentinel = (float)k->far_m;
  size_t m = 0;
  for (uint32_t v = 0; v < k->height; ++v)
    for (uint32_t u = 0; u < k->width; ++u) {
      const float z = depth[(size_t)v * k->width + u];
      if (z >= sentinel) continue;
      const double zd = z;
      out[3 * m + 0] = (u - k->cx) * zd / k->fx;
      out[3 * m + 1] = (v - k->cy) * zd / k->fy;
      out[3 * m + 2] = zd;
      ++m;
    }
  *n = m;
}

/* sample_observation (likelihood.cpp:44-80): |cloud| draws from one Rng
 * stream -- with probability p_outlier a point uniform in the viewing
 * frustum (depth density ~ z^2), else a rendered point drawn with
 * replacement plus N(0, sigma) per axis -- reprojected with lround and kept
 * as the nearest fp32 depth per pixel.  Returns 1 for invalid noise or an
 * all-sentinel render (the reference throws). */
int orc_sample_observation(const float* rendered, const orc_intrinsics* k, double p_outlier,
                           double sigma, uint64_t st[5], float* out) {
  if (!(k->far_m > 0) || !(sigma > 0) || !(p_outlier >= 0 && p_outlier <= 1)) return 1;
  const size_t npx = (size_t)k->width * k->height;
  double* cloud = (double*)malloc(sizeof(double) * 3 * (npx ? npx : 1));
  size_t n = 0;
  orc_depth_to_cloud(rendered, k, cloud, &n);
  if (n == 0) {
    free(cloud);
    return 1;
  }
  const double near3 = k->near_m * k->near_m * k->near_m;
  const double far3 = k->far_m * k->far_m * k->far_m;
  const float sentinel = (float)k->far_m;
  for (size_t i = 0; i < npx; ++i) out[i] = sentinel;
  for (size_t i = 0; i < n; ++i) {
    double x, y, z;
    if (orc_rng_uniform(st) < p_outlier) {
      z = cbrt(near3 + orc_rng_uniform(st) * (far3 - near3));
      const double xl = (0.0 - k->cx) * z / k->fx, xh = (k->width - k->cx) * z / k->fx;
      x = xl + (xh - xl) * orc_rng_uniform(st);
      const double yl = (0.0 - k->cy) * z / k->fy, yh = (k->height - k->cy) * z / k->fy;
      y = yl + (yh - yl) * orc_rng_uniform(st);
    } else {
      const size_t j = (size_t)orc_rng_uniform_int(st, n);
      x = cloud[3 * j];
      y = cloud[3 * j + 1];
      z = cloud[3 * j + 2];
      x += 0.0 + sigma * orc_rng_normal(st);
      y += 0.0 + sigma * orc_rng_normal(st);
      z += 0.0 + sigma * orc_rng_normal(st);
    }
    if (z < k->near_m || z >= k->far_m) continue;
    const long u = lround(k->fx * x / z + k->cx);
    const long v = lround(k->fy * y / z + k->cy);
    if (u < 0 || u >= (long)k->width || v < 0 || v >= (long)k->height) continue;
    float* cell = out + (size_t)v * k->width + (size_t)u;
    const float zf = (float)z;
    if (zf < *cell) *cell = zf;
  }
  free(cloud);
  return 0;
}

/* likelihood.cpp:82-104 */
int orc_full_loglik_points(const double* op, size_t no, const double* rp, size_t nr,
                           const orc_noise* np, double volume, double sigma_max, int prefactor,
                           double* out) {
  if (!noise_ok(np, sigma_max) || nr == 0 || !(volume > 0)) return 1;
  const double sigma2 = np->sigma_noise * np->sigma_noise;
  const double inv_two_sigma2 = 1.0 / (2.0 * sigma2);
  const double norm3 = pow(kTwoPi * sigma2, -1.5);
  const double coef = (1.0 - np->p_outlier) / nr * norm3;
  const double outlier_floor = np->p_outlier / volume;
  double total = log_prefactor(np, sigma_max, prefactor);
  for (size_t i = 0; i < no; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < nr; ++j) {
      const double dx = op[3 * i] - rp[3 * j], dy = op[3 * i + 1] - rp[3 * j + 1],
                   dz = op[3 * i + 2] - rp[3 * j + 2];
      s += exp(-(dx * dx + (dy * dy + dz * dz)) * inv_two_sigma2);
    }
    total += log(outlier_floor + coef * s);
  }
  *out = total;
  return 0;
}

/* likelihood.cpp:82-104 over depth_to_cloud of both images */
int orc_full_loglik(const float* obs, const float* rend, const orc_intrinsics* k,
                    const orc_noise* np, double volume, double sigma_max, int prefactor,
                    double* out) {
  const size_t npx = (size_t)k->width * k->height;
  double* op = (double*)malloc(npx * 3 * sizeof(double));
  double* rp = (double*)malloc(npx * 3 * sizeof(double));
  size_t no = 0, nr = 0;
  orc_depth_to_cloud(obs, k, op, &no);
  orc_depth_to_cloud(rend, k, rp, &nr);
  const int rc = orc_full_loglik_points(op, no, rp, nr, np, volume, sigma_max, prefactor, out);
  free(op);
  free(rp);
  return rc;
}

/* ------------------------------------------------------- batched scoring */
typedef struct score_job {
  const orc_intrinsics* k;
  orc_pose w2c;
  obs_cache oc;
  double* obs_pts; /* window < 0: the observed cloud (depth_to_cloud) */
  size_t n_obs;
  const float* base;
  const double* verts;
  uint64_t nv;
  const uint32_t* tris;
  uint64_t nt;
  const orc_pose* poses;
  size_t n;
  const orc_noise* noise;
  size_t n_noise;
  double volume, sigma_max;
  int window, prefactor;
  double* scores;
  uint8_t* status;
  size_t next; /* work counter (parallel.hpp:36-46) */
  pthread_mutex_t mu;
  orc_counters cnt;
} score_job;

static void score_one(score_job* J, size_t i, float* img, orc_counters* c) {
  const size_t npx = (size_t)J->k->width * J->k->height;
  const float far_f = (float)J->k->far_m;
  /* compose_render: copy the base render (inference.cpp:102-109) */
  if (J->base)
    memcpy(img, J->base, npx * sizeof(float));
  else
    for (size_t p = 0; p < npx; ++p) img[p] = far_f;
  orc_pose m2c;
  orc_compose(&J->w2c, &J->poses[i], &m2c);
  orc_raster_mesh(img, 0, J->k, J->verts, J->nv, J->tris, J->nt, &m2c, 0, c);
  if (J->window < 0) {
    /* ModelConfig::windowed = false: observation_loglik_cached
       (inference.cpp:40-56) per entry -- -inf outside the noise support,
       the full likelihood of the two clouds otherwise; an empty render is
       flagged like the windowed path's */
    double* rp = (double*)malloc(npx * 3 * sizeof(double));
    size_t nr = 0;
    orc_depth_to_cloud(img, J->k, rp, &nr);
    J->status[i] = (uint8_t)(nr == 0);
    for (size_t e = 0; e < J->n_noise; ++e) {
      double v = -INFINITY;
      if (nr > 0 && noise_ok(&J->noise[e], J->sigma_max) &&
          orc_full_loglik_points(J->obs_pts, J->n_obs, rp, nr, &J->noise[e], J->volume,
                                 J->sigma_max, J->prefactor, &v) != 0)
        v = -INFINITY;
      J->scores[i * J->n_noise + e] = v;
    }
    free(rp);
    return;
  }
  const int rc =
      windowed_loglik_cached(&J->oc, img, J->k, J->noise, J->n_noise, J->volume,
                             J->sigma_max, J->window, J->prefactor,
                             J->scores + i * J->n_noise, c);
  J->status[i] = (uint8_t)(rc != 0);
  if (rc)
    for (size_t e = 0; e < J->n_noise; ++e) J->scores[i * J->n_noise + e] = -INFINITY;
}

static void* score_worker(void* arg) {
  score_job* J = (score_job*)arg;
  float* img = (float*)malloc((size_t)J->k->width * J->k->height * sizeof(float));
  orc_counters c;
  memset(&c, 0, sizeof(c));
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const size_t i = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (i >= J->n) break;
    score_one(J, i, img, &c);
  }
  free(img);
  pthread_mutex_lock(&J->mu);
  J->cnt.vertices += c.vertices;
  J->cnt.triangles += c.triangles;
  J->cnt.bbox_px += c.bbox_px;
  J->cnt.fragments += c.fragments;
  J->cnt.rend_valid += c.rend_valid;
  J->cnt.obs_valid += c.obs_valid;
  J->cnt.pairs += c.pairs;
  pthread_mutex_unlock(&J->mu);
  return 0;
}

int orc_score_poses(const orc_intrinsics* k, const orc_pose* camera, const float* obs,
                    const float* base, const double* verts, uint64_t nv,
                    const uint32_t* tris, uint64_t nt, const orc_pose* poses, size_t n,
                    const orc_noise* noise, size_t n_noise, double sigma_max, int window,
                    int prefactor, double* scores, uint8_t* status, int threads,
                    orc_counters* counters) {
  score_job J;
  memset(&J, 0, sizeof(J));
  J.k = k;
  orc_inverse(camera, &J.w2c);
  obs_cache_build(&J.oc, obs, k); /* once per observation (inference.cpp:158) */
  if (window < 0) {
    J.obs_pts = (double*)malloc((size_t)k->width * k->height * 3 * sizeof(double));
    orc_depth_to_cloud(obs, k, J.obs_pts, &J.n_obs);
  }
  J.base = base;
  J.verts = verts;
  J.nv = nv;
  J.tris = tris;
  J.nt = nt;
  J.poses = poses;
  J.n = n;
  J.noise = noise;
  J.n_noise = n_noise;
  J.volume = orc_visible_volume(k);
  J.sigma_max = sigma_max;
  J.window = window;
  J.prefactor = prefactor;
  J.scores = scores;
  J.status = status;
  pthread_mutex_init(&J.mu, 0);
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (threads < 1) threads = 1;
  if ((size_t)threads > n) threads = (int)(n ? n : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], 0, score_worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], 0);
  free(th);
  pthread_mutex_destroy(&J.mu);
  obs_cache_free(&J.oc);
  free(J.obs_pts);
  if (counters) *counters = J.cnt;
  return 0;
}

/* ------------------------------------------------------ stage reductions */
/* inference.cpp:16-23 */
double orc_logsumexp(const double* xs, size_t n) {
  double m = -INFINITY;
  for (size_t i = 0; i < n; ++i) m = xs[i] > m ? xs[i] : m; /* std::max(m, x) */
  if (!isfinite(m)) return -INFINITY;
  double acc = 0;
  for (size_t i = 0; i < n; ++i) acc += exp(xs[i] - m);
  return m + log(acc);
}

/* inference.cpp:315-330 */
int orc_normalize(const double* lt, size_t n, double* probs) {
  double max_log = -INFINITY;
  for (size_t i = 0; i < n; ++i) max_log = lt[i] > max_log ? lt[i] : max_log;
  if (!isfinite(max_log)) {
    for (size_t i = 0; i < n; ++i) probs[i] = 1.0 / n;
    return 1;
  }
  double total = 0;
  for (size_t i = 0; i < n; ++i) {
    probs[i] = exp(lt[i] - max_log);
    total += probs[i];
  }
  for (size_t i = 0; i < n; ++i) probs[i] /= total;
  return 0;
}

/* inference.cpp:345-353 */
size_t orc_sample_categorical(const double* probs, size_t n, uint64_t st[5]) {
  const double u = orc_rng_uniform(st);
  double acc = 0;
  for (size_t i = 0; i < n; ++i) {
    acc += probs[i];
    if (u < acc) return i;
  }
  return n - 1;
}

/* tracking.cpp:132-134: first index of the strict max */
size_t orc_argmax(const double* xs, size_t n) {
  size_t best = 0;
  for (size_t i = 1; i < n; ++i)
    if (xs[i] > xs[best]) best = i;
  return best;
}

/* ------------------------------------------------------------ pose grid */
/* tracking.cpp:27-37 */
double orc_lattice(double center, double extent, int n, int i) {
  if (n == 1) return center;
  return center - extent + 2.0 * extent * i / (n - 1);
}

uint64_t orc_grid_size(const orc_pose_grid* g) {
  const uint64_t nt = (uint64_t)g->count[0] * g->count[1] * g->count[2];
  return g->mode == 0 ? nt * g->n_rot : nt;
}

void orc_grid_pose(const orc_pose_grid* g, uint64_t index, orc_pose* out) {
  uint64_t ti, ri;
  if (g->mode == 0) {
    ti = index / g->n_rot;
    ri = index % g->n_rot;
  } else {
    ti = index;
    ri = index;
  }
  const uint32_t nz = g->count[2], ny = g->count[1];
  const int iz = (int)(ti % nz);
  const int iy = (int)((ti / nz) % ny);
  const int ix = (int)(ti / ((uint64_t)nz * ny));
  const quat c = {g->center.qw, g->center.qx, g->center.qy, g->center.qz};
  const double* r = g->rotations + 4 * ri;
  const quat d = {r[0], r[1], r[2], r[3]};
  const quat q = q_normalized(q_mul(c, d));
  out->qw = q.w;
  out->qx = q.x;
  out->qy = q.y;
  out->qz = q.z;
  out->tx = orc_lattice(g->center.tx, g->extent[0], (int)g->count[0], ix);
  out->ty = orc_lattice(g->center.ty, g->extent[1], (int)g->count[1], iy);
  out->tz = orc_lattice(g->center.tz, g->extent[2], (int)g->count[2], iz);
}
