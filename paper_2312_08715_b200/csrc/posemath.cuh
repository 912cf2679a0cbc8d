// posemath.cuh -- fp64 pose arithmetic shared by the sm_100a kernels.
// Restates geometry.cpp:19-31 (compose / inverse) and Eigen's quaternion
// formulas in Eigen's scalar evaluation order; every TU that includes this
// is compiled with --fmad=false so results are bit-identical to the oracle.
#pragma once

#include "b3d_kernels.cuh"

namespace b3d200 {
namespace pm {

struct Q {
  double w, x, y, z;
};

// Eigen QuaternionBase::normalized(), scalar 4-term redux (x2+y2)+(z2+w2).
__device__ __forceinline__ Q q_normalized(Q q) {
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

// Eigen generic quat_product.
__device__ __forceinline__ Q q_mul(const Q& a, const Q& b) {
  Q r;
  r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  r.y = a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z;
  r.z = a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x;
  return r;
}

// Eigen _transformVector: uv = q.vec x v; uv += uv; v + w*uv + q.vec x uv.
__device__ __forceinline__ void q_rotate(const Q& q, const double v[3], double o[3]) {
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

// tracking.cpp:27-37
__device__ __forceinline__ double lattice(double c, double e, int n, int i) {
  if (n == 1) return c;
  return c - e + 2.0 * e * i / (n - 1);
}

// scene_graph.cpp:97-121 for the cell centre (inference.cpp:126-137,
// Interval::center inference.hpp:18) of contact cell (ix, iy, it).
__device__ __forceinline__ void contact_pose(const KGrid& g, long long index, KPose& out) {
  const KContact& c = g.contact;
  const int nt = g.count[2], ny = g.count[1], nx = g.count[0];
  const int it = (int)(index % nt);
  const int iy = (int)((index / nt) % ny);
  const int ix = (int)(index / ((long long)nt * ny));
  const double dx = 0.5 * ((c.dx_lo + c.dx_w * ix / nx) + (c.dx_lo + c.dx_w * (ix + 1) / nx));
  const double dy = 0.5 * ((c.dy_lo + c.dy_w * iy / ny) + (c.dy_lo + c.dy_w * (iy + 1) / ny));
  const double cs = c.spin[2 * it], sn = c.spin[2 * it + 1];
  const Q spin{cs, sn * 0.0, sn * 0.0, sn * 1.0};  // AngleAxis(dtheta, UnitZ)
  const double cx = -c.table_w / 2, cy = -c.table_h / 2, cz = 0.0;
  const double bt[3] = {cx + (dx - c.lo[0]), cy + (dy - c.lo[1]), cz + -c.lo[2]};
  const double pv[3] = {cx + (dx + c.w / 2), cy + (dy + c.h / 2), cz + 0.0};
  const Q q = q_normalized(q_mul(spin, Q{c.face_q[0], c.face_q[1], c.face_q[2], c.face_q[3]}));
  const double rel[3] = {bt[0] - pv[0], bt[1] - pv[1], bt[2] - pv[2]};
  double r[3];
  q_rotate(spin, rel, r);
  out.qw = q.w;
  out.qx = q.x;
  out.qy = q.y;
  out.qz = q.z;
  out.tx = r[0] + pv[0];
  out.ty = r[1] + pv[1];
  out.tz = r[2] + pv[2];
}

__device__ __forceinline__ void grid_pose(const KGrid& g, long long index, KPose& out) {
  if (g.mode == 2) {
    contact_pose(g, index, out);
    return;
  }
  long long ti, ri;
  if (g.mode == 0) {
    ti = index / g.n_rot;
    ri = index % g.n_rot;
  } else {
    ti = index;
    ri = index;
  }
  const KPose c = g.center_dev ? *g.center_dev : g.center;
  const int iz = (int)(ti % g.count[2]);
  const int iy = (int)((ti / g.count[2]) % g.count[1]);
  const int ix = (int)(ti / ((long long)g.count[2] * g.count[1]));
  const double* r = g.rotations + 4 * ri;
  const Q q = q_normalized(q_mul(Q{c.qw, c.qx, c.qy, c.qz}, Q{r[0], r[1], r[2], r[3]}));
  out.qw = q.w;
  out.qx = q.x;
  out.qy = q.y;
  out.qz = q.z;
  out.tx = lattice(c.tx, g.extent[0], g.count[0], ix);
  out.ty = lattice(c.ty, g.extent[1], g.count[1], iy);
  out.tz = lattice(c.tz, g.extent[2], g.count[2], iz);
}

// geometry.cpp:26-31 inverse(p): q' = normalized(conj q), t' = -(q' t)
// (same operation order as the host's pose_inverse in b3d_capi.cpp).
__device__ __forceinline__ KPose pose_inverse(const KPose& p) {
  const Q q = q_normalized(Q{p.qw, -p.qx, -p.qy, -p.qz});
  const double v[3] = {p.tx, p.ty, p.tz};
  double r[3];
  q_rotate(q, v, r);
  return KPose{q.w, q.x, q.y, q.z, -r[0], -r[1], -r[2]};
}

// geometry.cpp:19-24 compose(a, b) -> rotation matrix (Eigen
// toRotationMatrix) + translation.  R row-major.
__device__ __forceinline__ void pose_to_rt(const KPose& a, const KPose& b, double R[9], double t[3]) {
  const Q qa{a.qw, a.qx, a.qy, a.qz};
  const Q q = q_normalized(q_mul(qa, Q{b.qw, b.qx, b.qy, b.qz}));
  const double bt[3] = {b.tx, b.ty, b.tz};
  double r[3];
  q_rotate(qa, bt, r);
  t[0] = r[0] + a.tx;
  t[1] = r[1] + a.ty;
  t[2] = r[2] + a.tz;
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  R[0] = 1.0 - (tyy + tzz);
  R[1] = txy - twz;
  R[2] = txz + twy;
  R[3] = txy + twz;
  R[4] = 1.0 - (txx + tzz);
  R[5] = tyz - twx;
  R[6] = txz - twy;
  R[7] = tyz + twx;
  R[8] = 1.0 - (txx + tyy);
}

}  // namespace pm
}  // namespace b3d200
