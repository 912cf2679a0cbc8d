// render_score.cuh -- fused per-hypothesis rasterizer + windowed likelihood
// for sm_100a.  One CTA owns one hypothesis at a time (persistent over a
// strided hypothesis range):
//
//   A  pose     : hypothesis pose (array or on-device grid), compose with
//                 inverse(camera), rotation matrix              (fp64, no FMA)
//   B  vertices : R*v + t, project to (u, v, 1/z) into shared memory, and
//                 the screen-space region the object can touch  (fp64)
//   C  raster   : thread per triangle, reference edge functions + top-left
//                 rule, perspective 1/z, strict-less z-test via a shared
//                 memory atomicMin on fp32 depth bits (or on the 64-bit key
//                 (depth bits, draw index) when ids are requested)
//   D  score    : |y| count, then thread per pixel of the window-dilated
//                 region: sum_window exp(-d^2 / 2 sigma^2) over valid
//                 rendered pixels, log(floor + coef*S), fp64 block reduction
//
// The rendered image never leaves the SM in score mode.  The arithmetic of
// A-C follows renderer.cpp:61-151 / geometry.cpp:19-31 operation by
// operation (this TU is compiled with --fmad=false), so depth and ids are
// bit-identical to the CPU oracle.  D follows likelihood.cpp:128-220 with
// fp32 distances/exp/log and fp64 accumulation (north_star: 1e-4 relative).
#pragma once

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>
#include <type_traits>


#include "b3d_kernels.cuh"
#include "posemath.cuh"

#ifndef B3D_MINB
#define B3D_MINB 2
#endif
#ifndef B3D_L2_PREFETCH
#define B3D_L2_PREFETCH 1
#endif

namespace b3d200 {

namespace {

using namespace pm;


struct SV {
  double u, v, iz;
};

// renderer.cpp:26-59.  EdgeFn::eval is sign*(cdx*(py-oy) - cdy*(px-ox))
// with (cdx, cdy) = hi - lo of the canonically ordered endpoints.  Since
// sign*cdx == b.u - a.u bitwise (round-to-nearest is antisymmetric) and
// sign*(X - Y) == (sign*X') - (sign*Y') with X' = cdx*A, the edge value is
// (b.u-a.u)*(py-oy) - (b.v-a.v)*(px-ox) with the canonical origin o: the same
// bits except possibly the sign of an exact zero, which neither the fill
// rule (e > 0 / e < 0 / tie) nor the 1/z test (inv_z <= 0) can observe.
struct Edge {
  double ox, oy, dx, dy;
};

__device__ __forceinline__ Edge make_edge(const SV& a, const SV& b) {
  const bool canonical = a.u < b.u || (a.u == b.u && a.v < b.v);
  Edge e;
  e.ox = canonical ? a.u : b.u;
  e.oy = canonical ? a.v : b.v;
  e.dx = b.u - a.u;
  e.dy = b.v - a.v;
  return e;
}

__device__ __forceinline__ bool covers(const Edge& e, double v) {
  if (v > 0) return true;
  if (v < 0) return false;
  return e.dy < 0 || (e.dy == 0 && e.dx > 0);
}

template <bool kIds>
struct KeyT;
template <>
struct KeyT<false> {
  using T = unsigned int;
};
template <>
struct KeyT<true> {
  using T = unsigned long long;
};

// Strict-less z-test (renderer.cpp:99) as an atomic min on the key.
__device__ __forceinline__ void zmin(unsigned int* p, unsigned int v) {
  if (v < *p) atomicMin(p, v);
}
__device__ __forceinline__ void zmin(unsigned long long* p, unsigned long long v) {
  if (v < *p) atomicMin(p, v);
}

// Screen region of one hypothesis: interior [u0,u1]x[v0,v1] (clipped to the
// image) that the object can touch, stored with a background halo of `pad`
// pixels so the likelihood's window taps never need bounds checks.
// Buffer index of pixel (u, v): (v - oy) * rw + (u - ox).
struct Region {
  int u0, v0, u1, v1, ox, oy, rw, rh;
};

// renderer.cpp:63-102 for a triangle whose integer pixel bbox is known.
template <bool kIds>
__device__ __forceinline__ void raster_tri_box(const KParams& p, typename KeyT<kIds>::T* zb,
                                               const Region& rg, SV a, SV b, SV c, int u_min,
                                               int u_max, int v_min, int v_max, uint32_t draw) {
  double area2 = (b.u - a.u) * (c.v - a.v) - (b.v - a.v) * (c.u - a.u);
  if (area2 == 0) return;
  if (area2 < 0) {
    const SV t = b;
    b = c;
    c = t;
    area2 = -area2;
  }
  const Edge ab = make_edge(a, b);
  const Edge bc = make_edge(b, c);
  const Edge ca = make_edge(c, a);
  const double inv_area2 = __drcp_rn(area2);
  for (int pv = v_min; pv <= v_max; ++pv) {
    const double py = pv;
    const double r_ab = ab.dx * (py - ab.oy);
    const double r_bc = bc.dx * (py - bc.oy);
    const double r_ca = ca.dx * (py - ca.oy);
    typename KeyT<kIds>::T* row = zb + (pv - rg.oy) * rg.rw - rg.ox;
    for (int pu = u_min; pu <= u_max; ++pu) {
      const double px = pu;
      const double e_ab = r_ab - ab.dy * (px - ab.ox);
      const double e_bc = r_bc - bc.dy * (px - bc.ox);
      const double e_ca = r_ca - ca.dy * (px - ca.ox);
      if (!covers(ab, e_ab) || !covers(bc, e_bc) || !covers(ca, e_ca)) continue;
      const double inv_z = (e_bc * a.iz + e_ca * b.iz + e_ab * c.iz) * inv_area2;
      if (inv_z <= 0) continue;
      const double z = __drcp_rn(inv_z);
      if (z < p.near_lim || z > p.far_m) continue;
      const float zf = __double2float_rn(z);
      if (!(zf < p.far_f)) continue;
      if (kIds) {
        const unsigned long long key =
            ((unsigned long long)__float_as_uint(zf) << 32) | (unsigned long long)draw;
        zmin((unsigned long long*)(row + pu), key);
      } else {
        zmin((unsigned int*)(row + pu), __float_as_uint(zf));
      }
    }
  }
}

// renderer.cpp:61-103 -- one screen triangle into the region z-buffer
// (clipped path: the bbox comes from the fp64 vertex coordinates).  The
// bounds reproduce static_cast<int> on x86-64 exactly: a max u or v beyond
// the int range converts to INT_MIN there and empties the bbox.
template <bool kIds>
__device__ __forceinline__ void raster_tri(const KParams& p, typename KeyT<kIds>::T* zb,
                                           const Region& rg, SV a, SV b, SV c, uint32_t draw) {
  const double mnu = fmin(fmin(a.u, b.u), c.u), mxu = fmax(fmax(a.u, b.u), c.u);
  const double mnv = fmin(fmin(a.v, b.v), c.v), mxv = fmax(fmax(a.v, b.v), c.v);
  if (!(mxu < 2147483648.0) || !(mxv < 2147483648.0)) return;
  const double cu0 = fmax(ceil(mnu), 0.0), fu1 = fmin(floor(mxu), (double)(p.W - 1));
  const double cv0 = fmax(ceil(mnv), 0.0), fv1 = fmin(floor(mxv), (double)(p.H - 1));
  if (cu0 > fu1 || cv0 > fv1) return;
  raster_tri_box<kIds>(p, zb, rg, a, b, c, (int)cu0, (int)fu1, (int)cv0, (int)fv1, draw);
}

__device__ __forceinline__ SV project(const KParams& p, double x, double y, double z) {
  const double iz = __drcp_rn(z);
  SV s;
  s.u = p.fx * x * iz + p.cx;
  s.v = p.fy * y * iz + p.cy;
  s.iz = iz;
  return s;
}

__device__ __forceinline__ void cam_vertex(const double* R, const double* t, const double* v,
                                           double o[3]) {
  // Eigen 3x3 * 3x1 lazy product, scalar redux a0 + (a1 + a2), then + t
  o[0] = (R[0] * v[0] + (R[1] * v[1] + R[2] * v[2])) + t[0];
  o[1] = (R[3] * v[0] + (R[4] * v[1] + R[5] * v[2])) + t[1];
  o[2] = (R[6] * v[0] + (R[7] * v[1] + R[8] * v[2])) + t[2];
}

// Packed per-vertex integer bbox data (screen bounds of one vertex), used to
// reject triangles and size their pixel bbox with integer min/max:
//   x = ceil(u) clamped to [0, W], y = floor(u) clamped to [-1, W-1] or
//   kOvf when u >= 2^31 (the reference's static_cast<int> then yields INT_MIN
//   and an empty bbox, renderer.cpp:70-76), z/w the same for v;
//   x = kClipV marks a vertex in front of z = near (clipped path).
constexpr short kOvf = 32767;
constexpr short kClipV = -32768;

__device__ __forceinline__ short4 vertex_bbox(const KParams& p, double u, double v) {
  // fp64 -> int conversions with directed rounding saturate (PTX cvt), so
  // ceil/floor + clamp need no fp64 min/max; |u|, |v| >= 2^31 behave like the
  // clamped fp64 forms (upload rejects non-finite vertices)
  short4 r;
  r.x = (short)min(max(__double2int_ru(u), 0), p.W);
  r.y = u >= 2147483648.0 ? kOvf : (short)min(max(__double2int_rd(u), -1), p.W - 1);
  r.z = (short)min(max(__double2int_ru(v), 0), p.H);
  r.w = v >= 2147483648.0 ? kOvf : (short)min(max(__double2int_rd(v), -1), p.H - 1);
  return r;
}

// Per-warp queues of triangles that survive the cheap tests (non-empty
// integer bbox, non-zero area, not culled), one ring per tile class
// (bbox <= 2x2 and <= 3x3).  Entry: vertex ids after the orientation swap
// (renderer.cpp:63-69) + triangle index, and the packed bbox
// u_min | (bw-1) << 14 | v_min << 16 | (bh-1) << 30.
// B3D_PHASE_CLOCK=1 (diagnostic builds only, scripts/phase_probe.py): thread 0
// of CTAs < 256 stamps %globaltimer at the phase boundaries of its latest
// hypothesis into g_phase (read back by b3d_debug_phase_clock, rs_cam.cu).
#if B3D_PHASE_CLOCK
__device__ long long g_phase[256][8];
#define B3D_PCLK(i)                                                       \
  do {                                                                    \
    if (threadIdx.x == 0 && blockIdx.x < 256) {                           \
      long long t_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
      g_phase[blockIdx.x][i] = t_;                                        \
    }                                                                     \
  } while (0)
// one reader per translation unit (each holds its own g_phase)
#define B3D_PHASE_READER(NAME)                                                       \
  extern "C" __attribute__((visibility("default"))) int NAME(long long* out) {       \
    return (int)cudaMemcpyFromSymbol(out, b3d200::g_phase, sizeof(b3d200::g_phase)); \
  }
#else
#define B3D_PCLK(i) \
  do {              \
  } while (0)
#define B3D_PHASE_READER(NAME)
#endif
constexpr int kRing = 64;
struct WarpQ {
  uint4 tri[2][kRing];
  uint32_t box[2][kRing];
};

// Coverage of one edge over a KxK pixel tile at (u0, v0): the reference's
// edge value dx*(py - oy) - dy*(px - ox) (renderer.cpp:32-34, canonical
// origin) factored into K row products and K column products -- the same
// two fp64 products and difference per pixel, so bitwise the same values --
// and the top-left rule (renderer.cpp:39-43).  Bit 3*j + i = pixel
// (u0 + i, v0 + j).
template <int K>
__device__ __forceinline__ uint32_t tile_edge_mask(double2 a, double2 b, bool canon, bool tie,
                                                   int u0, int v0) {
  const double ox = canon ? a.x : b.x, oy = canon ? a.y : b.y;
  const double dx = b.x - a.x, dy = b.y - a.y;
  double A[K], B[K];
#pragma unroll
  for (int j = 0; j < K; ++j) A[j] = dx * ((double)(v0 + j) - oy);
#pragma unroll
  for (int i = 0; i < K; ++i) B[i] = dy * ((double)(u0 + i) - ox);
  // e > 0 || (tie && e == 0)  ==  e > thr: no double lies strictly between
  // -denorm_min and 0, and fp64 compares do not flush denormals
  const double thr = tie ? -4.9406564584124654e-324 : 0.0;
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (A[j] - B[i] > thr) m |= 1u << (K * j + i);
  return m;
}

// Edge flags: bit e = canonical origin is the edge's first vertex
// (renderer.cpp:47), bit 3+e = pixels exactly on the edge are covered
// (top-left rule, renderer.cpp:39-43).
__device__ __forceinline__ int edge_flags(const SV& a, const SV& b, int e) {
  const bool canonical = a.u < b.u || (a.u == b.u && a.v < b.v);
  const double dx = b.u - a.u, dy = b.v - a.v;
  const bool tie = dy < 0 || (dy == 0 && dx > 0);
  return ((int)canonical << e) | ((int)tie << (3 + e));
}

// Edge value of the directed edge (a -> b) at (px, py) with the canonical
// origin selected by `canon` -- bitwise the reference's EdgeFn::eval.
__device__ __forceinline__ double edge_at(double2 a, double2 b, bool canon, double px,
                                          double py) {
  const double ox = canon ? a.x : b.x, oy = canon ? a.y : b.y;
  return (b.x - a.x) * (py - oy) - (b.y - a.y) * (px - ox);
}

__device__ __forceinline__ bool edge_covers(double e, bool tie) {
  return e > 0 || (e == 0 && tie);
}

// renderer.cpp:124-150 for a triangle with a vertex in front of z = near.
template <bool kIds>
__device__ void raster_clipped(const KParams& p, typename KeyT<kIds>::T* zb,
                               const Region& rg, const double* R, const double* t,
                               uint32_t i0, uint32_t i1, uint32_t i2, uint32_t draw) {
  double v[3][3];
  cam_vertex(R, t, p.verts + 3 * (size_t)i0, v[0]);
  cam_vertex(R, t, p.verts + 3 * (size_t)i1, v[1]);
  cam_vertex(R, t, p.verts + 3 * (size_t)i2, v[2]);
  double poly[4][3];
  int n = 0;
  for (int i = 0; i < 3; ++i) {
    const double* cur = v[i];
    const double* nxt = v[(i + 1) % 3];
    const bool cin = cur[2] >= p.near_m;
    const bool nin = nxt[2] >= p.near_m;
    if (cin) {
      poly[n][0] = cur[0];
      poly[n][1] = cur[1];
      poly[n][2] = cur[2];
      ++n;
    }
    if (cin != nin) {
      const double s = (p.near_m - cur[2]) / (nxt[2] - cur[2]);
      for (int k = 0; k < 3; ++k) poly[n][k] = cur[k] + s * (nxt[k] - cur[k]);
      ++n;
    }
  }
  if (n < 3) return;
  const SV s0 = project(p, poly[0][0], poly[0][1], poly[0][2]);
  SV prev = project(p, poly[1][0], poly[1][1], poly[1][2]);
  for (int i = 2; i < n; ++i) {
    const SV cur = project(p, poly[i][0], poly[i][1], poly[i][2]);
    raster_tri<kIds>(p, zb, rg, s0, prev, cur, draw);
    prev = cur;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#ifndef B3D_TAP_ROOT
#define B3D_TAP_ROOT 1
#endif
#ifndef B3D_EX2_FTZ
#define B3D_EX2_FTZ 1
#endif
// One window tap's exp2.  exp2f keeps subnormal results (a compare and two
// predicated multiplies around MUFU.EX2 per tap); a tap below 2^-126 adds
// nothing an fp32 window sum or the log(floor + coef*S) term can register
// (the fp64 image path takes the settings where the floor vanishes, §5.5),
// so the flush-to-zero form is one instruction.
__device__ __forceinline__ float ex2_tap(float x) {
#if B3D_EX2_FTZ
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return exp2f(x);
#endif
}

// sum over the (2w+1)^2 window of exp(-|o - r|^2 / (2 sigma^2)) per distinct
// sigma (likelihood.cpp:198-214) in fp32: rendered points back-projected on
// the fly from the region buffer, exp as ex2 with the scale pre-multiplied
// by log2(e).  Background taps give d^2 >= (far - z_obs)^2 and an exact 0.
template <bool kIds, int kW, bool kS1>
__device__ __forceinline__ void window_sums_w(const KParams& p,
                                              const typename KeyT<kIds>::T* zb,
                                              const Region& rg, int u, int v, float4 o,
                                              float S[kMaxSlots]) {
#pragma unroll
  for (int s = 0; s < kMaxSlots; ++s) S[s] = 0.f;
  const float cu0 = ((float)(u - kW) - p.fcx) * p.inv_fx;
  const float cv0 = ((float)(v - kW) - p.fcy) * p.inv_fy;
  const typename KeyT<kIds>::T* row0 = zb + (v - kW - rg.oy) * rg.rw + (u - kW - rg.ox);
#if B3D_TAP_ROOT
  if constexpr (kS1) {
    // one sigma: scale both points by k = sqrt(log2(e)/(2 sigma^2)) so a tap
    // is three FFMAs, the squared norm and one ex2 (no dz subtraction and no
    // scale multiply per tap); the base-image sums use the same form
    const float k = p.lik.slot_root[0];
    const float kox = k * o.x, koy = k * o.y, koz = k * o.z;
#pragma unroll
    for (int j = 0; j < 2 * kW + 1; ++j) {
      const float kcv = k * (cv0 + (float)j * p.inv_fy);
#pragma unroll
      for (int c = 0; c < 2 * kW + 1; ++c) {
        const typename KeyT<kIds>::T key = row0[j * rg.rw + c];
        const float z = __uint_as_float(
            kIds ? (unsigned int)((unsigned long long)key >> 32) : (unsigned int)key);
        const float kcu = k * (cu0 + (float)c * p.inv_fx);
        const float dx = __fmaf_rn(-kcu, z, kox);
        const float dy = __fmaf_rn(-kcv, z, koy);
        const float dz = __fmaf_rn(-k, z, koz);
        S[0] += ex2_tap(-__fmaf_rn(dx, dx, __fmaf_rn(dy, dy, dz * dz)));
      }
    }
    return;
  }
#endif
#pragma unroll
  for (int j = 0; j < 2 * kW + 1; ++j) {
    const float cv = cv0 + (float)j * p.inv_fy;
#pragma unroll
    for (int k = 0; k < 2 * kW + 1; ++k) {
      const typename KeyT<kIds>::T key = row0[j * rg.rw + k];
      const float z = __uint_as_float(
          kIds ? (unsigned int)((unsigned long long)key >> 32) : (unsigned int)key);
      const float cu = cu0 + (float)k * p.inv_fx;
      const float dx = __fmaf_rn(-cu, z, o.x);
      const float dy = __fmaf_rn(-cv, z, o.y);
      const float dz = o.z - z;
      const float d2 = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, dz * dz));
#pragma unroll
      for (int s = 0; s < (kS1 ? 1 : kMaxSlots); ++s)
        if (kS1 || s < p.lik.n_slots) S[s] += ex2_tap(-d2 * p.lik.slot_scale[s]);
    }
  }
}

template <bool kIds, bool kS1>
__device__ __forceinline__ void window_sums_any(const KParams& p,
                                                const typename KeyT<kIds>::T* zb,
                                                const Region& rg, int u, int v, float4 o,
                                                float S[kMaxSlots]) {
#pragma unroll
  for (int s = 0; s < kMaxSlots; ++s) S[s] = 0.f;
  const int w = p.lik.window;
#if B3D_TAP_ROOT
  if constexpr (kS1) {  // the single-sigma form of window_sums_w
    const float k = p.lik.slot_root[0];
    const float kox = k * o.x, koy = k * o.y, koz = k * o.z;
    for (int rv = v - w; rv <= v + w; ++rv) {
      const float kcv = k * (((float)rv - p.fcy) * p.inv_fy);
      for (int ru = u - w; ru <= u + w; ++ru) {
        const typename KeyT<kIds>::T key = zb[(rv - rg.oy) * rg.rw + (ru - rg.ox)];
        const float z = __uint_as_float(
            kIds ? (unsigned int)((unsigned long long)key >> 32) : (unsigned int)key);
        const float kcu = k * (((float)ru - p.fcx) * p.inv_fx);
        const float dx = __fmaf_rn(-kcu, z, kox);
        const float dy = __fmaf_rn(-kcv, z, koy);
        const float dz = __fmaf_rn(-k, z, koz);
        S[0] += ex2_tap(-__fmaf_rn(dx, dx, __fmaf_rn(dy, dy, dz * dz)));
      }
    }
    return;
  }
#endif
  for (int rv = v - w; rv <= v + w; ++rv) {
    const float cv = ((float)rv - p.fcy) * p.inv_fy;
    for (int ru = u - w; ru <= u + w; ++ru) {
      const typename KeyT<kIds>::T key = zb[(rv - rg.oy) * rg.rw + (ru - rg.ox)];
      const float z = __uint_as_float(
          kIds ? (unsigned int)((unsigned long long)key >> 32) : (unsigned int)key);
      const float cu = ((float)ru - p.fcx) * p.inv_fx;
      const float dx = __fmaf_rn(-cu, z, o.x);
      const float dy = __fmaf_rn(-cv, z, o.y);
      const float dz = o.z - z;
      const float d2 = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, dz * dz));
#pragma unroll
      for (int s = 0; s < (kS1 ? 1 : kMaxSlots); ++s)
        if (kS1 || s < p.lik.n_slots) S[s] += ex2_tap(-d2 * p.lik.slot_scale[s]);
    }
  }
}

// kWin >= 0: the launch's window radius as a compile-time constant (one
// unrolled tap loop per kernel instantiation); kWin < 0: any radius.  kS1:
// a single distinct sigma.
template <bool kIds, int kWin, bool kS1>
__device__ __forceinline__ void window_sums(const KParams& p, const typename KeyT<kIds>::T* zb,
                                            const Region& rg, int u, int v, float4 o,
                                            float S[kMaxSlots]) {
  if constexpr (kWin >= 0)
    window_sums_w<kIds, kWin, kS1>(p, zb, rg, u, v, o, S);
  else
    window_sums_any<kIds, kS1>(p, zb, rg, u, v, o, S);
}

template <bool kIds>
__device__ __forceinline__ void window_sums_rt(const KParams& p, const typename KeyT<kIds>::T* zb,
                                               const Region& rg, int u, int v, float4 o,
                                               float S[kMaxSlots]) {
  // the score kernels take their single-sigma form when n_noise == 1
  // (pick_kernel): the same taps here, so S and S_base agree bitwise
  if (p.lik.n_noise == 1) {
    switch (p.lik.window) {
      case 0: window_sums_w<kIds, 0, true>(p, zb, rg, u, v, o, S); break;
      case 1: window_sums_w<kIds, 1, true>(p, zb, rg, u, v, o, S); break;
      case 2: window_sums_w<kIds, 2, true>(p, zb, rg, u, v, o, S); break;
      case 3: window_sums_w<kIds, 3, true>(p, zb, rg, u, v, o, S); break;
      default: window_sums_any<kIds, true>(p, zb, rg, u, v, o, S); break;
    }
    return;
  }
  switch (p.lik.window) {
    case 0: window_sums_w<kIds, 0, false>(p, zb, rg, u, v, o, S); break;
    case 1: window_sums_w<kIds, 1, false>(p, zb, rg, u, v, o, S); break;
    case 2: window_sums_w<kIds, 2, false>(p, zb, rg, u, v, o, S); break;
    case 3: window_sums_w<kIds, 3, false>(p, zb, rg, u, v, o, S); break;
    default: window_sums_any<kIds, false>(p, zb, rg, u, v, o, S); break;
  }
}

// Clenshaw evaluation of a Chebyshev series on [lo, hi].
__device__ __forceinline__ double cheb_eval(const double* c, double x, double lo, double hi) {
  const double t = (2.0 * x - (lo + hi)) / (hi - lo);
  double b1 = 0.0, b2 = 0.0;
  for (int j = kCheb - 1; j >= 1; --j) {
    const double b0 = 2.0 * t * b1 - b2 + c[j];
    b2 = b1;
    b1 = b0;
  }
  return t * b1 - b2 + 0.5 * c[0];
}

constexpr float kBgDepth = 1e30f;
#ifndef B3D_THREADS
#define B3D_THREADS 384
#endif
constexpr int kThreads = B3D_THREADS;
constexpr int kWarps = kThreads / 32;

}  // namespace

// Triangles whose bbox exceeds kHugeBox pixels (a table face filling the
// image): the whole warp sweeps the bbox of lane `src`'s triangle (vertex
// ids already in positive-area order), one pixel per lane per step, with the
// reference's per-pixel arithmetic (renderer.cpp:78-102).
constexpr int kHugeBox = 64;


template <bool kIds, typename VS, typename Key>
__device__ __forceinline__ void sweep_huge(const KParams& p, Key* const zb, const Region& rg,
                                           const VS& vs, int src, uint4 tr, uint32_t box,
                                           uint32_t box2, int lane) {
  const uint32_t ia = __shfl_sync(0xffffffffu, tr.x, src);
  const uint32_t ib = __shfl_sync(0xffffffffu, tr.y, src);
  const uint32_t ic = __shfl_sync(0xffffffffu, tr.z, src);
  const uint32_t draw = p.draw_base + __shfl_sync(0xffffffffu, tr.w, src);
  const uint32_t b1 = __shfl_sync(0xffffffffu, box, src);
  const uint32_t b2 = __shfl_sync(0xffffffffu, box2, src);
  const int u0 = b1 & 0xffff, v0 = b1 >> 16;
  const int bw = (int)(b2 & 0xffff) - u0 + 1, bh = (int)(b2 >> 16) - v0 + 1;
  const double2 A = vs.uv(ia), B = vs.uv(ib), C = vs.uv(ic);
  const double iza = vs.iz(ia), izb = vs.iz(ib), izc = vs.iz(ic);
  const SV a{A.x, A.y, 0.0}, b{B.x, B.y, 0.0}, c{C.x, C.y, 0.0};
  const int fl = edge_flags(a, b, 0) | edge_flags(b, c, 1) | edge_flags(c, a, 2);
  const double ia2 = __drcp_rn((B.x - A.x) * (C.y - A.y) - (B.y - A.y) * (C.x - A.x));
  for (int row = 0; row < bh; ++row) {
    const int pv = v0 + row;
    const double py = pv;
    for (int col = lane; col < bw; col += 32) {
      const int pu = u0 + col;
      const double px = pu;
      const double e_ab = edge_at(A, B, fl & 1, px, py);
      const double e_bc = edge_at(B, C, fl & 2, px, py);
      const double e_ca = edge_at(C, A, fl & 4, px, py);
      if (!edge_covers(e_ab, fl & 8) || !edge_covers(e_bc, fl & 16) || !edge_covers(e_ca, fl & 32))
        continue;
      const double inv_z = (e_bc * iza + e_ca * izb + e_ab * izc) * ia2;
      if (!(inv_z > 0)) continue;
      const double z = __drcp_rn(inv_z);
      if (z < p.near_lim || z > p.far_m) continue;
      const float zf = __double2float_rn(z);
      if (!(zf < p.far_f)) continue;
      Key* cell = zb + (pv - rg.oy) * rg.rw + (pu - rg.ox);
      if (kIds)
        zmin((unsigned long long*)cell,
             ((unsigned long long)__float_as_uint(zf) << 32) | (unsigned long long)draw);
      else
        zmin((unsigned int*)cell, __float_as_uint(zf));
    }
  }
}

// Camera mode: triangles whose bbox exceeds the 3x3 tile classes (table faces
// under a camera hypothesis cover much of the image) are collected per CTA
// and rasterized after the warps' passes by all kThreads threads over the
// concatenation of their bbox pixels -- not by the one lane (per-pixel loop)
// or warp (sweep) that met them, which serialises a single hypothesis when a
// small batch leaves one CTA per SM.  Per-pixel arithmetic as sweep_huge
// (renderer.cpp:78-102).  Overflow beyond kMaxHuge keeps the per-lane / per-
// warp paths.  Render-mode kernels use it too (a base scene or b3d_render is
// one hypothesis in one CTA); object-mode score kernels do not (the table is
// in the pre-rendered base scene there).
constexpr int kMaxHuge = 32;
template <int kCap>
struct HugeListT {
  uint4 tri[kCap];      // vertex ids (positive-area order), triangle index
  uint2 box[kCap];      // (u_min | v_min << 16, u_max | v_max << 16)
  double ia2[kCap];     // 1 / area2
  int fl[kCap];         // edge_flags
  int pre[kCap + 1];    // exclusive prefix of bbox pixel counts
  // entry count, double-buffered by hypothesis parity: thread 0 resets the
  // next hypothesis's count while slow warps may still read this one's
  // (render mode has no barrier after the read)
  int n[2];
};

// Warp 0: per-entry edge flags, 1/area2 and the pixel prefix (nh <= 32).
template <typename VS, int kCap>
__device__ __forceinline__ void huge_prepare(HugeListT<kCap>* hl, const VS& vs, int nh, int lane) {
  int area = 0;
  if (lane < nh) {
    const uint4 tr = hl->tri[lane];
    const uint2 bx = hl->box[lane];
    const double2 A = vs.uv(tr.x), B = vs.uv(tr.y), C = vs.uv(tr.z);
    const SV a{A.x, A.y, 0.0}, b{B.x, B.y, 0.0}, c{C.x, C.y, 0.0};
    hl->fl[lane] = edge_flags(a, b, 0) | edge_flags(b, c, 1) | edge_flags(c, a, 2);
    hl->ia2[lane] = __drcp_rn((B.x - A.x) * (C.y - A.y) - (B.y - A.y) * (C.x - A.x));
    area = ((int)(bx.y & 0xffff) - (int)(bx.x & 0xffff) + 1) *
           ((int)(bx.y >> 16) - (int)(bx.x >> 16) + 1);
    if (area > kHugeBox) area = 0;  // swept one triangle at a time (sweep_huge_cta)
  }
  int incl = area;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane < nh) hl->pre[lane + 1] = incl;
  if (lane == 0) hl->pre[0] = 0;
}

// One huge list entry, all threads: bbox pixels strided by kThreads.
template <bool kIds, typename VS, typename Key, int kCap>
__device__ __forceinline__ void sweep_huge_cta(const KParams& p, Key* const zb, const Region& rg,
                                               const VS& vs, const HugeListT<kCap>* hl, int j,
                                               int tid) {
  const uint4 tr = hl->tri[j];
  const uint2 bx = hl->box[j];
  const int u0 = bx.x & 0xffff, v0 = bx.x >> 16;
  const int bw = (int)(bx.y & 0xffff) - u0 + 1, bh = (int)(bx.y >> 16) - v0 + 1;
  const int n = bw * bh;
  if (n <= kHugeBox) return;  // in the flattened sweep
  const double2 A = vs.uv(tr.x), B = vs.uv(tr.y), C = vs.uv(tr.z);
  const double iza = vs.iz(tr.x), izb = vs.iz(tr.y), izc = vs.iz(tr.z);
  const int fl = hl->fl[j];
  const double ia2 = hl->ia2[j];
  const uint32_t draw = p.draw_base + tr.w;
  for (int i = tid; i < n; i += kThreads) {
    const int row = i / bw;
    const int pu = u0 + (i - row * bw), pv = v0 + row;
    const double px = pu, py = pv;
    const double e_ab = edge_at(A, B, fl & 1, px, py);
    const double e_bc = edge_at(B, C, fl & 2, px, py);
    const double e_ca = edge_at(C, A, fl & 4, px, py);
    if (!edge_covers(e_ab, fl & 8) || !edge_covers(e_bc, fl & 16) || !edge_covers(e_ca, fl & 32))
      continue;
    const double inv_z = (e_bc * iza + e_ca * izb + e_ab * izc) * ia2;
    if (!(inv_z > 0)) continue;
    const double z = __drcp_rn(inv_z);
    if (z < p.near_lim || z > p.far_m) continue;
    const float zf = __double2float_rn(z);
    if (!(zf < p.far_f)) continue;
    Key* cell = zb + (pv - rg.oy) * rg.rw + (pu - rg.ox);
    if (kIds)
      zmin((unsigned long long*)cell,
           ((unsigned long long)__float_as_uint(zf) << 32) | (unsigned long long)draw);
    else
      zmin((unsigned int*)cell, __float_as_uint(zf));
  }
}

// All entries with bboxes <= kHugeBox pixels at once: thread i takes pixel
// i of the concatenated bboxes (entry found by binary search of the prefix).
template <bool kIds, typename VS, typename Key, int kCap>
__device__ __forceinline__ void sweep_list_cta(const KParams& p, Key* const zb, const Region& rg,
                                               const VS& vs, const HugeListT<kCap>* hl, int nh,
                                               int tid) {
  const int total = hl->pre[nh];
  for (int i = tid; i < total; i += kThreads) {
    int j = 0;  // last entry whose prefix <= i
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (j + step < nh && hl->pre[j + step] <= i) j += step;
    const uint4 tr = hl->tri[j];
    const uint2 bx = hl->box[j];
    const int u0 = bx.x & 0xffff, v0 = bx.x >> 16;
    const int bw = (int)(bx.y & 0xffff) - u0 + 1;
    const int k = i - hl->pre[j];
    const int row = k / bw;
    const int pu = u0 + (k - row * bw), pv = v0 + row;
    const double px = pu, py = pv;
    const int fl = hl->fl[j];
    const double2 A = vs.uv(tr.x), B = vs.uv(tr.y), C = vs.uv(tr.z);
    const double e_ab = edge_at(A, B, fl & 1, px, py);
    const double e_bc = edge_at(B, C, fl & 2, px, py);
    const double e_ca = edge_at(C, A, fl & 4, px, py);
    if (!edge_covers(e_ab, fl & 8) || !edge_covers(e_bc, fl & 16) || !edge_covers(e_ca, fl & 32))
      continue;
    const double inv_z = (e_bc * vs.iz(tr.x) + e_ca * vs.iz(tr.y) + e_ab * vs.iz(tr.z)) * hl->ia2[j];
    if (!(inv_z > 0)) continue;
    const double z = __drcp_rn(inv_z);
    if (z < p.near_lim || z > p.far_m) continue;
    const float zf = __double2float_rn(z);
    if (!(zf < p.far_f)) continue;
    Key* cell = zb + (pv - rg.oy) * rg.rw + (pu - rg.ox);
    if (kIds)
      zmin((unsigned long long*)cell,
           ((unsigned long long)__float_as_uint(zf) << 32) | (unsigned long long)(p.draw_base + tr.w));
    else
      zmin((unsigned int*)cell, __float_as_uint(zf));
  }
}

// Pass 2 for the <= 2x2 class: lane l takes queue entry head + l (l < n)
// and finishes it alone -- the 4 tile pixels' edge values (renderer.cpp:32-34
// factored into 2 row and 2 column products per edge, bitwise the reference's
// values), the top-left coverage rule (renderer.cpp:39-43), then for each
// covered pixel the perspective 1/z, near/far tests, fp32 round and
// strict-less z-test (renderer.cpp:94-100) from the same edge values.
template <bool kIds, typename VS, typename Key>
__device__ __forceinline__ void drain_small(const KParams& p, Key* const zb, const Region& rg,
                                            const VS& vs, const uint4* qt, const uint32_t* qb,
                                            int head, int n, int lane) {
  if (lane >= n) return;
  const int s = (head + lane) & (kRing - 1);
  const uint4 tr = qt[s];
  const uint32_t box = qb[s];
  const int u0 = box & 0x3fff, v0 = (box >> 16) & 0x3fff;
  const double2 PA = vs.uv(tr.x), PB = vs.uv(tr.y), PC = vs.uv(tr.z);
  const double px0 = (double)u0, py0 = (double)v0;
  const double px1 = px0 + 1.0, py1 = py0 + 1.0;
  // bit 2*j + i = pixel (u0 + i, v0 + j)
  uint32_t cov = 1u | ((box >> 14) & 1u) << 1;
  if (box >> 30) cov |= cov << 2;
  double e[3][4];
  const double2 P[3] = {PA, PB, PC};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double2 a = P[k], b = P[(k + 1) % 3];
    const bool canon = a.x < b.x || (a.x == b.x && a.y < b.y);
    const double dx = b.x - a.x, dy = b.y - a.y;
    const bool tie = dy < 0 || (dy == 0 && dx > 0);
    const double thr = tie ? -4.9406564584124654e-324 : 0.0;
    const double ox = canon ? a.x : b.x, oy = canon ? a.y : b.y;
    const double A0 = dx * (py0 - oy), A1 = dx * (py1 - oy);
    const double B0 = dy * (px0 - ox), B1 = dy * (px1 - ox);
    e[k][0] = A0 - B0;
    e[k][1] = A0 - B1;
    e[k][2] = A1 - B0;
    e[k][3] = A1 - B1;
    uint32_t m = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (e[k][q] > thr) m |= 1u << q;
    cov &= m;
  }
  if (!cov) return;
  // area2 of the swapped order is bitwise the negated original
  // (renderer.cpp:66-68): the two products are the same, only swapped
  const double ia2 =
      __drcp_rn((PB.x - PA.x) * (PC.y - PA.y) - (PB.y - PA.y) * (PC.x - PA.x));
  const double iza = vs.iz(tr.x), izb = vs.iz(tr.y), izc = vs.iz(tr.z);
  Key* const cell0 = zb + (v0 - rg.oy) * rg.rw + (u0 - rg.ox);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!((cov >> q) & 1u)) continue;
    // e[0] = ab, e[1] = bc, e[2] = ca (renderer.cpp:94-95)
    const double inv_z = (e[1][q] * iza + e[2][q] * izb + e[0][q] * izc) * ia2;
    if (!(inv_z > 0)) continue;
    const double z = __drcp_rn(inv_z);
    if (z < p.near_lim || z > p.far_m) continue;
    const float zf = __double2float_rn(z);
    if (!(zf < p.far_f)) continue;
    Key* cell = cell0 + (q >> 1) * rg.rw + (q & 1);
    if (kIds)
      zmin((unsigned long long*)cell, ((unsigned long long)__float_as_uint(zf) << 32) |
                                                  (unsigned long long)(p.draw_base + tr.w));
    else
      zmin((unsigned int*)cell, __float_as_uint(zf));
  }
}

// Pass 2 of the raster: lane l takes queue entry head + l (l < n): edge
// flags (renderer.cpp:39-47), KxK tile coverage; the covered pixels (~0.6
// per triangle) are then dealt one per lane -- owner found by a 5-step
// shuffle search over the exclusive scan of coverage counts -- for the
// perspective 1/z, the near/far tests, the fp32 round and the strict-less
// z-test (renderer.cpp:94-100) with every lane busy.
template <int K, bool kIds, typename VS, typename Key>
__device__ __forceinline__ void drain_queue(const KParams& p, Key* const zb, const Region& rg,
                                            const VS& vs, const uint4* qt, const uint32_t* qb,
                                            int head, int n, int lane) {
  uint32_t cov = 0, box = 0;
  uint4 tr = make_uint4(0u, 0u, 0u, 0u);
  int fl = 0;
  double inv_area2 = 0.0;
  if (lane < n) {
    const int s = (head + lane) & (kRing - 1);
    tr = qt[s];
    box = qb[s];
    const double2 PA = vs.uv(tr.x), PB = vs.uv(tr.y), PC = vs.uv(tr.z);
    const SV a{PA.x, PA.y, 0.0}, b{PB.x, PB.y, 0.0}, c{PC.x, PC.y, 0.0};
    fl = edge_flags(a, b, 0) | edge_flags(b, c, 1) | edge_flags(c, a, 2);
    const int u0 = box & 0x3fff, v0 = (box >> 16) & 0x3fff;
    const int bw = ((box >> 14) & 3) + 1, bh = (int)(box >> 30) + 1;
    const uint32_t colm = (1u << bw) - 1u;
    uint32_t valid = colm;  // bit K*j + i = pixel (u0 + i, v0 + j)
#pragma unroll
    for (int j = 1; j < K; ++j)
      if (bh > j) valid |= colm << (K * j);
    cov = valid & tile_edge_mask<K>(PA, PB, fl & 1, fl & 8, u0, v0) &
          tile_edge_mask<K>(PB, PC, fl & 2, fl & 16, u0, v0) &
          tile_edge_mask<K>(PC, PA, fl & 4, fl & 32, u0, v0);
    // area2 of the swapped order is bitwise the negated original
    // (renderer.cpp:66-68): the two products are the same, only swapped
    if (cov) inv_area2 = __drcp_rn((PB.x - PA.x) * (PC.y - PA.y) - (PB.y - PA.y) * (PC.x - PA.x));
  }
  const int cnt = __popc(cov);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int start = incl - cnt;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  for (int c0 = 0; c0 < total; c0 += 32) {
    const int item = c0 + lane;
    int own = 0;  // last lane whose start <= item (never a zero-count lane)
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int sp = __shfl_sync(0xffffffffu, start, own + step);
      if (sp <= item) own += step;
    }
    const int st = __shfl_sync(0xffffffffu, start, own);
    uint32_t m = __shfl_sync(0xffffffffu, cov, own);
    const uint32_t bx = __shfl_sync(0xffffffffu, box, own);
    const int flo = __shfl_sync(0xffffffffu, fl, own);
    const uint32_t ia = __shfl_sync(0xffffffffu, tr.x, own);
    const uint32_t ib = __shfl_sync(0xffffffffu, tr.y, own);
    const uint32_t ic = __shfl_sync(0xffffffffu, tr.z, own);
    const uint32_t tri = __shfl_sync(0xffffffffu, tr.w, own);
    const double ia2 = __shfl_sync(0xffffffffu, inv_area2, own);
    if (item < total) {
      for (int k = item - st; k > 0; --k) m &= m - 1;  // k-th covered pixel
      const int bit = __ffs(m) - 1;
      const int pu = (int)(bx & 0x3fff) + bit % K, pv = (int)((bx >> 16) & 0x3fff) + bit / K;
      const double2 A = vs.uv(ia), B = vs.uv(ib), C = vs.uv(ic);
      const double px = pu, py = pv;
      const double e_ab = edge_at(A, B, flo & 1, px, py);
      const double e_bc = edge_at(B, C, flo & 2, px, py);
      const double e_ca = edge_at(C, A, flo & 4, px, py);
      // renderer.cpp:94-100
      const double inv_z = (e_bc * vs.iz(ia) + e_ca * vs.iz(ib) + e_ab * vs.iz(ic)) * ia2;
      if (inv_z > 0) {
        const double z = __drcp_rn(inv_z);
        if (!(z < p.near_lim || z > p.far_m)) {
          const float zf = __double2float_rn(z);
          if (zf < p.far_f) {
            Key* cell = zb + (pv - rg.oy) * rg.rw + (pu - rg.ox);
            if (kIds)
              zmin((unsigned long long*)cell,
                           ((unsigned long long)__float_as_uint(zf) << 32) |
                               (unsigned long long)(p.draw_base + tri));
            else
              zmin((unsigned int*)cell, __float_as_uint(zf));
          }
        }
      }
    }
  }
}

// Shared state of one CTA while it processes one hypothesis.
struct HypCtx {
  const double* R;  // rotation (row-major) in shared memory
  const double* t;
  Region rg;
  bool empty_region, clip;
  int rpx;
  int q1;  // largest bbox side of the tile classes (2 or 3)
};

// Observation staging (north_star (3)): after the raster the on-chip vertex
// cache is dead, so the window-dilated region's observation rows (float4
// x, y, z, valid) are fetched into it by the bulk-copy engine
// (cp.async.bulk, completion counted on an mbarrier) while the CTA counts
// |y|; the window sums then read shared memory instead of L2.
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(a), "r"(phase) : "memory");
}

// Work of one hypothesis after the vertex phase: z-buffer init, raster,
// render-many output and/or likelihood.  Instantiated twice per kernel so
// that the z-buffer accesses compile to shared-memory instructions (kZS) or
// global ones (overflow scratch), never to generic ones.
template <bool kIds, bool kScore, bool kOut, int kWin, bool kS1, bool kCam, bool kQA,
          typename VS, typename Key>
__device__ __forceinline__ void hyp_body(const KParams& p, const HypCtx& hc, Key* const zb,
                                         const VS& vs, WarpQ* const wq, int* const s_seg,
                                         int* s_count, double* s_coef,
                                         double (*s_red)[kMaxNoise],
                                         int (*s_redi)[kMaxNoise + 1], long long h,
                                         const double* inst_rt, HugeListT<(kCam || !kScore) ? kMaxHuge : 1>* hl,
                                         int par, unsigned long long* obs_bar, unsigned& obs_phase) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Region& rg = hc.rg;
  const double* const R = hc.R;
  const double* const t = hc.t;
  // background depth 1e30 (not the far sentinel) so window taps on empty
  // pixels give d^2 = inf and an exact 0 term for any sigma; the z-test is
  // unchanged because every fragment is also tested zf < (float)far.
  const Key bg = kIds ? (Key)(((unsigned long long)__float_as_uint(kBgDepth) << 32) |
                              0xffffffffull)
                      : (Key)__float_as_uint(kBgDepth);
  if (p.base_keys) {  // compose_render: start from the fixed scene (inference.cpp:104)
    for (int i = tid; i < hc.rpx; i += kThreads) {
      const int v = rg.oy + i / rg.rw, u = rg.ox + (i - (i / rg.rw) * rg.rw);
      Key k = bg;
      if (u >= 0 && u < p.W && v >= 0 && v < p.H) {
        const unsigned long long b = __ldg(p.base_keys + (size_t)v * p.W + u);
        k = kIds ? (Key)b : (Key)(unsigned int)(b >> 32);
      }
      zb[i] = k;
    }
  } else {
    for (int i = tid; i < hc.rpx; i += kThreads) zb[i] = bg;
  }
  // score mode: the work list is the front part of each axis class (the cut
  // of phase B) plus all of class 6; s_seg[0..7] = running work counts,
  // s_seg[8..14] = first tris_s index of each segment
  constexpr bool kSorted = kScore && !kIds && !kCam;
  if (kSorted && tid == 0) {
    const bool cut = p.cull != 0 && !hc.clip;
    int cum = 0;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const int b = p.cls_start[c], e = (cut && c < 6) ? s_seg[16 + c] : p.cls_start[c + 1];
      s_seg[c] = cum;
      s_seg[8 + c] = b;
      cum += e - b;
    }
    s_seg[7] = cum;
  }
  __syncthreads();
  B3D_PCLK(3);

  // ---- C: raster, in two passes per 32-triangle chunk of each warp.
  // Pass 1, lane = triangle (mesh order): integer bbox reject, signed area,
  // back-face cull (closed meshes, score mode), orientation
  // swap (renderer.cpp:63-69); survivors are appended to the warp's queue of
  // their tile class (bbox <= 2x2 or <= 3x3; larger bboxes run the
  // reference's per-pixel loop in place).  Pass 2 (drain_queue) runs once a
  // queue holds 32 triangles, so the fp64 coverage work is done by full warps.
  if (!hc.empty_region || hc.clip) {
    WarpQ& q = wq[warp];
    const int cull = (kScore && !kIds && !hc.clip) ? p.cull : 0;
    const uint32_t lt_mask = (1u << lane) - 1u;
    int head0 = 0, tail0 = 0, head1 = 0, tail1 = 0;  // warp-uniform ring cursors
    const int n_work = kSorted ? s_seg[7] : p.nt;
    const uint4* const tl = kSorted ? p.tris_s : p.tris;
    auto work_tri = [&](int w) -> uint4 {
      int phys = w;
      if (kSorted) {
        int c = 0;
#pragma unroll
        for (int j = 1; j < 7; ++j) c += w >= s_seg[j];
        phys = s_seg[8 + c] + (w - s_seg[c]);
      }
      return __ldg(tl + phys);
    };
    const int c_first = warp * 32, c_stride = kThreads;
    for (int base = c_first; base < n_work; base += c_stride) {
      __syncwarp();
      const int ti = base + lane;
      int cls = -1;
      uint4 ent = make_uint4(0u, 0u, 0u, 0u);
      uint32_t box = 0, box2 = 0;
      if (ti < n_work) {
        const uint4 tri = work_tri(ti);
        uint32_t ia = tri.x, ib = tri.y, ic = tri.z;
        const short4 A = vs.bb(ia), B = vs.bb(ib), C = vs.bb(ic);
        if (A.x == kClipV || B.x == kClipV || C.x == kClipV) {
          if (kCam) {  // the triangle's instance transform (camera mode)
            int ins = 0;
            while (ins + 1 < p.n_inst && (int)ia >= p.inst_v0[ins + 1]) ++ins;
            raster_clipped<kIds>(p, zb, rg, inst_rt + 12 * ins, inst_rt + 12 * ins + 9, ia, ib,
                                 ic, p.draw_base + (uint32_t)ti);
          } else {
            raster_clipped<kIds>(p, zb, rg, R, t, ia, ib, ic, p.draw_base + (uint32_t)ti);
          }
        } else {
          const int u_min = min(min(A.x, B.x), C.x), v_min = min(min(A.z, B.z), C.z);
          const int u_max = max(max(A.y, B.y), C.y), v_max = max(max(A.w, B.w), C.w);
          if (u_max != kOvf && v_max != kOvf && u_min <= u_max && v_min <= v_max) {
            const double2 PA = vs.uv(ia);
            double2 PB = vs.uv(ib), PC = vs.uv(ic);
            double area2 = (PB.x - PA.x) * (PC.y - PA.y) - (PB.y - PA.y) * (PC.x - PA.x);
            if (area2 != 0 && !(cull > 0 ? area2 > 0 : (cull < 0 && area2 < 0))) {
              if (area2 < 0) {
                const double2 T = PB;
                PB = PC;
                PC = T;
                const uint32_t tt = ib;
                ib = ic;
                ic = tt;
                area2 = -area2;
              }
              const int bw = u_max - u_min + 1, bh = v_max - v_min + 1;
              if (bw <= (kQA ? hc.q1 : 3) && bh <= (kQA ? hc.q1 : 3)) {
                cls = (bw <= 2 && bh <= 2) ? 0 : 1;
                ent = make_uint4(ia, ib, ic, (uint32_t)ti);
                box = (uint32_t)u_min | (uint32_t)(bw - 1) << 14 | (uint32_t)v_min << 16 |
                      (uint32_t)(bh - 1) << 30;
              } else {
                int j = kMaxHuge;
                if (kCam || !kScore) {  // to the CTA's list (camera / render mode)
                  j = atomicAdd(&hl->n[par], 1);
                  if (j < kMaxHuge) {
                    hl->tri[j] = make_uint4(ia, ib, ic, (uint32_t)ti);
                    hl->box[j] = make_uint2((uint32_t)u_min | (uint32_t)v_min << 16,
                                            (uint32_t)u_max | (uint32_t)v_max << 16);
                  }
                }
                if (j < kMaxHuge) {
                } else if (bw * bh <= kHugeBox) {  // the reference's per-pixel loop
                  raster_tri_box<kIds>(p, zb, rg, SV{PA.x, PA.y, vs.iz(ia)},
                                       SV{PB.x, PB.y, vs.iz(ib)}, SV{PC.x, PC.y, vs.iz(ic)},
                                       u_min, u_max, v_min, v_max, p.draw_base + (uint32_t)ti);
                } else {  // huge bbox: swept by the whole warp below
                  cls = 3;
                  ent = make_uint4(ia, ib, ic, (uint32_t)ti);
                  box = (uint32_t)u_min | (uint32_t)v_min << 16;
                  box2 = (uint32_t)u_max | (uint32_t)v_max << 16;
                }
              }
            }
          }
        }
      }
      for (uint32_t hb = __ballot_sync(0xffffffffu, cls == 3); hb; hb &= hb - 1)
        sweep_huge<kIds>(p, zb, rg, vs, __ffs(hb) - 1, ent, box, box2, lane);
      const uint32_t b0 = __ballot_sync(0xffffffffu, cls == 0);
      const uint32_t b1 = __ballot_sync(0xffffffffu, cls == 1);
      if (cls == 0) {
        const int s = (tail0 + __popc(b0 & lt_mask)) & (kRing - 1);
        q.tri[0][s] = ent;
        q.box[0][s] = box;
      } else if (cls == 1) {
        const int s = (tail1 + __popc(b1 & lt_mask)) & (kRing - 1);
        q.tri[1][s] = ent;
        q.box[1][s] = box;
      }
      tail0 += __popc(b0);
      tail1 += __popc(b1);
      __syncwarp();
      if (tail0 - head0 >= 32) {
        drain_small<kIds>(p, zb, rg, vs, q.tri[0], q.box[0], head0, 32, lane);
        head0 += 32;
      }
      if (tail1 - head1 >= 32) {
        drain_queue<3, kIds>(p, zb, rg, vs, q.tri[1], q.box[1], head1, 32, lane);
        head1 += 32;
      }
    }
    if (tail0 > head0) drain_small<kIds>(p, zb, rg, vs, q.tri[0], q.box[0], head0, tail0 - head0, lane);
    if (tail1 > head1) drain_queue<3, kIds>(p, zb, rg, vs, q.tri[1], q.box[1], head1, tail1 - head1, lane);
  }
  __syncthreads();
  B3D_PCLK(4);
  if (const int nh = (kCam || !kScore) ? min(hl->n[par], kMaxHuge) : 0) {  // uniform after the barrier
    if (warp == 0) huge_prepare(hl, vs, nh, lane);
    __syncthreads();
    sweep_list_cta<kIds>(p, zb, rg, vs, hl, nh, tid);
    for (int j = 0; j < nh; ++j) sweep_huge_cta<kIds>(p, zb, rg, vs, hl, j, tid);
    __syncthreads();
  }
  B3D_PCLK(5);

  // ---- observation staging into the (now dead) on-chip vertex cache
  float4* staged = nullptr;
  if (kScore && !kIds && !kCam && !kQA && p.obs_stage && !hc.empty_region) {
    const int w = p.lik.window;
    const int du0 = max(rg.u0 - w, 0), du1 = min(rg.u1 + w, p.W - 1);
    const int dv0 = max(rg.v0 - w, 0), dv1 = min(rg.v1 + w, p.H - 1);
    const int dw = du1 - du0 + 1, dh = dv1 - dv0 + 1;
    if ((long long)dw * dh * 16 <= 32ll * p.vcap) {  // uniform across the CTA
      staged = reinterpret_cast<float4*>(vs.uvp);
      if (tid == 0) {
        // the raster's generic reads of this buffer (ordered by the barrier
        // above) before the bulk engine's writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(obs_bar, (unsigned)(dw * dh * 16));
        for (int r = 0; r < dh; ++r)
          bulk_g2s(staged + r * dw, p.obs + (size_t)(dv0 + r) * p.W + du0, (unsigned)(dw * 16),
                   obs_bar);
      }
    }
  }

  // ---- render-many output (sentinel = (float)far, id -1 = background)
  if (kOut) {
    const size_t npx = (size_t)p.W * p.H;
    float* od = p.out_depth ? p.out_depth + (size_t)h * npx : nullptr;
    int32_t* oi = p.out_ids ? p.out_ids + (size_t)h * npx : nullptr;
    unsigned long long* ok = p.out_keys ? p.out_keys + (size_t)h * npx : nullptr;
    for (int i = tid; i < (int)npx; i += kThreads) {
      const int u = i % p.W, v = i / p.W;
      Key k = bg;
      if (!hc.empty_region && u >= rg.u0 && u <= rg.u1 && v >= rg.v0 && v <= rg.v1)
        k = zb[(v - rg.oy) * rg.rw + (u - rg.ox)];
      else if (p.base_keys)
        k = kIds ? (Key)__ldg(p.base_keys + i) : (Key)(unsigned int)(__ldg(p.base_keys + i) >> 32);
      if (ok) ok[i] = kIds ? (unsigned long long)k : ((unsigned long long)k << 32) | 0xffffffffull;
      const float z = __uint_as_float(
          kIds ? (unsigned int)((unsigned long long)k >> 32) : (unsigned int)k);
      if (od) od[i] = z < p.far_f ? z : p.far_f;
      if (kIds && oi) {
        const unsigned int d = (unsigned int)((unsigned long long)k & 0xffffffffull);
        oi[i] = d == 0xffffffffu ? -1 : (int32_t)d;
      }
    }
  }

  if (kScore) {
    // launched with programmatic serialization behind the observation cache
    // (b3d_gpu_enumerate_observed's graph): everything above ran before it
    // finished; wait for it here (a no-op otherwise, and after the first time)
    if (!kCam) asm volatile("griddepcontrol.wait;" ::: "memory");
    // ---- D1: |y| = number of valid rendered pixels (likelihood.cpp:144-158)
    // With a base image: |y| = base count - base pixels of the region +
    // composed pixels of the region (the halo holds base pixels too, so the
    // interior [u0,u1]x[v0,v1] is counted).
    {
      int cnt = 0;
      const int iw = rg.u1 - rg.u0 + 1, ipx = iw * (rg.v1 - rg.v0 + 1);
      for (int i = tid; i < ipx; i += kThreads) {
        const int v = rg.v0 + i / iw, u = rg.u0 + (i - (i / iw) * iw);
        const Key k = zb[(v - rg.oy) * rg.rw + (u - rg.ox)];
        const float z = __uint_as_float(
            kIds ? (unsigned int)((unsigned long long)k >> 32) : (unsigned int)k);
        cnt += z < p.far_f;
        if (p.base_keys)
          cnt -= __uint_as_float((unsigned int)(__ldg(p.base_keys + (size_t)v * p.W + u) >> 32)) <
                 p.far_f;
      }
      cnt = warp_sum_i(cnt);
      if (lane == 0 && cnt) atomicAdd(s_count, cnt);
      __syncthreads();
      B3D_PCLK(6);
    }
    const int rend_count = *s_count + p.base_valid;
    // |y| = 0 (never with a non-empty base image): the reference throws
    // (likelihood.cpp:159-160); batched callers get -inf and a status flag
    // (DESIGN.md §5).
    const bool empty_render = rend_count == 0;
    // kS1 kernels: exactly one noise entry (and sigma); else up to kMaxNoise.
    // coef in fp64 in likelihood.cpp:167's order, by every thread (no
    // shared copy, no barrier)
    constexpr int kNN = kS1 ? 1 : kMaxNoise;
    float coef_f[kNN], floor_f[kNN];
#pragma unroll
    for (int e = 0; e < kNN; ++e) {
      coef_f[e] = (e < p.lik.n_noise && !empty_render)
                      ? (float)(p.lik.one_minus_p[e] / (double)rend_count * p.lik.norm3[e])
                      : 0.f;
      floor_f[e] = e < p.lik.n_noise ? (float)p.lik.floor_term[e] : 0.f;
    }

    // ---- D2: window sums over the dilated region.  Observed pixels whose
    // window holds no valid rendered pixel contribute exactly log(floor)
    // (likelihood.cpp:209-216 with an empty dist2 list); they are counted.
    // Taps are unconditional: the halo and every non-rendered pixel hold the
    // background depth, whose Gaussian term underflows to exactly 0.
    const int w = p.lik.window;
    const int du0 = max(rg.u0 - w, 0), du1 = min(rg.u1 + w, p.W - 1);
    const int dv0 = max(rg.v0 - w, 0), dv1 = min(rg.v1 + w, p.H - 1);
    const int dw = du1 - du0 + 1;
    const int dpx = (hc.empty_region || empty_render) ? 0 : dw * (dv1 - dv0 + 1);
    if (staged) {  // every thread waits, so the phase completes even unused
      mbar_wait(obs_bar, obs_phase);
      obs_phase ^= 1u;
    }
    double acc[kNN];
    int npos[kNN];
#pragma unroll
    for (int e = 0; e < kNN; ++e) {
      acc[e] = 0.0;
      npos[e] = 0;
    }
    for (int i = tid; i < dpx; i += kThreads) {
      const int pv = dv0 + i / dw;
      const int pu = du0 + (i - (pv - dv0) * dw);
      const float4 o = staged ? staged[i] : __ldg(p.obs + (size_t)pv * p.W + pu);
      if (o.w == 0.f) continue;
      float S[kMaxSlots];
      window_sums<kIds, kWin, kS1>(p, zb, rg, pu, pv, o, S);
      if (p.base_keys) {
        // g(S) - g(S_base): the pixel's term relative to the base-only sum G
#pragma unroll
        for (int e = 0; e < kNN; ++e) {
          if (e < p.lik.n_noise) {
            const int sl = p.lik.slot_of[e];
            const float Sb = __ldg(p.sbase + (size_t)sl * p.W * p.H + (size_t)pv * p.W + pu);
            if (S[sl] != Sb)
              acc[e] += (double)(__logf(floor_f[e] + coef_f[e] * S[sl]) -
                                 __logf(floor_f[e] + coef_f[e] * Sb));
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < kNN; ++e) {
          if (e < p.lik.n_noise) {
            const float Se = S[p.lik.slot_of[e]];
            if (Se > 0.f) {
              acc[e] += (double)__logf(floor_f[e] + coef_f[e] * Se);
              npos[e] += 1;
            }
          }
        }
      }
    }
    // ---- D3: fp64 block reduction -> one score per noise entry
#pragma unroll
    for (int e = 0; e < kNN; ++e) {
      acc[e] = warp_sum(acc[e]);
      npos[e] = warp_sum_i(npos[e]);
    }
    if (lane == 0) {
#pragma unroll
      for (int e = 0; e < kNN; ++e) {
        s_red[warp][e] = acc[e];
        s_redi[warp][e] = npos[e];
      }
    }
    __syncthreads();
    double a = 0.0;
    int np = 0;
    if (tid < p.lik.n_noise) {
      for (int k = 0; k < kWarps; ++k) {
        a += s_red[k][tid];
        np += s_redi[k][tid];
      }
    }
    if (tid < p.lik.n_noise) {
      const int e = tid;
      double total = p.lik.prefactor[e] + a;
      if (empty_render) {
        total = -__longlong_as_double(0x7ff0000000000000ll);
      } else if (p.base_keys) {
        // + G(log |y|): the base-only sum over all observed pixels, a smooth
        // function of |y| through coef; Chebyshev interpolant tabulated per
        // observation and noise entry (base_scene.cu)
        total += cheb_eval(p.cheb + e * kCheb, log((double)rend_count), p.cheb_lo, p.cheb_hi);
      } else {
        const int m_zero = *p.obs_count - np;
        if (m_zero > 0) total += (double)m_zero * p.lik.log_floor[e];
      }
      p.scores[h * p.lik.n_noise + e] = total;
      if (p.scores_mirror) p.scores_mirror[h * p.lik.n_noise + e] = total;
      if (p.n_score_peers) {  // the all-gather, fused: remote stores over NVLink
        const long long g = (p.score_peer_offset + h) * p.lik.n_noise + e;
        if (g < p.score_peer_cap)
          for (int r = 0; r < p.n_score_peers; ++r) p.score_peers[r][g] = total;
        __threadfence_system();
      }
    }
    if (tid == 0 && p.status) p.status[h] = empty_render ? 1 : 0;
  }
}

// Projected-vertex cache: (u, v) and 1/z in fp64 plus the packed integer
// bbox, in shared memory (kVS) or in the CTA's global scratch.
// Projected-vertex cache, structure of arrays (random gathers of 16-byte
// (u, v) pairs hit all bank groups): uv[n] | iz[n] | bb[n].
struct VertexCache {
  double2* uvp;
  double* izp;
  short4* bbp;
  __device__ __forceinline__ double2 uv(uint32_t i) const { return uvp[i]; }
  __device__ __forceinline__ double iz(uint32_t i) const { return izp[i]; }
  __device__ __forceinline__ short4 bb(uint32_t i) const { return bbp[i]; }
  __device__ __forceinline__ void put(uint32_t i, double u, double v, double iz, short4 bb) const {
    uvp[i] = make_double2(u, v);
    izp[i] = iz;
    bbp[i] = bb;
  }
  __device__ __forceinline__ void put_clipped(uint32_t i) const {
    bbp[i] = make_short4(kClipV, 0, 0, 0);
  }
};

// kIds: 64-bit (depth, draw) keys; kScore: run the likelihood epilogue;
// kOut: write the full depth / id images to HBM (render-many); kVS: the
// projected vertices fit in shared memory.
template <bool kIds, bool kScore, bool kOut, bool kVS, int kWin, bool kS1, bool kCam>
__global__ void __launch_bounds__(kThreads, B3D_MINB) render_score_kernel(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_pose[32][12];  // R (row-major) | t per upcoming hypothesis
  __shared__ int s_lo_u, s_hi_u, s_lo_v, s_hi_v, s_clip;
  __shared__ double s_red[kWarps][kMaxNoise];
  __shared__ int s_redi[kWarps][kMaxNoise + 1];
  __shared__ double s_coef[kMaxNoise];
  __shared__ int s_count;
  __shared__ int s_seg[24];  // score-mode work segments (hyp_body) + per-class cuts
  __shared__ double s_inst[kCam ? kMaxInst : 1][12];  // camera mode: R | t per instance
  __shared__ HugeListT<(kCam || !kScore) ? kMaxHuge : 1> s_huge;
  __shared__ __align__(8) unsigned long long s_obs_bar;  // observation staging
  using Key = typename KeyT<kIds>::T;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  // dynamic shared memory: per-warp triangle queues, region z-buffer (zcap
  // keys, a multiple of 8), projected-vertex cache (vcap x 32 B; in the CTA's
  // global scratch when the mesh does not fit).  The first two start at
  // compile-time offsets.
  WarpQ* const wq = reinterpret_cast<WarpQ*>(smem_raw);
  Key* const zb_s = reinterpret_cast<Key*>(smem_raw + sizeof(WarpQ) * kWarps);
  VertexCache vs;
  {
    const int n = kVS ? p.vcap : p.nv;
    double* const b = kVS ? reinterpret_cast<double*>(smem_raw + sizeof(WarpQ) * kWarps +
                                                      (size_t)p.zcap * sizeof(Key))
                          : p.vscratch + (size_t)blockIdx.x * 4 * p.nv;
    vs.uvp = reinterpret_cast<double2*>(b);
    vs.izp = b + 2 * (size_t)n;
    vs.bbp = reinterpret_cast<short4*>(b + 3 * (size_t)n);
  }

  // let a dependent launch (the stage reduction, launched with programmatic
  // stream serialization) be scheduled into SMs this grid leaves idle; it
  // waits for this grid's completion itself (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;");
  if (p.rng_dst && blockIdx.x == 0 && threadIdx.x < 5) p.rng_dst[threadIdx.x] = p.rng_init[threadIdx.x];
  unsigned obs_phase = 0;
  if (kScore && !kIds && !kCam && kVS && p.obs_stage && threadIdx.x == 0) mbar_init(&s_obs_bar, 1);
  B3D_PCLK(0);
#if B3D_L2_PREFETCH
  // Shared read-only inputs (mesh, sorted triangles, observation) into L2 in
  // one parallel burst spread over all CTAs, instead of every CTA's first
  // hypothesis meeting them at DRAM latency one dependent load at a time.
  {
    auto pf = [&](const void* base, size_t bytes) {
      const char* b = static_cast<const char*>(base);
      if (!b) return;
      for (size_t off = ((size_t)blockIdx.x * kThreads + threadIdx.x) * 128; off < bytes;
           off += (size_t)gridDim.x * kThreads * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b + off));
    };
    pf(p.verts, 24ull * p.nv);
    pf(kScore && !kIds && !kCam ? (const void*)p.tris_s : (const void*)p.tris, 16ull * p.nt);
    if (kScore) pf(p.obs, 16ull * p.W * p.H);
  }
#endif
  // camera mode may be launched with programmatic serialization behind the
  // kernel that wrote the camera poses (track.cu): wait for it here, after
  // the prefetch of the inputs it does not write (a no-op otherwise)
  if (kCam) asm volatile("griddepcontrol.wait;" ::: "memory");
  // Hypotheses one per CTA, strided by the grid (persistent CTAs).
  const long long G = gridDim.x;
  int kk = 0;  // hypotheses this CTA has processed
  for (long long h = blockIdx.x; h < p.n_hyp; h += G, ++kk) {
    // ---- A: poses of this CTA's next 32 hypotheses, one per lane of warp 0
    // (compose with inverse(camera) -> rotation matrix + translation)
    if (kCam) {
      // camera mode: M2C_i = compose(inverse(camera_h), model_to_world_i)
      // (renderer.cpp:164-170) for every instance
      if (tid < p.n_inst) {
        const KPose w2c = pm::pose_inverse(p.cams[h]);
        pose_to_rt(w2c, p.inst_pose[tid], s_inst[tid], s_inst[tid] + 9);
      }
    } else if ((kk & 31) == 0 && warp == 0) {
      const long long hh = h + (long long)lane * G;
      if (hh < p.n_hyp) {
        KPose hp;
        if (p.poses)
          hp = p.poses[hh];
        else
          grid_pose(p.grid, p.index0 + hh, hp);
        pose_to_rt(p.w2c, hp, s_pose[lane], s_pose[lane] + 9);
      }
    }
    if (tid == 0) {
      s_lo_u = INT_MAX;
      s_lo_v = INT_MAX;
      s_hi_u = INT_MIN;
      s_hi_v = INT_MIN;
      s_clip = 0;
      s_count = 0;
      if (kCam || !kScore) s_huge.n[kk & 1] = 0;
    }
    __syncthreads();
    B3D_PCLK(1);
    HypCtx hc;
    hc.R = s_pose[kk & 31];  // broadcast reads from shared memory
    hc.t = hc.R + 9;
    const double* const R = hc.R;
    const double* const t = hc.t;

    // ---- B: vertices -> (u, v, 1/z), packed bbox, region bounds
    int lo_u = INT_MAX, lo_v = INT_MAX, hi_u = INT_MIN, hi_v = INT_MIN, clip = 0;
    for (int i = tid; i < p.nv; i += kThreads) {
      double c[3];
      if (kCam) {
        int ins = 0;
        while (ins + 1 < p.n_inst && i >= p.inst_v0[ins + 1]) ++ins;
        cam_vertex(s_inst[ins], s_inst[ins] + 9, p.verts + 3 * (size_t)i, c);
      } else {
        cam_vertex(R, t, p.verts + 3 * (size_t)i, c);
      }
      if (c[2] >= p.near_m) {
        const SV s = project(p, c[0], c[1], c[2]);
        const short4 bb = vertex_bbox(p, s.u, s.v);
        vs.put(i, s.u, s.v, s.iz, bb);
        lo_u = min(lo_u, (int)bb.x);
        hi_u = max(hi_u, bb.y == kOvf ? p.W - 1 : (int)bb.y);
        lo_v = min(lo_v, (int)bb.z);
        hi_v = max(hi_v, bb.w == kOvf ? p.H - 1 : (int)bb.w);
      } else {
        vs.put_clipped(i);
        clip = 1;
      }
    }
    // score mode: per axis class c (warp c), the faces turned towards the
    // camera centre C = -R^T t (model frame) are those with plane offset
    // o <= n . C: a prefix of the class (b3d_kernels.cuh).  The small margin
    // keeps near-edge-on planes; they go through the exact tests.
    if (kScore && !kIds && !kCam && warp < 6) {
      const int k = warp >> 1;
      const double Ck = -(R[k] * t[0] + R[3 + k] * t[1] + R[6 + k] * t[2]);
      const double thr = (warp & 1) ? -Ck : Ck;
      const double lim = thr + 1e-9 * (1.0 + fabs(thr));
      const int pb = p.plane_begin[warp], pe = p.plane_begin[warp + 1];
      int n_le = 0;
      for (int j0 = pb; j0 < pe; j0 += 32) {
        const int j = j0 + lane;
        n_le += __popc(__ballot_sync(0xffffffffu, j < pe && __ldg(p.plane_off + j) <= lim));
      }
      if (lane == 0) s_seg[16 + warp] = n_le ? __ldg(p.plane_end + pb + n_le - 1) : p.cls_start[warp];
    }
  #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo_u = min(lo_u, __shfl_xor_sync(0xffffffffu, lo_u, o));
      lo_v = min(lo_v, __shfl_xor_sync(0xffffffffu, lo_v, o));
      hi_u = max(hi_u, __shfl_xor_sync(0xffffffffu, hi_u, o));
      hi_v = max(hi_v, __shfl_xor_sync(0xffffffffu, hi_v, o));
      clip |= __shfl_xor_sync(0xffffffffu, clip, o);
    }
    if (lane == 0) {
      atomicMin(&s_lo_u, lo_u);
      atomicMin(&s_lo_v, lo_v);
      atomicMax(&s_hi_u, hi_u);
      atomicMax(&s_hi_v, hi_v);
      if (clip) s_clip = 1;
    }
    __syncthreads();
    B3D_PCLK(2);
    Region& rg = hc.rg;
    hc.clip = s_clip != 0;
    if (hc.clip) {
      rg.u0 = 0;
      rg.v0 = 0;
      rg.u1 = p.W - 1;
      rg.v1 = p.H - 1;
    } else {
      rg.u0 = max(s_lo_u, 0);
      rg.v0 = max(s_lo_v, 0);
      rg.u1 = min(s_hi_u, p.W - 1);
      rg.v1 = min(s_hi_v, p.H - 1);
    }
    hc.empty_region = rg.u0 > rg.u1 || rg.v0 > rg.v1;
    // The tile classes (queues + dealt fragments) pay off for small projected
    // triangles; when the mesh's faces span ~2 px or more (region area >
    // p.q1_ratio / 100 x triangles, default 0.2; a voxel blob's ratio grows
    // with the squared projected voxel size: cfg1 0.19 at 1.7 px, cfg2 0.24
    // at 2.1 px, cfg4 0.68 at 3.3 px) the per-lane loop is faster for every
    // bbox above p.q1_small px a side (cfg3/cfg4 +15 %, cfg2 +1.5 %).
    // Meshes whose vertex cache fits on chip are small and keep the class;
    // so does camera mode, whose full-frame region says nothing about the
    // triangles' size (bench-tracking 200 px 1.7k -> 2.3k FPS with it).
    hc.q1 = (!kVS && !hc.empty_region &&
             100ll * (rg.u1 - rg.u0 + 1) * (rg.v1 - rg.v0 + 1) > (long long)p.q1_ratio * p.nt)
                ? p.q1_small
                : 3;
    if (hc.empty_region) {  // keep one valid (unused) pixel so indexing stays sane
      rg.u1 = rg.u0 = min(max(rg.u0, 0), p.W - 1);
      rg.v1 = rg.v0 = min(max(rg.v0, 0), p.H - 1);
    }
    const int pad = kScore ? 2 * p.lik.window : 0;
    rg.ox = rg.u0 - pad;
    rg.oy = rg.v0 - pad;
    rg.rw = rg.u1 - rg.u0 + 1 + 2 * pad;
    rg.rh = rg.v1 - rg.v0 + 1 + 2 * pad;
    hc.rpx = rg.rw * rg.rh;
    if (hc.rpx <= p.zcap)
      hyp_body<kIds, kScore, kOut, kWin, kS1, kCam, !kVS && !kCam>(p, hc, zb_s, vs, wq, s_seg, &s_count, s_coef,
                                                    s_red, s_redi, h, &s_inst[0][0], &s_huge, kk & 1, &s_obs_bar, obs_phase);
    else
      hyp_body<kIds, kScore, kOut, kWin, kS1, kCam, !kVS && !kCam>(
          p, hc, reinterpret_cast<Key*>(p.zscratch + (size_t)blockIdx.x * p.zstride), vs, wq,
          s_seg, &s_count, s_coef, s_red, s_redi, h, &s_inst[0][0], &s_huge, kk & 1, &s_obs_bar, obs_phase);
    B3D_PCLK(7);
    // No barrier here: before the next hypothesis's first barrier only
    // s_pose (warp 0), the region / count words (thread 0) and s_inst are
    // written, and none of them is read after hyp_body's last barrier; the
    // z-buffer and the vertex cache are rewritten only after that barrier.
  }
}

}  // namespace b3d200

// Explicit instantiations of the score kernels, one translation unit per
// window radius (rs_score_w*.cu) so they compile in parallel.
#define B3D_RS_SCORE_KERNELS2(X, W, C)                                                           \
  X template __global__ void render_score_kernel<false, true, false, true, W, true, C>(const KParams); \
  X template __global__ void render_score_kernel<false, true, false, false, W, true, C>(const KParams); \
  X template __global__ void render_score_kernel<false, true, false, true, W, false, C>(const KParams); \
  X template __global__ void render_score_kernel<false, true, false, false, W, false, C>(const KParams);
#define B3D_RS_SCORE_KERNELS(X, W) B3D_RS_SCORE_KERNELS2(X, W, false)
// camera mode (multi-instance scene under per-hypothesis cameras): score
// kernels with the generic window loop, and the render kernels
#define B3D_RS_CAM_KERNELS(X)                                                                    \
  B3D_RS_SCORE_KERNELS2(X, -1, true)                                                             \
  X template __global__ void render_score_kernel<true, false, true, true, -1, false, true>(const KParams);  \
  X template __global__ void render_score_kernel<true, false, true, false, -1, false, true>(const KParams); \
  X template __global__ void render_score_kernel<false, false, true, true, -1, false, true>(const KParams); \
  X template __global__ void render_score_kernel<false, false, true, false, -1, false, true>(const KParams);
