// render_score.cu -- fused per-hypothesis rasterizer + windowed likelihood
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
#include <cfloat>
#include <climits>
#include <cstdint>

#include "b3d_kernels.cuh"
#include "posemath.cuh"

namespace b3d200 {

namespace {

using namespace pm;

// static_cast<int>(double) as the x86-64 reference build executes it
// (cvttsd2si: out of range or NaN -> INT_MIN).
__device__ __forceinline__ int to_int_x86(double x) {
  if (!(x > -2147483649.0 && x < 2147483648.0)) return (int)0x80000000u;
  return __double2int_rz(x);
}

struct SV {
  double u, v, iz;
};

// renderer.cpp:26-59, with the orientation sign folded into the canonical
// deltas: sign*(cdx*A - cdy*B) == (sign*cdx)*A - (sign*cdy)*B bitwise for
// sign = +-1 (round-to-nearest is symmetric; only the sign of an exact zero
// can differ, which neither the fill rule nor the depth test observes).
struct Edge {
  double ox, oy, scdx, scdy, dx, dy;
};

__device__ __forceinline__ Edge make_edge(const SV& a, const SV& b) {
  const bool canonical = a.u < b.u || (a.u == b.u && a.v < b.v);
  const double lou = canonical ? a.u : b.u, lov = canonical ? a.v : b.v;
  const double hiu = canonical ? b.u : a.u, hiv = canonical ? b.v : a.v;
  Edge e;
  e.ox = lou;
  e.oy = lov;
  const double cdx = hiu - lou, cdy = hiv - lov;
  e.scdx = canonical ? cdx : -cdx;
  e.scdy = canonical ? cdy : -cdy;
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

__device__ __forceinline__ void zmin(unsigned int* p, unsigned int v) {
  if (v < *p) atomicMin(p, v);
}
__device__ __forceinline__ void zmin(unsigned long long* p, unsigned long long v) {
  if (v < *p) atomicMin(p, v);
}

struct Region {
  int u0, v0, u1, v1, rw;
};

// renderer.cpp:61-103 -- one screen triangle into the region z-buffer.
template <bool kIds>
__device__ void raster_tri(const KParams& p, typename KeyT<kIds>::T* zb, const Region& rg,
                           SV a, SV b, SV c, uint32_t draw) {
  double area2 = (b.u - a.u) * (c.v - a.v) - (b.v - a.v) * (c.u - a.u);
  if (area2 == 0) return;
  if (area2 < 0) {
    const SV t = b;
    b = c;
    c = t;
    area2 = -area2;
  }
  double mnu = a.u, mxu = a.u, mnv = a.v, mxv = a.v;
  if (b.u < mnu) mnu = b.u;
  if (c.u < mnu) mnu = c.u;
  if (mxu < b.u) mxu = b.u;
  if (mxu < c.u) mxu = c.u;
  if (b.v < mnv) mnv = b.v;
  if (c.v < mnv) mnv = c.v;
  if (mxv < b.v) mxv = b.v;
  if (mxv < c.v) mxv = c.v;
  int u_min = to_int_x86(ceil(mnu));
  if (u_min < 0) u_min = 0;
  int u_max = to_int_x86(floor(mxu));
  if (u_max > p.W - 1) u_max = p.W - 1;
  int v_min = to_int_x86(ceil(mnv));
  if (v_min < 0) v_min = 0;
  int v_max = to_int_x86(floor(mxv));
  if (v_max > p.H - 1) v_max = p.H - 1;
  if (u_min > u_max || v_min > v_max) return;

  const Edge ab = make_edge(a, b);
  const Edge bc = make_edge(b, c);
  const Edge ca = make_edge(c, a);
  const double inv_area2 = 1.0 / area2;

  for (int pv = v_min; pv <= v_max; ++pv) {
    const double py = pv;
    const double r_ab = ab.scdx * (py - ab.oy);
    const double r_bc = bc.scdx * (py - bc.oy);
    const double r_ca = ca.scdx * (py - ca.oy);
    typename KeyT<kIds>::T* row = zb + (pv - rg.v0) * rg.rw - rg.u0;
    for (int pu = u_min; pu <= u_max; ++pu) {
      const double px = pu;
      const double e_ab = r_ab - ab.scdy * (px - ab.ox);
      const double e_bc = r_bc - bc.scdy * (px - bc.ox);
      const double e_ca = r_ca - ca.scdy * (px - ca.ox);
      if (!covers(ab, e_ab) || !covers(bc, e_bc) || !covers(ca, e_ca)) continue;
      const double inv_z = (e_bc * a.iz + e_ca * b.iz + e_ab * c.iz) * inv_area2;
      if (inv_z <= 0) continue;
      const double z = 1.0 / inv_z;
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

__device__ __forceinline__ SV project(const KParams& p, double x, double y, double z) {
  const double iz = 1.0 / z;
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

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

}  // namespace

// kIds: 64-bit (depth, draw) keys; kScore: run the likelihood epilogue;
// kOut: write the full depth / id images to HBM (render-many).
template <bool kIds, bool kScore, bool kOut>
__global__ void __launch_bounds__(kThreads) render_score_kernel(const KParams p) {
  using Key = typename KeyT<kIds>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_R[9], s_t[3];
  __shared__ int s_lo_u, s_hi_u, s_lo_v, s_hi_v, s_clip;
  __shared__ double s_red[kWarps][kMaxNoise];
  __shared__ int s_redi[kWarps][kMaxNoise + 1];
  __shared__ double s_coef[kMaxNoise];
  __shared__ int s_count;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  double* const sv_u_s = reinterpret_cast<double*>(smem_raw);
  const bool v_in_smem = p.nv <= p.vcap;
  double* const vu = v_in_smem ? sv_u_s : p.vscratch + (size_t)blockIdx.x * 3 * p.nv;
  const int vstride = v_in_smem ? p.vcap : p.nv;
  double* const vv = vu + vstride;
  double* const viz = vv + vstride;
  Key* const zb_s = reinterpret_cast<Key*>(sv_u_s + 3 * (size_t)p.vcap);

  for (long long h = blockIdx.x; h < p.n_hyp; h += gridDim.x) {
    // ---- A: pose
    if (tid == 0) {
      KPose hp;
      if (p.poses)
        hp = p.poses[h];
      else
        grid_pose(p.grid, h, hp);
      pose_to_rt(p.w2c, hp, s_R, s_t);
      s_lo_u = INT_MAX;
      s_lo_v = INT_MAX;
      s_hi_u = INT_MIN;
      s_hi_v = INT_MIN;
      s_clip = 0;
      s_count = 0;
    }
    __syncthreads();
    double R[9], t[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = s_R[i];
    t[0] = s_t[0];
    t[1] = s_t[1];
    t[2] = s_t[2];

    // ---- B: vertices -> (u, v, 1/z), region bounds
    int lo_u = INT_MAX, lo_v = INT_MAX, hi_u = INT_MIN, hi_v = INT_MIN, clip = 0;
    for (int i = tid; i < p.nv; i += kThreads) {
      double c[3];
      cam_vertex(R, t, p.verts + 3 * (size_t)i, c);
      if (c[2] >= p.near_m) {
        const SV s = project(p, c[0], c[1], c[2]);
        vu[i] = s.u;
        vv[i] = s.v;
        viz[i] = s.iz;
        // clamp before converting: the region only has to contain every
        // triangle bbox (which raster_tri recomputes exactly)
        const double cu = fmin(fmax(ceil(s.u), -1.0), (double)p.W);
        const double fu = fmin(fmax(floor(s.u), -1.0), (double)p.W);
        const double cv = fmin(fmax(ceil(s.v), -1.0), (double)p.H);
        const double fv = fmin(fmax(floor(s.v), -1.0), (double)p.H);
        lo_u = min(lo_u, (int)cu);
        hi_u = max(hi_u, (int)fu);
        lo_v = min(lo_v, (int)cv);
        hi_v = max(hi_v, (int)fv);
      } else {
        vu[i] = __longlong_as_double(0x7ff8000000000000ll);  // NaN marks "clip"
        clip = 1;
      }
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
    Region rg;
    if (s_clip) {
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
    const bool empty_region = rg.u0 > rg.u1 || rg.v0 > rg.v1;
    if (empty_region) {  // keep one valid (unused) pixel so indexing stays sane
      rg.u1 = rg.u0 = min(max(rg.u0, 0), p.W - 1);
      rg.v1 = rg.v0 = min(max(rg.v0, 0), p.H - 1);
    }
    rg.rw = rg.u1 - rg.u0 + 1;
    const int rpx = rg.rw * (rg.v1 - rg.v0 + 1);
    Key* const zb = rpx <= p.zcap ? zb_s
                                  : reinterpret_cast<Key*>(p.zscratch +
                                                           (size_t)blockIdx.x * p.W * p.H);
    const Key bg = kIds ? (Key)(((unsigned long long)__float_as_uint(p.far_f) << 32) |
                                0xffffffffull)
                        : (Key)__float_as_uint(p.far_f);
    for (int i = tid; i < rpx; i += kThreads) zb[i] = bg;
    __syncthreads();

    // ---- C: raster, thread per triangle in mesh order
    if (!empty_region || s_clip) {
      for (int ti = tid; ti < p.nt; ti += kThreads) {
        const uint32_t i0 = __ldg(p.tris + 3 * ti), i1 = __ldg(p.tris + 3 * ti + 1),
                       i2 = __ldg(p.tris + 3 * ti + 2);
        const double au = vu[i0], bu = vu[i1], cu = vu[i2];
        const uint32_t draw = p.draw_base + (uint32_t)ti;
        if (isnan(au) || isnan(bu) || isnan(cu)) {
          raster_clipped<kIds>(p, zb, rg, R, t, i0, i1, i2, draw);
        } else {
          raster_tri<kIds>(p, zb, rg, SV{au, vv[i0], viz[i0]}, SV{bu, vv[i1], viz[i1]},
                           SV{cu, vv[i2], viz[i2]}, draw);
        }
      }
    }
    __syncthreads();

    // ---- render-many output
    if (kOut) {
      const size_t npx = (size_t)p.W * p.H;
      float* od = p.out_depth + (size_t)h * npx;
      int32_t* oi = p.out_ids ? p.out_ids + (size_t)h * npx : nullptr;
      for (int i = tid; i < (int)npx; i += kThreads) {
        const int u = i % p.W, v = i / p.W;
        Key k = bg;
        if (!empty_region && u >= rg.u0 && u <= rg.u1 && v >= rg.v0 && v <= rg.v1)
          k = zb[(v - rg.v0) * rg.rw + (u - rg.u0)];
        if (kIds) {
          od[i] = __uint_as_float((unsigned int)((unsigned long long)k >> 32));
          if (oi) {
            const unsigned int d = (unsigned int)((unsigned long long)k & 0xffffffffull);
            oi[i] = d == 0xffffffffu ? -1 : (int32_t)d;
          }
        } else {
          od[i] = __uint_as_float((unsigned int)k);
        }
      }
    }

    if (kScore) {
      // ---- D1: |y| = number of valid rendered pixels (likelihood.cpp:144-158)
      int cnt = 0;
      if (!empty_region)
        for (int i = tid; i < rpx; i += kThreads) {
          const float z = __uint_as_float(
              kIds ? (unsigned int)((unsigned long long)zb[i] >> 32) : (unsigned int)zb[i]);
          cnt += z < p.far_f;
        }
      cnt = warp_sum_i(cnt);
      if (lane == 0 && cnt) atomicAdd(&s_count, cnt);
      __syncthreads();
      const int rend_count = s_count;
      if (rend_count == 0) {
        // the reference throws (likelihood.cpp:159-160); batched callers get
        // -inf and a status flag instead
        if (tid == 0) {
          for (int e = 0; e < p.lik.n_noise; ++e)
            p.scores[h * p.lik.n_noise + e] = -__longlong_as_double(0x7ff0000000000000ll);
          if (p.status) p.status[h] = 1;
        }
        __syncthreads();
        continue;
      }
      if (tid < p.lik.n_noise)  // likelihood.cpp:167 coefficient order
        s_coef[tid] = p.lik.one_minus_p[tid] / (double)rend_count * p.lik.norm3[tid];
      __syncthreads();
      float coef_f[kMaxNoise], floor_f[kMaxNoise];
#pragma unroll
      for (int e = 0; e < kMaxNoise; ++e) {
        coef_f[e] = e < p.lik.n_noise ? (float)s_coef[e] : 0.f;
        floor_f[e] = e < p.lik.n_noise ? (float)p.lik.floor_term[e] : 0.f;
      }

      // ---- D2: window sums over the dilated region.  Observed pixels whose
      // window holds no valid rendered pixel contribute exactly log(floor)
      // (likelihood.cpp:209-216 with an empty dist2 list); they are counted.
      const int w = p.lik.window;
      const int du0 = max(rg.u0 - w, 0), du1 = min(rg.u1 + w, p.W - 1);
      const int dv0 = max(rg.v0 - w, 0), dv1 = min(rg.v1 + w, p.H - 1);
      const int dw = du1 - du0 + 1;
      const int dpx = dw * (dv1 - dv0 + 1);
      double acc[kMaxNoise];
      int npos[kMaxNoise];
#pragma unroll
      for (int e = 0; e < kMaxNoise; ++e) {
        acc[e] = 0.0;
        npos[e] = 0;
      }
      for (int i = tid; i < dpx; i += kThreads) {
        const int u = du0 + i % dw, v = dv0 + i / dw;
        const float4 o = __ldg(p.obs + (size_t)v * p.W + u);
        if (o.w == 0.f) continue;
        float S[kMaxNoise];
#pragma unroll
        for (int s = 0; s < kMaxNoise; ++s) S[s] = 0.f;
        const int rv0 = max(v - w, rg.v0), rv1 = min(v + w, rg.v1);
        const int ru0 = max(u - w, rg.u0), ru1 = min(u + w, rg.u1);
        for (int rv = rv0; rv <= rv1; ++rv) {
          const Key* row = zb + (rv - rg.v0) * rg.rw - rg.u0;
          const float fyr = ((float)rv - p.fcy) * p.inv_fy;
          for (int ru = ru0; ru <= ru1; ++ru) {
            const Key k = row[ru];
            const float z = __uint_as_float(
                kIds ? (unsigned int)((unsigned long long)k >> 32) : (unsigned int)k);
            if (!(z < p.far_f)) continue;
            const float dx = o.x - ((float)ru - p.fcx) * p.inv_fx * z;
            const float dy = o.y - fyr * z;
            const float dz = o.z - z;
            const float d2 = dx * dx + (dy * dy + dz * dz);
#pragma unroll
            for (int s = 0; s < kMaxNoise; ++s)
              if (s < p.lik.n_slots) S[s] += __expf(-d2 * p.lik.slot_scale[s]);
          }
        }
#pragma unroll
        for (int e = 0; e < kMaxNoise; ++e) {
          if (e < p.lik.n_noise) {
            const float Se = S[p.lik.slot_of[e]];
            if (Se > 0.f) {
              acc[e] += (double)__logf(floor_f[e] + coef_f[e] * Se);
              npos[e] += 1;
            }
          }
        }
      }
      // ---- D3: fp64 block reduction -> one score per noise entry
#pragma unroll
      for (int e = 0; e < kMaxNoise; ++e) {
        acc[e] = warp_sum(acc[e]);
        npos[e] = warp_sum_i(npos[e]);
      }
      if (lane == 0) {
#pragma unroll
        for (int e = 0; e < kMaxNoise; ++e) {
          s_red[warp][e] = acc[e];
          s_redi[warp][e] = npos[e];
        }
      }
      __syncthreads();
      if (tid < p.lik.n_noise) {
        const int e = tid;
        double a = 0.0;
        int np = 0;
        for (int k = 0; k < kWarps; ++k) {
          a += s_red[k][e];
          np += s_redi[k][e];
        }
        const int m_zero = *p.obs_count - np;
        double total = p.lik.prefactor[e] + a;
        if (m_zero > 0) total += (double)m_zero * p.lik.log_floor[e];
        p.scores[h * p.lik.n_noise + e] = total;
      }
      if (tid == 0 && p.status) p.status[h] = 0;
    }
    __syncthreads();
  }
}

// Observation cache (likelihood.cpp:106-126) as per-pixel fp32 points plus
// the valid count M.
__global__ void obs_prepare_kernel(const float* depth, int W, int H, float far_f, float fcx,
                                   float fcy, float inv_fx, float inv_fy, float4* out,
                                   int* count) {
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int c = 0;
  const int n = W * H;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float z = depth[i];
    const int u = i % W, v = i / W;
    if (z < far_f) {
      out[i] = make_float4(((float)u - fcx) * inv_fx * z, ((float)v - fcy) * inv_fy * z, z, 1.f);
      ++c;
    } else {
      out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  c = warp_sum_i(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) atomicAdd(count, s_cnt);
}

// Host-side launch helpers (declared in b3d_host.cpp).
template <bool kIds, bool kScore, bool kOut>
cudaError_t launch_render_score(const KParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = render_score_kernel<kIds, kScore, kOut>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

template <bool kIds, bool kScore, bool kOut>
cudaError_t occupancy_render_score(int* blocks, size_t smem) {
  auto kern = render_score_kernel<kIds, kScore, kOut>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kern, kThreads, smem);
}

template cudaError_t launch_render_score<false, true, false>(const KParams&, int, size_t,
                                                             cudaStream_t);
template cudaError_t launch_render_score<true, false, true>(const KParams&, int, size_t,
                                                            cudaStream_t);
template cudaError_t launch_render_score<false, false, true>(const KParams&, int, size_t,
                                                             cudaStream_t);
template cudaError_t occupancy_render_score<false, true, false>(int*, size_t);
template cudaError_t occupancy_render_score<true, false, true>(int*, size_t);
template cudaError_t occupancy_render_score<false, false, true>(int*, size_t);

cudaError_t launch_obs_prepare(const float* depth, int W, int H, float far_f, float fcx,
                               float fcy, float inv_fx, float inv_fy, float4* out, int* count,
                               cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  const int n = W * H;
  int grid = (n + 255) / 256;
  if (grid > 1184) grid = 1184;
  obs_prepare_kernel<<<grid, 256, 0, st>>>(depth, W, H, far_f, fcx, fcy, inv_fx, inv_fy, out,
                                           count);
  return cudaGetLastError();
}

int render_score_threads() { return kThreads; }

}  // namespace b3d200
