// mesh_build.cu -- voxel_to_mesh (geometry.cpp:142-177) on the device.
//
// The reference walks the voxels in stored order, emits the exterior faces of
// each voxel (neighbour not occupied) as two triangles, and numbers quad
// corners in first-seen order through a hash map.  The device restatement
// gives the same vertex numbering and triangle order without any sequential
// walk:
//   1. voxel hash set (open addressing, 63-bit packed keys);
//   2. exterior flag per (voxel, face) slot t = 6 i + face;
//      face slot = exclusive scan of the flags (face order == the walk's);
//   3. every corner of every exterior face has sequence number
//      s = 4 * face_slot + corner -- the order of the reference's corner_id
//      calls; a corner hash map keeps the minimum s per corner (atomicMin);
//   4. "s is a first occurrence" flags, exclusive scan -> vertex id of each
//      first occurrence (= the reference's vertices.size() at that call);
//   5. one thread per exterior face: vertex ids of its 4 corners, the first
//      occurrences write their vertex (origin + resolution * corner, fp64
//      without FMA), and the two triangles (q0,q1,q2), (q0,q2,q3).
// Duplicate voxels in the input are walked twice, as in the reference
// (their faces repeat; the occupancy set holds them once).
#include <cuda_runtime.h>

#include <cstdint>

#include <cub/device/device_scan.cuh>

namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kBias = 1 << 20;  // coordinates (and corners/neighbours) in [-2^20, 2^20)

__constant__ int c_off[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0},
                                {0, 1, 0},  {0, 0, -1}, {0, 0, 1}};
// geometry.cpp:128-135, counter-clockwise seen from outside
__constant__ int c_corner[6][4][3] = {
    {{0, 0, 0}, {0, 0, 1}, {0, 1, 1}, {0, 1, 0}},
    {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}, {1, 0, 1}},
    {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}, {0, 0, 1}},
    {{0, 1, 0}, {0, 1, 1}, {1, 1, 1}, {1, 1, 0}},
    {{0, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 0, 0}},
    {{0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}},
};

__device__ __forceinline__ unsigned long long pack(int x, int y, int z) {
  return (unsigned long long)(unsigned)(x + kBias) << 42 |
         (unsigned long long)(unsigned)(y + kBias) << 21 | (unsigned long long)(unsigned)(z + kBias);
}

__device__ __forceinline__ unsigned long long mix(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  return k ^ (k >> 33);
}

// slot of key (inserting it when absent); capacity is a power of two > keys
__device__ __forceinline__ unsigned long long insert(unsigned long long* keys,
                                                     unsigned long long mask,
                                                     unsigned long long key) {
  for (unsigned long long h = mix(key) & mask;; h = (h + 1) & mask) {
    const unsigned long long prev = atomicCAS(keys + h, kEmpty, key);
    if (prev == kEmpty || prev == key) return h;
  }
}

__device__ __forceinline__ long long find(const unsigned long long* keys,
                                          unsigned long long mask, unsigned long long key) {
  for (unsigned long long h = mix(key) & mask;; h = (h + 1) & mask) {
    const unsigned long long k = keys[h];
    if (k == key) return (long long)h;
    if (k == kEmpty) return -1;
  }
}

__global__ void fill_u64(unsigned long long* p, unsigned long long n, unsigned long long v) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void fill_u32(unsigned* p, unsigned long long n, unsigned v) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void insert_voxels(const int* vox, unsigned long long n, unsigned long long* keys,
                              unsigned long long mask, int* bad) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const int x = vox[3 * i], y = vox[3 * i + 1], z = vox[3 * i + 2];
    if (x < -kBias + 1 || x > kBias - 2 || y < -kBias + 1 || y > kBias - 2 || z < -kBias + 1 ||
        z > kBias - 2) {
      atomicOr(bad, 1);
      continue;
    }
    insert(keys, mask, pack(x, y, z));
  }
}

__global__ void face_flags(const int* vox, unsigned long long n, const unsigned long long* keys,
                           unsigned long long mask, unsigned* flags) {
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       t < 6 * n; t += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = t / 6;
    const int f = (int)(t - 6 * i);
    const unsigned long long nb = pack(vox[3 * i] + c_off[f][0], vox[3 * i + 1] + c_off[f][1],
                                       vox[3 * i + 2] + c_off[f][2]);
    flags[t] = find(keys, mask, nb) < 0 ? 1u : 0u;
  }
}

// exterior face slot -> (voxel, face) index t; every corner's minimum sequence number
__global__ void corner_first(const int* vox, unsigned long long n, const unsigned* flags,
                             const unsigned* slot, unsigned long long* face_src,
                             unsigned long long* ckeys, unsigned long long cmask,
                             unsigned* cfirst) {
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       t < 6 * n; t += (unsigned long long)gridDim.x * blockDim.x) {
    if (!flags[t]) continue;
    const unsigned long long i = t / 6;
    const int f = (int)(t - 6 * i);
    const unsigned s = slot[t];
    face_src[s] = t;
    for (int c = 0; c < 4; ++c) {
      const unsigned long long key =
          pack(vox[3 * i] + c_corner[f][c][0], vox[3 * i + 1] + c_corner[f][c][1],
               vox[3 * i + 2] + c_corner[f][c][2]);
      atomicMin(cfirst + insert(ckeys, cmask, key), 4u * s + (unsigned)c);
    }
  }
}

__device__ __forceinline__ unsigned long long corner_key(const int* vox, unsigned long long t,
                                                         int c) {
  const unsigned long long i = t / 6;
  const int f = (int)(t - 6 * i);
  return pack(vox[3 * i] + c_corner[f][c][0], vox[3 * i + 1] + c_corner[f][c][1],
              vox[3 * i + 2] + c_corner[f][c][2]);
}

__global__ void first_flags(const int* vox, unsigned long long n_faces,
                            const unsigned long long* face_src, const unsigned long long* ckeys,
                            unsigned long long cmask, const unsigned* cfirst, unsigned* is_first) {
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       s < 4 * n_faces; s += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long key = corner_key(vox, face_src[s >> 2], (int)(s & 3));
    is_first[s] = cfirst[find(ckeys, cmask, key)] == (unsigned)s ? 1u : 0u;
  }
}

__global__ void emit(const int* vox, unsigned long long n_faces,
                     const unsigned long long* face_src, const unsigned long long* ckeys,
                     unsigned long long cmask, const unsigned* cfirst, const unsigned* vid,
                     double res, double ox, double oy, double oz, double* verts,
                     unsigned* tris) {
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       s < n_faces; s += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long t = face_src[s];
    const unsigned long long i = t / 6;
    const int f = (int)(t - 6 * i);
    unsigned q[4];
    for (int c = 0; c < 4; ++c) {
      const int cx = vox[3 * i] + c_corner[f][c][0], cy = vox[3 * i + 1] + c_corner[f][c][1],
                cz = vox[3 * i + 2] + c_corner[f][c][2];
      const unsigned first = cfirst[find(ckeys, cmask, pack(cx, cy, cz))];
      q[c] = vid[first];
      if (first == 4u * (unsigned)s + (unsigned)c) {  // voxel_corner (geometry.hpp)
        verts[3ull * q[c] + 0] = __dadd_rn(ox, __dmul_rn(res, (double)cx));
        verts[3ull * q[c] + 1] = __dadd_rn(oy, __dmul_rn(res, (double)cy));
        verts[3ull * q[c] + 2] = __dadd_rn(oz, __dmul_rn(res, (double)cz));
      }
    }
    unsigned* tr = tris + 6 * s;
    tr[0] = q[0];
    tr[1] = q[1];
    tr[2] = q[2];
    tr[3] = q[0];
    tr[4] = q[2];
    tr[5] = q[3];
  }
}

unsigned long long pow2_at_least(unsigned long long x) {
  unsigned long long p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct Scratch {
  cudaStream_t s;
  void* ptrs[16] = {};
  int n = 0;
  cudaError_t err = cudaSuccess;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    if (err == cudaSuccess) err = cudaMallocAsync(&p, count * sizeof(T) + 16, s);
    if (err == cudaSuccess) ptrs[n++] = p;
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], s);
  }
};

int grid_for(unsigned long long n) {
  const unsigned long long b = (n + 255) / 256;
  return (int)(b < 148ull * 16 ? (b ? b : 1) : 148ull * 16);
}

}  // namespace

namespace b3d200 {

// Returns cudaSuccess, or cudaErrorInvalidValue for coordinates outside
// [-2^20 + 1, 2^20 - 2] (the packed-key range).  d_vox: device int32 n x 3;
// d_verts / d_tris: device, capacity 8n x 3 doubles / 12n x 3 uint32.
cudaError_t voxel_to_mesh_device(const int* d_vox, unsigned long long n, double res,
                                 const double origin[3], double* d_verts, unsigned* d_tris,
                                 unsigned long long* n_vertices, unsigned long long* n_triangles,
                                 cudaStream_t stream) {
  Scratch sc{stream};
  const unsigned long long vcap = pow2_at_least(2 * n + 16), vmask = vcap - 1;
  unsigned long long* vkeys = sc.get<unsigned long long>(vcap);
  unsigned* flags = sc.get<unsigned>(6 * n + 1);
  unsigned* slot = sc.get<unsigned>(6 * n + 1);
  int* bad = sc.get<int>(1);
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, slot, (int)(6 * n + 1), stream);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, flags, slot, (int)(24 * n + 1), stream);
  void* tmp = sc.get<char>(tmp_bytes > tmp2 ? tmp_bytes : tmp2);
  if (sc.err != cudaSuccess) return sc.err;
  if (6 * n + 1 > 0x7fffffffull / 4) return cudaErrorInvalidValue;
  fill_u64<<<grid_for(vcap), 256, 0, stream>>>(vkeys, vcap, kEmpty);
  cudaMemsetAsync(bad, 0, sizeof(int), stream);
  insert_voxels<<<grid_for(n), 256, 0, stream>>>(d_vox, n, vkeys, vmask, bad);
  face_flags<<<grid_for(6 * n), 256, 0, stream>>>(d_vox, n, vkeys, vmask, flags);
  cudaMemsetAsync(flags + 6 * n, 0, sizeof(unsigned), stream);
  size_t tb = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, tb, flags, slot, (int)(6 * n + 1), stream);
  unsigned n_faces = 0;
  int h_bad = 0;
  cudaMemcpyAsync(&n_faces, slot + 6 * n, sizeof(unsigned), cudaMemcpyDeviceToHost, stream);
  cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, stream);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  if (h_bad) return cudaErrorInvalidValue;

  const unsigned long long nc = 4ull * n_faces;
  const unsigned long long ccap = pow2_at_least(2 * nc + 16), cmask = ccap - 1;
  unsigned long long* ckeys = sc.get<unsigned long long>(ccap);
  unsigned* cfirst = sc.get<unsigned>(ccap);
  unsigned long long* face_src = sc.get<unsigned long long>(n_faces + 1);
  unsigned* is_first = sc.get<unsigned>(nc + 1);
  unsigned* vid = sc.get<unsigned>(nc + 1);
  if (sc.err != cudaSuccess) return sc.err;
  fill_u64<<<grid_for(ccap), 256, 0, stream>>>(ckeys, ccap, kEmpty);
  fill_u32<<<grid_for(ccap), 256, 0, stream>>>(cfirst, ccap, 0xffffffffu);
  corner_first<<<grid_for(6 * n), 256, 0, stream>>>(d_vox, n, flags, slot, face_src, ckeys, cmask,
                                                    cfirst);
  first_flags<<<grid_for(nc), 256, 0, stream>>>(d_vox, n_faces, face_src, ckeys, cmask, cfirst,
                                                is_first);
  cudaMemsetAsync(is_first + nc, 0, sizeof(unsigned), stream);
  tb = tmp_bytes > tmp2 ? tmp_bytes : tmp2;
  cub::DeviceScan::ExclusiveSum(tmp, tb, is_first, vid, (int)(nc + 1), stream);
  emit<<<grid_for(n_faces), 256, 0, stream>>>(d_vox, n_faces, face_src, ckeys, cmask, cfirst, vid,
                                              res, origin[0], origin[1], origin[2], d_verts,
                                              d_tris);
  unsigned nv = 0;
  cudaMemcpyAsync(&nv, vid + nc, sizeof(unsigned), cudaMemcpyDeviceToHost, stream);
  e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *n_vertices = nv;
  *n_triangles = 2ull * n_faces;
  return cudaSuccess;
}

}  // namespace b3d200
