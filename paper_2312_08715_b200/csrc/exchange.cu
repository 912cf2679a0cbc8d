// exchange.cu -- the device side of the sharded stage exchange.
//
// Ranks own contiguous hypothesis shards (inference.cpp:290's fan-out split
// across GPUs).  The score kernel stores each score straight into every
// rank's copy of the global score array over NVLink (render_score.cuh, the
// all-gather fused into the scoring), then this barrier makes the ranks meet
// before each reduces its now-complete copy: rank `rank` announces `epoch` in
// slot `rank` of every rank's signal pad (release, system scope, after a
// system fence that orders its remote score stores before the flag) and waits
// until every slot of its own pad holds `epoch` (acquire).  Epochs only grow,
// so pads never need resetting.  A peer that never arrives traps the kernel
// after 20 s (the call then fails) instead of hanging the GPU.
#include <cstdint>

#include "b3d_kernels.cuh"

namespace b3d200 {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void shard_barrier_kernel(KBarrier b) {
  const int t = threadIdx.x;
  __threadfence_system();
  if (t < b.n_ranks) st_release_sys(b.sig[t] + b.rank, b.epoch);
  if (t < b.n_ranks) {
    const unsigned long long* mine = b.sig[b.rank] + t;
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(mine) < b.epoch) {
      __nanosleep(64);
      if (global_ns() - t0 > 20000000000ull) __trap();
    }
  }
  __syncwarp();
}

// scores computed off the fused path (chunked / fp64 launches) stored to the
// peers afterwards: the same elements the fused kernel would have written
__global__ void copy_to_peers_kernel(const double* src, long long n, double* p0, double* p1,
                                     double* p2, double* p3, double* p4, double* p5, double* p6,
                                     double* p7, int n_peers, long long offset, long long cap) {
  double* peers[8] = {p0, p1, p2, p3, p4, p5, p6, p7};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long g = offset + i;
    if (g >= cap) continue;
    const double v = src[i];
    for (int r = 0; r < n_peers; ++r) peers[r][g] = v;
  }
  __threadfence_system();
}

}  // namespace

cudaError_t launch_copy_to_peers(const double* src, long long n, double* const* peers,
                                 int n_peers, long long offset, long long cap, cudaStream_t st) {
  const long long b = (n + 255) / 256;
  copy_to_peers_kernel<<<(int)(b < 1024 ? (b > 0 ? b : 1) : 1024), 256, 0, st>>>(
      src, n, peers[0], peers[1], peers[2], peers[3], peers[4], peers[5], peers[6], peers[7],
      n_peers, offset, cap);
  return cudaGetLastError();
}

cudaError_t launch_shard_barrier(const KBarrier& b, cudaStream_t st) {
  shard_barrier_kernel<<<1, 32, 0, st>>>(b);
  return cudaGetLastError();
}

}  // namespace b3d200
