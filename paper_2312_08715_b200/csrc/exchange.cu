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

// One rank's barrier episode: announce `epoch` in slot `rank` of every pad,
// then wait (thread t) until slot t of this rank's pad holds it.
__device__ __forceinline__ void barrier_episode(const KBarrier& b, int t,
                                                unsigned long long timeout_ns) {
  __threadfence_system();
  if (t < b.n_ranks) st_release_sys(b.sig[t] + b.rank, b.epoch);
  if (t < b.n_ranks) {
    const unsigned long long* mine = b.sig[b.rank] + t;
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(mine) < b.epoch) {
      __nanosleep(64);
      if (global_ns() - t0 > timeout_ns) __trap();
    }
  }
  __syncwarp();
}

__global__ void shard_barrier_kernel(KBarrier b) {
  barrier_episode(b, threadIdx.x, 20000000000ull);
}

// The exchange protocol with every rank emulated by one block of one
// cooperative launch (ranks that wait on one another must run concurrently;
// separate launches on one GPU give no such guarantee).  Epoch e: rank r
// stores e * 16 + r into slot r of every rank's array -- half e & 1 when
// double-buffered, else half 0 -- as the score kernel's remote stores do,
// meets the others at the barrier, then reads its own half twice; one rank
// per epoch holds `hold_ns` between the reads (a slow reduction).  A value
// that is not epoch e's is a peer's next-epoch store that landed early.
__global__ void exchange_emulation_kernel(unsigned long long* sig, double* arr, int n_ranks,
                                          int rounds, int double_buffered,
                                          unsigned long long hold_ns, unsigned int* errors) {
  const int r = blockIdx.x, t = threadIdx.x;
  KBarrier b{};
  for (int q = 0; q < n_ranks; ++q) b.sig[q] = sig + 8 * q;
  b.n_ranks = n_ranks;
  b.rank = r;
  for (int e = 1; e <= rounds; ++e) {
    const int half = double_buffered ? (e & 1) : 0;
    if (t < n_ranks) arr[(t * 2 + half) * 8 + r] = (double)(e * 16 + r);
    b.epoch = (unsigned long long)e;
    barrier_episode(b, t, 2000000000ull);
    unsigned int bad = 0;
    if (t < n_ranks) {
      const volatile double* mine = arr + (r * 2 + half) * 8;
      const double want = (double)(e * 16 + t);
      bad += mine[t] != want;
      const unsigned long long t0 = global_ns();
      const unsigned long long hold = r == e % n_ranks ? hold_ns : 0ull;
      while (global_ns() - t0 < hold) __nanosleep(128);
      bad += mine[t] != want;
    }
    if (bad) atomicAdd(errors, bad);
    __syncwarp();
  }
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

cudaError_t launch_exchange_emulation(unsigned long long* sig, double* arr, int n_ranks,
                                      int rounds, int double_buffered,
                                      unsigned long long hold_ns, unsigned int* errors,
                                      cudaStream_t st) {
  void* args[] = {&sig, &arr, &n_ranks, &rounds, &double_buffered, &hold_ns, &errors};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(exchange_emulation_kernel),
                                     dim3(n_ranks), dim3(32), args, 0, st);
}

}  // namespace b3d200
