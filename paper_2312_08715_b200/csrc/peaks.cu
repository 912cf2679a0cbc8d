// peaks.cu -- measurement helper (not product): the non-FMA FP64 issue rate
// of this B200, the denominator of the render+score kernel's roofline
// (the kernel is FP64-pipe bound: no FMA contraction is allowed on the
// bit-exact raster path).  Built into _lib/libb3d_peaks.so.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

// kChains independent chains of alternating DMUL / DADD per thread.
__global__ void fp64_nofma_kernel(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      x[c] = __dmul_rn(x[c], a);
      x[c] = __dadd_rn(x[c], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int b3d_bench_fp64_rate(int device,
                                                                          double* ops_per_s) {
  if (cudaSetDevice(device) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_nofma_kernel<<<blocks, threads>>>(d, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fp64_nofma_kernel<<<blocks, threads>>>(d, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * kChains * (double)kIters * blocks * threads;
  *ops_per_s = ops / (best * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
