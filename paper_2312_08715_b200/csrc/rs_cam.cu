// Camera-mode kernel instantiations (render_score.cuh): a multi-instance
// scene rendered (and scored) under per-hypothesis camera poses.
#include "render_score.cuh"

namespace b3d200 {
B3D_RS_CAM_KERNELS()
}  // namespace b3d200

#if B3D_PHASE_CLOCK  // diagnostic builds: scripts/phase_probe.py
extern "C" __attribute__((visibility("default"))) int b3d_debug_phase_clock(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, b3d200::g_phase, sizeof(b3d200::g_phase));
}
#endif
