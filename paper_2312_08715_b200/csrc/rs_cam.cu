// Camera-mode kernel instantiations (render_score.cuh): a multi-instance
// scene rendered (and scored) under per-hypothesis camera poses.
#include "render_score.cuh"

namespace b3d200 {
B3D_RS_CAM_KERNELS()
}  // namespace b3d200

B3D_PHASE_READER(b3d_debug_phase_clock)  // B3D_PHASE_CLOCK builds only
