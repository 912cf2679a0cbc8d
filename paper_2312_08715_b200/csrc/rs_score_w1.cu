// Score-kernel instantiations for window radius 1 (render_score.cuh).
#include "render_score.cuh"

namespace b3d200 {
B3D_RS_SCORE_KERNELS(, 1)
}  // namespace b3d200

B3D_PHASE_READER(b3d_debug_phase_clock_w1)  // B3D_PHASE_CLOCK builds only
