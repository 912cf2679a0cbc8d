// Camera-mode score kernels specialised for window radius 1 (the
// bench-tracking resolutions' default_window: 25 / 50 px -> 1, 100 -> 2,
// 200 -> 4), so the window taps unroll as in the object-mode kernels.
#include "render_score.cuh"

namespace b3d200 {
B3D_RS_SCORE_KERNELS2(, 1, true)
}  // namespace b3d200

B3D_PHASE_READER(b3d_debug_phase_clock_cam1)  // B3D_PHASE_CLOCK builds only
