// hj_fast.cu -- routing of fused stages to the brick-tiled kernels.
#include <cstdlib>
#include <string>
#include "hj_kernels.cuh"

namespace hj {
cudaError_t launch_brick_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int variant);
cudaError_t launch_brick_eno(int scheme, const StageArgs& P, cudaStream_t s, bool* handled);

// HJ_STAGE_KERNEL selects the stage kernel for A/B measurements:
//   unset / "brick" : brick-tiled kernels, 2 CTAs per SM (default)
//   "brick1"        : brick-tiled WENO5 kernel compiled for 1 CTA per SM
//   "generic"       : per-node generic kernel everywhere
static int stage_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("HJ_STAGE_KERNEL");
    v = 1;
    if (e && std::string(e) == "generic") v = 0;
    if (e && std::string(e) == "brick1") v = 2;
  }
  return v;
}

// The brick kernels cover 3-D stages without range statistics whose grid
// fits the launch geometry; everything else runs the generic per-node kernel.
cudaError_t launch_stage_fast(int scheme, const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = false;
  const int variant = stage_variant();
  if (variant == 0 || (P.g.dim != 3 && P.g.dim != 4) || P.want_ranges) return cudaSuccess;
  if (scheme == HJ_WENO5) return launch_brick_weno5(P, s, handled, variant);
  return launch_brick_eno(scheme, P, s, handled);
}
}  // namespace hj
