// hj_axes_weno.cu -- WENO5 instantiations of the per-axis walk pipeline (hj_axes.cuh).
#include "hj_axes.cuh"

namespace hj {
cudaError_t launch_axes_weno5(const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = true;
  double* scratch = P.aux0;
  if (P.g.dim == 4) {
    if (P.ham.kind == HJ_HAM_DI4) return launch_axes_t<HJ_WENO5, HJ_HAM_DI4, 4>(P, s, scratch);
    return launch_axes_t<HJ_WENO5, HJ_HAM_ADVECTION, 4>(P, s, scratch);
  }
  switch (P.ham.kind) {
    case HJ_HAM_AIR3D: return launch_axes_t<HJ_WENO5, HJ_HAM_AIR3D, 3>(P, s, scratch);
    case HJ_HAM_ROCKETS: return launch_axes_t<HJ_WENO5, HJ_HAM_ROCKETS, 3>(P, s, scratch);
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_axes_t<HJ_WENO5, HJ_HAM_ROCKETS_EXTREMAL, 3>(P, s, scratch);
    default: return launch_axes_t<HJ_WENO5, HJ_HAM_ADVECTION, 3>(P, s, scratch);
  }
}
}  // namespace hj
