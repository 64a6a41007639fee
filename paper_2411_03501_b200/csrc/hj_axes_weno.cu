// hj_axes_weno.cu -- WENO5 instantiations of the per-axis walk pipeline (hj_axes.cuh).
#include "hj_axes.cuh"

namespace hj {
int axes_unroll();   // hj_fast.cu

template <int SEGC>
static cudaError_t axes_weno5(const StageArgs& P, cudaStream_t s, int parts) {
  double* scratch = P.aux0;
  // A/B variants (the C2 / C4 / C5 Hamiltonians only): every walk rolled (the
  // round-2 r02g pipeline), or the contiguous-axis walk unrolled as well
  switch (P.ham.kind == HJ_HAM_DI4 || P.ham.kind == HJ_HAM_AIR3D ? axes_unroll() : -1) {
    case 0:
      if (P.g.dim == 4) return launch_axes_t<HJ_WENO5, HJ_HAM_DI4, 4, SEGC, 0>(P, s, scratch, parts);
      return launch_axes_t<HJ_WENO5, HJ_HAM_AIR3D, 3, SEGC, 0>(P, s, scratch, parts);
    case 5:
      if (P.g.dim == 4) return launch_axes_t<HJ_WENO5, HJ_HAM_DI4, 4, SEGC, 5>(P, s, scratch, parts);
      return launch_axes_t<HJ_WENO5, HJ_HAM_AIR3D, 3, SEGC, 5>(P, s, scratch, parts);
    case 20:
      if (P.g.dim == 4) return launch_axes_t<HJ_WENO5, HJ_HAM_DI4, 4, SEGC, 20>(P, s, scratch, parts);
      return launch_axes_t<HJ_WENO5, HJ_HAM_AIR3D, 3, SEGC, 20>(P, s, scratch, parts);
    default: break;
  }
  if (P.g.dim == 4) {
    if (P.ham.kind == HJ_HAM_DI4) return launch_axes_t<HJ_WENO5, HJ_HAM_DI4, 4, SEGC>(P, s, scratch, parts);
    return launch_axes_t<HJ_WENO5, HJ_HAM_ADVECTION, 4, SEGC>(P, s, scratch, parts);
  }
  switch (P.ham.kind) {
    case HJ_HAM_AIR3D: return launch_axes_t<HJ_WENO5, HJ_HAM_AIR3D, 3, SEGC>(P, s, scratch, parts);
    case HJ_HAM_ROCKETS: return launch_axes_t<HJ_WENO5, HJ_HAM_ROCKETS, 3, SEGC>(P, s, scratch, parts);
    case HJ_HAM_ROCKETS_EXTREMAL:
      return launch_axes_t<HJ_WENO5, HJ_HAM_ROCKETS_EXTREMAL, 3, SEGC>(P, s, scratch, parts);
    default: return launch_axes_t<HJ_WENO5, HJ_HAM_ADVECTION, 3, SEGC>(P, s, scratch, parts);
  }
}

// Column kernels walk 32-node segments (AX_SEGC), the contiguous-axis kernel
// 16-node ones (AX_SEG): with 128-thread CTAs the halved window-fill work
// pays (A/B on one B200: C2 +1.2 %, C4 +2.8 %, C5 +0.9 %; with 256-thread
// CTAs it had measured +1.5 % C4, -1.8 % C5, -0.2 % C2)
constexpr int AX_SEGC = 2 * AX_SEG;

cudaError_t launch_axes_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int parts) {
  *handled = true;
  if (axes_unroll() == 64 && (P.ham.kind == HJ_HAM_DI4 || P.ham.kind == HJ_HAM_AIR3D))   // A/B "axes_s16"
    return P.g.dim == 4 ? launch_axes_t<HJ_WENO5, HJ_HAM_DI4, 4, AX_SEG>(P, s, P.aux0, parts)
                        : launch_axes_t<HJ_WENO5, HJ_HAM_AIR3D, 3, AX_SEG>(P, s, P.aux0, parts);
  return axes_weno5<AX_SEGC>(P, s, parts);
}
}  // namespace hj
