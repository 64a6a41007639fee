// hj_brick_weno.cu -- WENO5 instantiations of the brick-tiled fused stage (hj_brick.cuh).
#include "hj_brick.cuh"

namespace hj {
cudaError_t launch_brick_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int variant) {
  if (variant == 2) return launch_brick_ham<HJ_WENO5, 1, 4>(P, s, handled);      // "brick1"
  if (variant == 4) return launch_brick_ham<HJ_WENO5, 2, 1, 1>(P, s, handled);   // "brick_u2": rolled walks (A/B)
  if (variant == 7) return launch_brick_ham<HJ_WENO5, 2, 2, 1 | UNR_PREREG>(P, s, handled);   // "brick_x": A/B slot
  // 3-D walks unrolled x2 (+1.4% at 301^3), 4-D walks rolled (x2 costs 5% on 121^4)
  return launch_brick_ham<HJ_WENO5, 2, 2, 1>(P, s, handled);
}
}  // namespace hj
