// hj_brick_weno.cu -- WENO5 instantiations of the brick-tiled fused stage (hj_brick.cuh).
#include "hj_brick.cuh"

namespace hj {
cudaError_t launch_brick_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int variant) {
  if (variant == 2) return launch_brick_ham<HJ_WENO5, 1, 4>(P, s, handled);   // "brick1"
  if (variant == 4) return launch_brick_ham<HJ_WENO5, 2, 2>(P, s, handled);   // "brick_u2"
  return launch_brick_ham<HJ_WENO5, 2>(P, s, handled);
}
}  // namespace hj
