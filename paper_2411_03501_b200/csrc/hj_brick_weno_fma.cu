// hj_brick_weno_fma.cu -- tolerance-mode WENO5 (HJ_WENO5_FMA) instantiations of the
// brick-tiled fused stage (hj_brick.cuh).
#include "hj_brick.cuh"

namespace hj {
cudaError_t launch_brick_weno5_fma(const StageArgs& P, cudaStream_t s, bool* handled, int variant) {
  // walks unrolled by 4 = the window's rotation period (no register moves,
  // independent steps interleave): +6% (x2) and +3% more (x4) over rolled;
  // "brick_u2" selects the x2 unroll for A/B runs
  if (variant == 4) return launch_brick_ham<HJ_WENO5_FMA, 2, 2>(P, s, handled);
  return launch_brick_ham<HJ_WENO5_FMA, 2, 4>(P, s, handled);
}
}  // namespace hj
