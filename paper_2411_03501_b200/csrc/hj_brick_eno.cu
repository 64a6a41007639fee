// hj_brick_eno.cu -- ENO3 / ENO2 / first-order instantiations of the brick-tiled fused stage.
#include "hj_brick.cuh"

namespace hj {
cudaError_t launch_brick_eno(int scheme, const StageArgs& P, cudaStream_t s, bool* handled) {
  switch (scheme) {
    case HJ_ENO3: return launch_brick_ham<HJ_ENO3, 2>(P, s, handled);
    case HJ_ENO2: return launch_brick_ham<HJ_ENO2, 2>(P, s, handled);
    default: return launch_brick_ham<HJ_FIRST, 2>(P, s, handled);
  }
}
}  // namespace hj
