// hj_stage_adv.cu -- generic fused stage kernel instantiations (see hj_stage_generic.cuh).
#include "hj_stage_generic.cuh"

namespace hj {
cudaError_t launch_stage_adv(int scheme, const StageArgs& P, cudaStream_t s) {
  const int dim = P.g.dim;
  if (dim == 1) return launch_stage_s<1, HJ_HAM_ADVECTION>(scheme, P, s);
  if (dim == 2) return launch_stage_s<2, HJ_HAM_ADVECTION>(scheme, P, s);
  if (dim == 3) return launch_stage_s<3, HJ_HAM_ADVECTION>(scheme, P, s);
  return launch_stage_s<4, HJ_HAM_ADVECTION>(scheme, P, s);
}
}  // namespace hj
