// hj_stage_air3d.cu -- generic fused stage kernel instantiations (see hj_stage_generic.cuh).
#include "hj_stage_generic.cuh"

namespace hj {
cudaError_t launch_stage_air3d(int scheme, const StageArgs& P, cudaStream_t s) {
  return launch_stage_s<3, HJ_HAM_AIR3D>(scheme, P, s);
}
}  // namespace hj
