// hj_stage_di4.cu -- generic fused stage kernel instantiations (see hj_stage_generic.cuh).
#include "hj_stage_generic.cuh"

namespace hj {
cudaError_t launch_stage_di4(int scheme, const StageArgs& P, cudaStream_t s) {
  return launch_stage_s<4, HJ_HAM_DI4>(scheme, P, s);
}
cudaError_t launch_persist_di4(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  return launch_persist_s<4, HJ_HAM_DI4>(scheme, P, A, s);
}
}  // namespace hj
