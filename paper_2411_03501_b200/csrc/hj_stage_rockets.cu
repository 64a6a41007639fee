// hj_stage_rockets.cu -- generic fused stage kernel instantiations (see hj_stage_generic.cuh).
#include "hj_tile.cuh"

namespace hj {
cudaError_t launch_stage_rockets(int scheme, const StageArgs& P, cudaStream_t s) {
  if (P.ham.kind == HJ_HAM_ROCKETS) return launch_stage_s<3, HJ_HAM_ROCKETS>(scheme, P, s);
  return launch_stage_s<3, HJ_HAM_ROCKETS_EXTREMAL>(scheme, P, s);
}
cudaError_t launch_persist_rockets(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  if (P.ham.kind == HJ_HAM_ROCKETS) return launch_tile_persist_s<HJ_HAM_ROCKETS>(scheme, P, A, s);
  return launch_tile_persist_s<HJ_HAM_ROCKETS_EXTREMAL>(scheme, P, A, s);
}
cudaError_t launch_tile_rockets(int scheme, const StageArgs& P, cudaStream_t s) {
  if (P.ham.kind == HJ_HAM_ROCKETS) return launch_tile_s<HJ_HAM_ROCKETS>(scheme, P, s);
  return launch_tile_s<HJ_HAM_ROCKETS_EXTREMAL>(scheme, P, s);
}
}  // namespace hj
