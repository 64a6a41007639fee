// hj_stage_adv.cu -- generic fused stage kernel instantiations (see hj_stage_generic.cuh).
#include "hj_tile.cuh"

namespace hj {
cudaError_t launch_stage_adv(int scheme, const StageArgs& P, cudaStream_t s) {
  const int dim = P.g.dim;
  if (dim == 1) return launch_stage_s<1, HJ_HAM_ADVECTION>(scheme, P, s);
  if (dim == 2) return launch_stage_s<2, HJ_HAM_ADVECTION>(scheme, P, s);
  if (dim == 3) return launch_stage_s<3, HJ_HAM_ADVECTION>(scheme, P, s);
  return launch_stage_s<4, HJ_HAM_ADVECTION>(scheme, P, s);
}
cudaError_t launch_persist_adv(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  const int dim = P.g.dim;
  if (dim == 1) return launch_persist_s<1, HJ_HAM_ADVECTION>(scheme, P, A, s);
  if (dim == 2) return launch_persist_s<2, HJ_HAM_ADVECTION>(scheme, P, A, s);
  if (dim == 3) return launch_tile_persist_s<HJ_HAM_ADVECTION>(scheme, P, A, s);
  return launch_persist_s<4, HJ_HAM_ADVECTION>(scheme, P, A, s);
}
cudaError_t launch_tile_adv(int scheme, const StageArgs& P, cudaStream_t s) {
  return launch_tile_s<HJ_HAM_ADVECTION>(scheme, P, s);
}
}  // namespace hj
