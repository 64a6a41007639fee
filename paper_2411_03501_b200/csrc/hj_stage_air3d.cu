// hj_stage_air3d.cu -- generic fused stage kernel instantiations (see hj_stage_generic.cuh).
#include "hj_tile.cuh"

namespace hj {
cudaError_t launch_stage_air3d(int scheme, const StageArgs& P, cudaStream_t s) {
  return launch_stage_s<3, HJ_HAM_AIR3D>(scheme, P, s);
}
cudaError_t launch_persist_air3d(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  return launch_tile_persist_s<HJ_HAM_AIR3D>(scheme, P, A, s);
}
cudaError_t launch_tile_air3d(int scheme, const StageArgs& P, cudaStream_t s) {
  return launch_tile_s<HJ_HAM_AIR3D>(scheme, P, s);
}
}  // namespace hj
