// hj_stage.cu -- stage dispatch plus the unfused derivative / workspace
// kernels behind the spatial API (spatial.py:119-276).
#include "hj_kernels.cuh"

namespace hj {

// derivative_pair along one axis (spatial.py:268-276)
template <int SCHEME>
__global__ void __launch_bounds__(256) k_derivs(const GridArgs G, int axis, int eps_mode,
                                                const double* __restrict__ v, double* __restrict__ left,
                                                double* __restrict__ right) {
  constexpr int W = Width<SCHEME>::value;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= G.cells * G.batch) return;
  int ix[HJ_MAX_DIM];
  const long long off = locate(G, idx, ix);
  const AxisView& A = G.ax[axis];
  const double* line = v + (off - (long long)ix[axis] * A.stride);
  double u[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    if (k >= 3 - W && k <= 3 + W) u[k] = fetch(line, A, ix[axis] - 3 + k);
    else u[k] = 0.0;
  }
  const LR lr = scheme_lr<SCHEME>(u, G.sp[axis], eps_mode);
  left[off] = lr.l;
  right[off] = lr.r;
}

// weno5_workspace (spatial.py:250-257): 10 diagnostic fields of one side
__global__ void __launch_bounds__(256) k_weno_ws(const GridArgs G, int axis, int side, int eps_mode,
                                                 const double* __restrict__ v, double* __restrict__ ws) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = G.cells * G.batch;
  if (idx >= total) return;
  int ix[HJ_MAX_DIM];
  const long long off = locate(G, idx, ix);
  const AxisView& A = G.ax[axis];
  const double* line = v + (off - (long long)ix[axis] * A.stride);
  double u[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) u[k] = fetch(line, A, ix[axis] - 3 + k);
  const double h = G.sp[axis].h;
  double f[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) f[k] = (u[k + 1] - u[k]) / h;
  WenoDiag d;
  if (side == 0) weno_side<true>(f[0], f[1], f[2], f[3], f[4], eps_mode, &d);
  else weno_side<true>(f[5], f[4], f[3], f[2], f[1], eps_mode, &d);
  const double vals[10] = {d.sigma1, d.sigma2, d.sigma3, d.alpha1, d.alpha2,
                           d.alpha3, d.eps, d.w1, d.w2, d.w3};
#pragma unroll
  for (int k = 0; k < 10; ++k) ws[(long long)k * total + idx] = vals[k];
}

cudaError_t launch_stage_adv(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_stage_rockets(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_stage_air3d(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_stage_di4(int scheme, const StageArgs& P, cudaStream_t s);

cudaError_t launch_stage_generic(int scheme, const StageArgs& P, cudaStream_t s) {
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: return launch_stage_adv(scheme, P, s);
    case HJ_HAM_ROCKETS:
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_stage_rockets(scheme, P, s);
    case HJ_HAM_AIR3D: return launch_stage_air3d(scheme, P, s);
    default: return launch_stage_di4(scheme, P, s);
  }
}

cudaError_t launch_persist_adv(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s);
cudaError_t launch_persist_rockets(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s);
cudaError_t launch_persist_air3d(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s);
cudaError_t launch_persist_di4(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s);

cudaError_t launch_persist(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: return launch_persist_adv(scheme, P, A, s);
    case HJ_HAM_ROCKETS:
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_persist_rockets(scheme, P, A, s);
    case HJ_HAM_AIR3D: return launch_persist_air3d(scheme, P, A, s);
    default: return launch_persist_di4(scheme, P, A, s);
  }
}

cudaError_t launch_tile_adv(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_tile_rockets(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_tile_air3d(int scheme, const StageArgs& P, cudaStream_t s);

// small 3-D grids: the tile kernel (hj_tile.cuh); *handled = false for a
// Hamiltonian without a 3-D tile instantiation
cudaError_t launch_tile(int scheme, const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = P.g.dim == 3;
  if (!*handled) return cudaSuccess;
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: return launch_tile_adv(scheme, P, s);
    case HJ_HAM_ROCKETS:
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_tile_rockets(scheme, P, s);
    case HJ_HAM_AIR3D: return launch_tile_air3d(scheme, P, s);
    default: *handled = false; return cudaSuccess;
  }
}

cudaError_t launch_derivs(int scheme, const GridArgs& G, int axis, int eps_mode, const double* v,
                          double* left, double* right, cudaStream_t s) {
  const long long total = G.cells * G.batch;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  switch (scheme) {
    case HJ_FIRST: k_derivs<HJ_FIRST><<<blocks, 256, 0, s>>>(G, axis, eps_mode, v, left, right); break;
    case HJ_ENO2: k_derivs<HJ_ENO2><<<blocks, 256, 0, s>>>(G, axis, eps_mode, v, left, right); break;
    case HJ_ENO3: k_derivs<HJ_ENO3><<<blocks, 256, 0, s>>>(G, axis, eps_mode, v, left, right); break;
    case HJ_WENO5_FMA: k_derivs<HJ_WENO5_FMA><<<blocks, 256, 0, s>>>(G, axis, eps_mode, v, left, right); break;
    default: k_derivs<HJ_WENO5><<<blocks, 256, 0, s>>>(G, axis, eps_mode, v, left, right); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_weno_ws(const GridArgs& G, int axis, int side, int eps_mode, const double* v,
                           double* ws, cudaStream_t s) {
  const long long total = G.cells * G.batch;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  k_weno_ws<<<blocks, 256, 0, s>>>(G, axis, side, eps_mode, v, ws);
  return cudaGetLastError();
}

}  // namespace hj

namespace hj {
// Specialised fast kernels (hj_fast.cu) claim the configurations they cover;
// everything else runs the generic fused kernel above.
__attribute__((weak)) cudaError_t launch_stage_fast(int, const StageArgs&, cudaStream_t, bool* handled) {
  *handled = false;
  return cudaSuccess;
}
}  // namespace hj
