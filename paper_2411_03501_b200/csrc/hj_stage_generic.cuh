// hj_stage_generic.cuh -- the generic fused grid-update kernel (one launch
// per TVD-RK stage), instantiated per Hamiltonian in hj_stage_*.cu.
//
// Fused pass per node (term.py:90-126 + integrator.py:92-103):
//   ghosts (grid.py:203-225) -> per-axis upwind pair (spatial.py:119-247)
//   -> p_avg = 0.5*(L+R) (term.py:101) -> H(x, p_avg) (device functor)
//   -> diss = sum (alpha_i*0.5)*(R_i-L_i) (term.py:84-86) -> delta = diss - H
//   -> stage update -> optional tube mask (reachability.py:249) -> store.
#pragma once
#include "hj_kernels.cuh"

namespace hj {

template <int DIM, int SCHEME, int HAM>
__global__ void __launch_bounds__(256) k_stage_generic(const StageArgs P) {
  constexpr int W = Width<SCHEME>::value;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = P.g.cells * P.g.batch;
  unsigned flags = 0u;
  long long lo[DIM], hi[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) { lo[a] = KEY_POS_INF; hi[a] = KEY_NEG_INF; }

  int ix[HJ_MAX_DIM];
  const long long off = idx < total ? locate(P.g, idx, ix) : 0;
  if (idx < total && P.zp.has(ix[0])) {
    double pbar[DIM];
    double diss = 0.0;
    // every stencil value of every axis first: a node whose stencils stay
    // inside the owned block takes them with plain loads, all in flight at
    // once (small grids are latency-bound); other nodes go through fetch()
    bool inner = true;
#pragma unroll
    for (int a = 0; a < DIM; ++a) inner = inner && ix[a] >= W && ix[a] < P.g.ax[a].n - W;
    double uu[DIM][7];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const AxisView& A = P.g.ax[a];
      const double* line = P.y_in + (off - (long long)ix[a] * A.stride);
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        if (k >= 3 - W && k <= 3 + W)
        {
          if (inner) HJ_CHK(P, in, line + (long long)(ix[a] - 3 + k) * A.stride, 8);
          uu[a][k] = inner ? line[(long long)(ix[a] - 3 + k) * A.stride] : fetch(line, A, ix[a] - 3 + k);
        }
        else
          uu[a][k] = 0.0;
      }
    }
    // ENO / first-order: every axis' quotients on the branch-free fast path
    // (independent chains the scheduler can interleave), one rarely taken
    // exact redo of the node; WENO5 keeps its per-division form here
    LR lrs[DIM];
    constexpr bool kFast = SCHEME == HJ_FIRST || SCHEME == HJ_ENO2 || SCHEME == HJ_ENO3;
    bool ok = kFast;
    if constexpr (kFast) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const EnoRecips K = eno_recips(P.g.sp[a]);
        if (SCHEME == HJ_FIRST) lrs[a] = scheme_first_q(uu[a], K, ok);
        else if (SCHEME == HJ_ENO2) lrs[a] = scheme_eno2_q(uu[a], P.g.sp[a], K, ok);
        else lrs[a] = scheme_eno3_q(uu[a], P.g.sp[a], K, ok);
      }
    }
    if (!ok) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) lrs[a] = scheme_lr<SCHEME>(uu[a], P.g.sp[a], P.eps_mode);
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const LR lr = lrs[a];
      if (!finite(lr.l) || !finite(lr.r)) flags |= HJ_NF_DERIV;
      if (P.want_ranges) {
        lo[a] = min(order_key(lr.l), order_key(lr.r));
        hi[a] = max(order_key(lr.l), order_key(lr.r));
      }
      pbar[a] = 0.5 * (lr.l + lr.r);
      diss = diss + P.alpha_half[a] * (lr.r - lr.l);
    }
    const double H = hamiltonian<HAM, DIM>(P.ham, P.g.nodes, ix, pbar);
    if (!finite(H)) flags |= HJ_NF_HAM;
    if (P.want_hnz && H != 0.0) flags |= HJ_FLAG_HAM_NONZERO;
    const double delta = diss - H;
    if (!finite(delta)) flags |= HJ_NF_DELTA;
    const double y = P.y_in[off];
    if (!finite(y)) flags |= HJ_NF_INPUT;
    const double y0 = (P.stage >= HJ_STAGE_RK2_AVG) ? P.y0[off] : 0.0;
    double out = stage_update(P.stage, P.dt, y, y0, delta);
    if (P.mask == HJ_MASK_MIN) {
      const double pv = P.mask_prev[off];
      out = (pv < out) ? pv : out;
    } else if (P.mask == HJ_MASK_MAX) {
      const double pv = P.mask_prev[off];
      out = (pv > out) ? pv : out;
    }
    if (!finite(out)) flags |= HJ_NF_OUTPUT;
    HJ_CHK(P, out, P.y_out + off, 8);
    P.y_out[off] = out;
  }
  if (P.stats) reduce_stats<DIM>(P.stats, flags, P.tag, P.want_ranges != 0, lo, hi);
}

// ------------------------------------------------------------------ launchers
template <int DIM, int SCHEME, int HAM>
static inline cudaError_t launch_stage_t(const StageArgs& P, cudaStream_t s) {
  const long long total = P.g.cells * P.g.batch;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  k_stage_generic<DIM, SCHEME, HAM><<<blocks, 256, 0, s>>>(P);
  return cudaGetLastError();
}

template <int DIM, int HAM>
static inline cudaError_t launch_stage_s(int scheme, const StageArgs& P, cudaStream_t s) {
  switch (scheme) {
    case HJ_FIRST: return launch_stage_t<DIM, HJ_FIRST, HAM>(P, s);
    case HJ_ENO2: return launch_stage_t<DIM, HJ_ENO2, HAM>(P, s);
    case HJ_ENO3: return launch_stage_t<DIM, HJ_ENO3, HAM>(P, s);
    case HJ_WENO5_FMA: return launch_stage_t<DIM, HJ_WENO5_FMA, HAM>(P, s);
    default: return launch_stage_t<DIM, HJ_WENO5, HAM>(P, s);
  }
}

}  // namespace hj
