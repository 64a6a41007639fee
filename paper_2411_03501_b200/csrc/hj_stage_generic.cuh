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

// The per-stage inputs of one launch (the rest of StageArgs is per grid).
struct StageIO {
  const double* y_in;
  const double* y0;
  double* y_out;
  const double* mask_prev;
  double dt;
  int stage;
  int mask;
};

// One node of one fused stage.  CG: field loads through L2 only (the
// persistent kernel below reads fields other CTAs wrote in the same launch).
template <int DIM, int SCHEME, int HAM, bool CG>
__device__ __forceinline__ void stage_node(const StageArgs& P, const StageIO& io, long long idx, unsigned& flags,
                                           long long* lo, long long* hi) {
  constexpr int W = Width<SCHEME>::value;
  int ix[HJ_MAX_DIM];
  const long long off = locate(P.g, idx, ix);
  if (!P.zp.has(ix[0])) return;
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
    const double* line = io.y_in + (off - (long long)ix[a] * A.stride);
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      if (k >= 3 - W && k <= 3 + W)
      {
        if (inner) HJ_CHK(P, in, line + (long long)(ix[a] - 3 + k) * A.stride, 8);
        uu[a][k] = inner ? ldf<CG>(line + (long long)(ix[a] - 3 + k) * A.stride) : fetch<CG>(line, A, ix[a] - 3 + k);
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
  const double y = ldf<CG>(io.y_in + off);
  if (!finite(y)) flags |= HJ_NF_INPUT;
  const double y0 = (io.stage >= HJ_STAGE_RK2_AVG) ? ldf<CG>(io.y0 + off) : 0.0;
  double out = stage_update(io.stage, io.dt, y, y0, delta);
  if (io.mask == HJ_MASK_MIN) {
    const double pv = ldf<CG>(io.mask_prev + off);
    out = (pv < out) ? pv : out;
  } else if (io.mask == HJ_MASK_MAX) {
    const double pv = ldf<CG>(io.mask_prev + off);
    out = (pv > out) ? pv : out;
  }
  if (!finite(out)) flags |= HJ_NF_OUTPUT;
  HJ_CHK(P, out, io.y_out + off, 8);
  io.y_out[off] = out;
}

template <int DIM, int SCHEME, int HAM>
__global__ void __launch_bounds__(256) k_stage_generic(const StageArgs P) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = P.g.cells * P.g.batch;
  unsigned flags = 0u;
  long long lo[DIM], hi[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) { lo[a] = KEY_POS_INF; hi[a] = KEY_NEG_INF; }
  if (idx < total) {
    const StageIO io{P.y_in, P.y0, P.y_out, P.mask_prev, P.dt, P.stage, P.mask};
    stage_node<DIM, SCHEME, HAM, false>(P, io, idx, flags, lo, hi);
  }
  if (P.stats) reduce_stats<DIM>(P.stats, flags, P.tag, P.want_ranges != 0, lo, hi);
}

// ------------------------------------------------------------------ persistent integration
// Small grids (C1's 51x51x36: ~10 us per stage launch for 94 k nodes) are
// bound by per-launch latency, not by arithmetic.  The native integration
// loop (hj_integrate) therefore runs an interval's whole stage sequence in ONE
// cooperative launch: every CTA stays resident, walks its nodes of a stage,
// and meets the others at a grid barrier before the next stage reads them.
// The step schedule (dt per step, buffer rotation, mask on the interval's last
// stage, error tags) is computed on the host exactly as the per-stage loop
// computes it, so every node update is the same arithmetic, bit for bit.
// Grid-wide barrier of a co-resident (cooperative) grid, two-level: CTA b
// arrives on group counter b % BAR_GROUPS; the last arriver of a group
// arrives on the top counter; the last group releases everyone by bumping the
// generation word.  Each word has its own 128-byte line, so the arrivals of
// ~850 CTAs spread over 32 L2 lines instead of serialising on one (measured
// per barrier with one counter: 2.5-3.3 us at 740-888 CTAs,
// scripts/grid_barrier_probe.cu).  Stage outputs are plain stores; readers
// after the barrier load through L2 (ldf<true>), so no CTA sees a stale L1
// line.  Layout (unsigned words): [0] generation, [32 (1 + g)] group g,
// [32 (1 + BAR_GROUPS)] top; BAR_WORDS words, zeroed before each launch.
constexpr int BAR_GROUPS = 32;
constexpr int BAR_WORDS = 32 * (BAR_GROUPS + 2);
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x;
    const unsigned ngroups = nb < BAR_GROUPS ? nb : BAR_GROUPS;
    const unsigned grp = blockIdx.x % BAR_GROUPS;
    const unsigned gsize = nb / BAR_GROUPS + (grp < nb % BAR_GROUPS ? 1u : 0u);
    unsigned* gc = bar + 32 * (1 + grp);
    unsigned* top = bar + 32 * (1 + BAR_GROUPS);
    __threadfence();
    bool released = false;
    if (atomicAdd(gc, 1u) == gsize - 1) {
      atomicExch(gc, 0u);   // no member of this group arrives again before the release
      if (atomicAdd(top, 1u) == ngroups - 1) {
        atomicExch(top, 0u);
        __threadfence();
        atomicAdd(&bar[0], 1u);
        released = true;
      }
    }
    if (!released) {
      unsigned spins = 0;
      while (*(volatile unsigned*)&bar[0] == gen) {
        // ~2^28 polls (seconds): a scheduling bug ends the launch with an error instead of hanging
        if (++spins > (1u << 28)) asm volatile("trap;");
      }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

// 128-thread CTAs, register budget for 5 per SM (640 threads: C1's 94 k
// nodes are one node per thread on 148 SMs) for the first-order / ENO2
// schemes, 4 per SM for the wider stencils
constexpr int PERSIST_THREADS = 128;
template <int SCHEME>
struct PersistMinBlocks {
  static constexpr int value = (SCHEME == HJ_FIRST || SCHEME == HJ_ENO2) ? 5 : 4;
};

template <int DIM, int SCHEME, int HAM>
__global__ void __launch_bounds__(PERSIST_THREADS, PersistMinBlocks<SCHEME>::value)
    k_stage_persist(const __grid_constant__ StageArgs P, const __grid_constant__ PersistArgs A) {
  const long long total = P.g.cells * P.g.batch;
  const long long nth = (long long)gridDim.x * blockDim.x;
  unsigned gen = 0u;   // generations counted from the launcher's zeroed word
  long long lo[DIM], hi[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) { lo[a] = KEY_POS_INF; hi[a] = KEY_NEG_INF; }
  for (int s = 0; s < A.nstages; ++s) {
    const PersistStage& d = A.st[s];
    const StageIO io{A.buf[d.src], d.y0 >= 0 ? A.buf[d.y0] : nullptr, const_cast<double*>(A.buf[d.dst]),
                     A.mask_prev, d.dt, d.kind, d.mask};
    unsigned flags = 0u;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += nth)
      stage_node<DIM, SCHEME, HAM, true>(P, io, idx, flags, lo, hi);
    if (P.stats) reduce_stats<DIM>(P.stats, flags, d.tag, false, lo, hi);
    if (s + 1 < A.nstages) grid_barrier(A.bar, gen);
  }
}

// ------------------------------------------------------------------ launchers
template <int DIM, int SCHEME, int HAM>
static inline cudaError_t launch_stage_t(const StageArgs& P, cudaStream_t s) {
  const long long total = P.g.cells * P.g.batch;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  k_stage_generic<DIM, SCHEME, HAM><<<blocks, 256, 0, s>>>(P);
  return cudaGetLastError();
}

template <int DIM, int SCHEME, int HAM>
static inline cudaError_t launch_persist_t(const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  auto kern = k_stage_persist<DIM, SCHEME, HAM>;
  static std::atomic<int> occ[64];   // resident CTAs per SM, per device (0: not yet queried)
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = (dev >= 0 && dev < 64) ? occ[dev].load(std::memory_order_relaxed) : 0;
  if (per_sm <= 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PERSIST_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (per_sm <= 0) return cudaErrorInvalidConfiguration;
    if (dev >= 0 && dev < 64) occ[dev].store(per_sm, std::memory_order_relaxed);
  }
  const long long total = P.g.cells * P.g.batch;
  const long long want = (total + PERSIST_THREADS - 1) / PERSIST_THREADS;
  const long long cap = (long long)per_sm * sm_count(dev);
  const unsigned blocks = (unsigned)(want < cap ? want : cap);
  void* args[] = {const_cast<StageArgs*>(&P), const_cast<PersistArgs*>(&A)};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(blocks), dim3(PERSIST_THREADS), args, 0, s);
}

template <int DIM, int HAM>
static inline cudaError_t launch_persist_s(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  switch (scheme) {
    case HJ_FIRST: return launch_persist_t<DIM, HJ_FIRST, HAM>(P, A, s);
    case HJ_ENO2: return launch_persist_t<DIM, HJ_ENO2, HAM>(P, A, s);
    case HJ_ENO3: return launch_persist_t<DIM, HJ_ENO3, HAM>(P, A, s);
    case HJ_WENO5_FMA: return launch_persist_t<DIM, HJ_WENO5_FMA, HAM>(P, A, s);
    default: return launch_persist_t<DIM, HJ_WENO5, HAM>(P, A, s);
  }
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
