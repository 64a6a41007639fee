// hj_tile.cuh -- the fused LF + TVD-RK stage for SMALL 3-D grids (fewer
// bricks than two per SM, e.g. C1's 51 x 51 x 36): one CTA of 128 threads per
// 4 x 4 x 8 tile of nodes, one node per thread.
//
// The per-node kernel (hj_stage_generic.cuh) spends ~1300 instructions per
// node at C1, 88 % of them integer: the linear index split into (i, j, k), the
// ghost logic of every stencil load, 64-bit addresses of 15 loads.  Here the
// CTA stages its tile with the stencil halo of each axis (the "plus" shape:
// core, plus up to 3 planes beyond each face, never edges or corners) in
// shared memory once -- boundary ghosts synthesised there by the rule of
// _extend_axis (grid.py:203-225, fetch) -- and every thread then reads its
// 7-point lines from shared memory with constant offsets.  The per-node
// arithmetic is the same functions, in the same order, as the per-node kernel
// (scheme fast path + exact redo, H, dissipation in axis order, stage update,
// mask), so the two are bit-identical.
#pragma once
#include "hj_stage_generic.cuh"

namespace hj {

constexpr int TLZ = 4, TLY = 4, TLX = 8;          // tile extents along axes 0, 1, 2
constexpr int TL_THREADS = TLZ * TLY * TLX;        // 128
constexpr int TLH = 3;                             // halo held per face (WENO5 / ENO3 width)
constexpr int TBX = TLX + 2 * TLH, TBY = TLY + 2 * TLH, TBZ = TLZ + 2 * TLH;
constexpr int TBOX = TBZ * TBY * TBX;              // 1400 doubles (11.2 KB)
// register budget: 6 resident CTAs per SM (768 threads) for the first-order /
// ENO2 schemes -- C1's 845 tiles are then one round on 148 SMs -- and 4 for
// the wider stencils (no spills)
template <int SCHEME>
struct TileMinBlocks {
  static constexpr int value = (SCHEME == HJ_FIRST || SCHEME == HJ_ENO2) ? 6 : 4;
};

__host__ __device__ __forceinline__ long long tile_count(const GridArgs& G) {
  return (long long)((G.n[0] + TLZ - 1) / TLZ) * ((G.n[1] + TLY - 1) / TLY) * ((G.n[2] + TLX - 1) / TLX) *
         G.batch;
}

// Stage of one tile.  CG: field loads through L2 only (persistent launches).
// Every thread of the CTA calls it; box is reused by the caller after a
// __syncthreads().
template <int SCHEME, int HAM, bool CG>
__device__ __forceinline__ void tile_stage(const StageArgs& P, const StageIO& io, long long tile,
                                           double* __restrict__ box, unsigned& flags) {
  constexpr int W = Width<SCHEME>::value;
  const GridArgs& G = P.g;
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];
  const long long s0 = G.stride[0], s1 = G.stride[1];
  const int ntx = (n2 + TLX - 1) / TLX, nty = (n1 + TLY - 1) / TLY, ntz = (n0 + TLZ - 1) / TLZ;
  long long t = tile;
  const int x0 = (int)(t % ntx) * TLX;
  t /= ntx;
  const int y0 = (int)(t % nty) * TLY;
  t /= nty;
  const int z0 = (int)(t % ntz) * TLZ;
  const long long b = t / ntz;
  const double* __restrict__ vin = io.y_in + b * G.batch_stride;

  // ---- stage the plus-shaped box: a position is read only as the stencil of
  // an in-domain tile node along ONE axis, so it is the core or lies in one of
  // the six face slabs (at most W deep): at most 6 positions per thread.
  // Positions in memory are loaded together (all in flight, then stored);
  // positions outside the domain along exactly one axis are that axis'
  // ghosts (fetch: periodic wrap, extrapolation, dirichlet, exchanged halo
  // planes); positions outside the domain along two axes are never read.
  constexpr int NPUT = 1 + (2 * TLH * TLY * TLX + TL_THREADS - 1) / TL_THREADS +
                       (2 * TLH * TLZ * TLX + TL_THREADS - 1) / TL_THREADS +
                       (2 * TLH * TLZ * TLY + TL_THREADS - 1) / TL_THREADS;
  const double* srcs[NPUT];   // slot k: the load of the k-th position (nullptr: none / ghost)
  int dsts[NPUT];
  // a tile whose stencils stay inside the domain (most of them) takes every
  // position from memory without the per-position domain tests
  const bool interior = x0 >= W && x0 + TLX + W <= n2 && y0 >= W && y0 + TLY + W <= n1 && z0 >= W &&
                        z0 + TLZ + W <= n0;
  auto put = [&](int k, int lz, int ly, int lx) {
    const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
    const int di = ((lz + TLH) * TBY + (ly + TLH)) * TBX + (lx + TLH);
    if (interior) {
      srcs[k] = vin + (gz * s0 + gy * s1 + gx);
      HJ_CHK(P, in, srcs[k], 8);
      dsts[k] = di;
      return;
    }
    const bool ix = gx >= 0 && gx < n2, iy = gy >= 0 && gy < n1, iz = gz >= 0 && gz < n0;
    if (ix && iy && iz) {
      srcs[k] = vin + (gz * s0 + gy * s1 + gx);
      HJ_CHK(P, in, srcs[k], 8);
      dsts[k] = di;
    } else if (!ix && iy && iz) {
      box[di] = fetch<CG>(vin + (gz * s0 + gy * s1), G.ax[2], gx);
    } else if (ix && !iy && iz) {
      box[di] = fetch<CG>(vin + (gz * s0 + gx), G.ax[1], gy);
    } else if (ix && iy && !iz) {
      box[di] = fetch<CG>(vin + (gy * s1 + gx), G.ax[0], gz);
    }
  };
  {
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < NPUT; ++k) srcs[k] = nullptr;
    int slot = 0;
    put(slot++, t / (TLY * TLX), (t / TLX) % TLY, t % TLX);               // core
    // first-axis faces: 2W planes of TLY x TLX
#pragma unroll
    for (int r = 0; r < (2 * TLH * TLY * TLX + TL_THREADS - 1) / TL_THREADS; ++r) {
      const int i = t + r * TL_THREADS;
      if (i < 2 * W * TLY * TLX) {
        const int k = i / (TLY * TLX), rem = i % (TLY * TLX);
        put(slot, k < W ? k - W : TLZ + k - W, rem / TLX, rem % TLX);
      }
      ++slot;
    }
    // second-axis faces: 2W rows of TLZ x TLX
#pragma unroll
    for (int r = 0; r < (2 * TLH * TLZ * TLX + TL_THREADS - 1) / TL_THREADS; ++r) {
      const int i = t + r * TL_THREADS;
      if (i < 2 * W * TLZ * TLX) {
        const int k = i / (TLZ * TLX), rem = i % (TLZ * TLX);
        put(slot, rem / TLX, k < W ? k - W : TLY + k - W, rem % TLX);
      }
      ++slot;
    }
    // third-axis faces: 2W columns of TLZ x TLY
#pragma unroll
    for (int r = 0; r < (2 * TLH * TLZ * TLY + TL_THREADS - 1) / TL_THREADS; ++r) {
      const int i = t + r * TL_THREADS;
      if (i < 2 * W * TLZ * TLY) {
        const int k = i / (TLZ * TLY), rem = i % (TLZ * TLY);
        put(slot, rem / TLY, rem % TLY, k < W ? k - W : TLX + k - W);
      }
      ++slot;
    }
    double vals[NPUT];
#pragma unroll
    for (int k = 0; k < NPUT; ++k)
      if (srcs[k]) vals[k] = ldf<CG>(srcs[k]);
#pragma unroll
    for (int k = 0; k < NPUT; ++k)
      if (srcs[k]) box[dsts[k]] = vals[k];
  }
  __syncthreads();

  // ---- one node per thread
  const int lx = threadIdx.x % TLX, ly = (threadIdx.x / TLX) % TLY, lz = threadIdx.x / (TLX * TLY);
  int ixs[HJ_MAX_DIM] = {z0 + lz, y0 + ly, x0 + lx, 0, 0};
  if (ixs[0] >= n0 || ixs[1] >= n1 || ixs[2] >= n2 || !P.zp.has(ixs[0])) return;
  const double* c = box + ((lz + TLH) * TBY + (ly + TLH)) * TBX + (lx + TLH);
  double uu[3][7];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const bool use = k >= 3 - W && k <= 3 + W;
    uu[0][k] = use ? c[(k - 3) * (TBY * TBX)] : 0.0;
    uu[1][k] = use ? c[(k - 3) * TBX] : 0.0;
    uu[2][k] = use ? c[k - 3] : 0.0;
  }
  LR lrs[3];
  constexpr bool kFast = SCHEME == HJ_FIRST || SCHEME == HJ_ENO2 || SCHEME == HJ_ENO3;
  bool ok = kFast;
  if constexpr (kFast) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const EnoRecips K = eno_recips(G.sp[a]);
      if (SCHEME == HJ_FIRST) lrs[a] = scheme_first_q(uu[a], K, ok);
      else if (SCHEME == HJ_ENO2) lrs[a] = scheme_eno2_q(uu[a], G.sp[a], K, ok);
      else lrs[a] = scheme_eno3_q(uu[a], G.sp[a], K, ok);
    }
  }
  if (!ok) {
#pragma unroll
    for (int a = 0; a < 3; ++a) lrs[a] = scheme_lr<SCHEME>(uu[a], G.sp[a], P.eps_mode);
  }
  double pbar[3];
  double diss = 0.0;
  unsigned big = 0u;   // largest exponent field of the node's checked values (finite <=> < 0x7FF00000)
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const LR lr = lrs[a];
    big = max(big, max(abs_hi(lr.l), abs_hi(lr.r)));
    pbar[a] = 0.5 * (lr.l + lr.r);                        // term.py:101
    diss = diss + P.alpha_half[a] * (lr.r - lr.l);        // term.py:84-86
  }
  const double H = hamiltonian<HAM, 3>(P.ham, G.nodes, ixs, pbar);
  if (P.want_hnz && H != 0.0) flags |= HJ_FLAG_HAM_NONZERO;
  const double delta = diss - H;                          // term.py:113
  const double y = c[0];
  const long long off = b * G.batch_stride + ixs[0] * s0 + ixs[1] * s1 + ixs[2];
  const double yz = (io.stage >= HJ_STAGE_RK2_AVG) ? ldf<CG>(io.y0 + off) : 0.0;
  double out = stage_update(io.stage, io.dt, y, yz, delta);
  if (io.mask == HJ_MASK_MIN) {
    const double pv = ldf<CG>(io.mask_prev + off);
    out = (pv < out) ? pv : out;
  } else if (io.mask == HJ_MASK_MAX) {
    const double pv = ldf<CG>(io.mask_prev + off);
    out = (pv > out) ? pv : out;
  }
  big = max(max(big, abs_hi(H)), max(max(abs_hi(delta), abs_hi(y)), abs_hi(out)));
  if (big >= 0x7FF00000u) {   // rare: the per-class flags (one compare on the common path)
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (!finite(lrs[a].l) || !finite(lrs[a].r)) flags |= HJ_NF_DERIV;
    if (!finite(H)) flags |= HJ_NF_HAM;
    if (!finite(delta)) flags |= HJ_NF_DELTA;
    if (!finite(y)) flags |= HJ_NF_INPUT;
    if (!finite(out)) flags |= HJ_NF_OUTPUT;
  }
  HJ_CHK(P, out, io.y_out + off, 8);
  io.y_out[off] = out;
}

template <int SCHEME, int HAM>
__global__ void __launch_bounds__(TL_THREADS, TileMinBlocks<SCHEME>::value) k_stage_tile(const StageArgs P) {
  __shared__ double box[TBOX];
  unsigned flags = 0u;
  const StageIO io{P.y_in, P.y0, P.y_out, P.mask_prev, P.dt, P.stage, P.mask};
  tile_stage<SCHEME, HAM, false>(P, io, blockIdx.x, box, flags);
  if (P.stats) {
    long long dummy[3] = {0, 0, 0};
    reduce_stats<3>(P.stats, flags, P.tag, false, dummy, dummy);
  }
}

// the persistent form (hj_integrate): every stage of the schedule over the
// CTA's tiles, a grid barrier between stages (hj_stage_generic.cuh)
template <int SCHEME, int HAM>
__global__ void __launch_bounds__(TL_THREADS, TileMinBlocks<SCHEME>::value)
    k_stage_tile_persist(const __grid_constant__ StageArgs P, const __grid_constant__ PersistArgs A) {
  __shared__ double box[TBOX];
  const long long ntiles = tile_count(P.g);
  unsigned gen = 0u;
  for (int s = 0; s < A.nstages; ++s) {
    const PersistStage& d = A.st[s];
    const StageIO io{A.buf[d.src], d.y0 >= 0 ? A.buf[d.y0] : nullptr, const_cast<double*>(A.buf[d.dst]),
                     A.mask_prev, d.dt, d.kind, d.mask};
    unsigned flags = 0u;
    for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
      tile_stage<SCHEME, HAM, true>(P, io, tl, box, flags);
      __syncthreads();
    }
    if (P.stats) {
      long long dummy[3] = {0, 0, 0};
      reduce_stats<3>(P.stats, flags, d.tag, false, dummy, dummy);
    }
    if (s + 1 < A.nstages) grid_barrier(A.bar, gen);
  }
}

template <int SCHEME, int HAM>
static inline cudaError_t launch_tile_t(const StageArgs& P, cudaStream_t s) {
  const long long n = tile_count(P.g);
  k_stage_tile<SCHEME, HAM><<<(unsigned)n, TL_THREADS, 0, s>>>(P);
  return cudaGetLastError();
}

template <int SCHEME, int HAM>
static inline cudaError_t launch_tile_persist_t(const StageArgs& P, const PersistArgs& A, cudaStream_t s) {
  auto kern = k_stage_tile_persist<SCHEME, HAM>;
  static std::atomic<int> occ[64];   // resident CTAs per SM, per device (0: not yet queried)
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = (dev >= 0 && dev < 64) ? occ[dev].load(std::memory_order_relaxed) : 0;
  if (per_sm <= 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TL_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (per_sm <= 0) return cudaErrorInvalidConfiguration;
    if (dev >= 0 && dev < 64) occ[dev].store(per_sm, std::memory_order_relaxed);
  }
  const long long want = tile_count(P.g);
  const long long cap = (long long)per_sm * sm_count(dev);
  const unsigned blocks = (unsigned)(want < cap ? want : cap);
  void* args[] = {const_cast<StageArgs*>(&P), const_cast<PersistArgs*>(&A)};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(blocks), dim3(TL_THREADS), args, 0, s);
}

template <int HAM>
static inline cudaError_t launch_tile_s(int scheme, const StageArgs& P, cudaStream_t s) {
  switch (scheme) {
    case HJ_FIRST: return launch_tile_t<HJ_FIRST, HAM>(P, s);
    case HJ_ENO2: return launch_tile_t<HJ_ENO2, HAM>(P, s);
    case HJ_ENO3: return launch_tile_t<HJ_ENO3, HAM>(P, s);
    case HJ_WENO5_FMA: return launch_tile_t<HJ_WENO5_FMA, HAM>(P, s);
    default: return launch_tile_t<HJ_WENO5, HAM>(P, s);
  }
}

template <int HAM>
static inline cudaError_t launch_tile_persist_s(int scheme, const StageArgs& P, const PersistArgs& A,
                                                cudaStream_t s) {
  switch (scheme) {
    case HJ_FIRST: return launch_tile_persist_t<HJ_FIRST, HAM>(P, A, s);
    case HJ_ENO2: return launch_tile_persist_t<HJ_ENO2, HAM>(P, A, s);
    case HJ_ENO3: return launch_tile_persist_t<HJ_ENO3, HAM>(P, A, s);
    case HJ_WENO5_FMA: return launch_tile_persist_t<HJ_WENO5_FMA, HAM>(P, A, s);
    default: return launch_tile_persist_t<HJ_WENO5, HAM>(P, A, s);
  }
}

}  // namespace hj
