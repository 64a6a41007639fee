// hj_brick.cuh -- the fused LF + TVD-RK stage, brick-tiled, templated on the
// upwind scheme, the device Hamiltonian and the axis offset AO.
//
// AO = 0 (3-D grids): one CTA (256 threads, ~110 KB shared memory, 2 CTAs per
// SM, persistent over a brick sequence) owns an 8 x 16 x 16 brick of axes
// (0, 1, 2).  Per stage and brick:
//   load:   the brick's values, their axis-1/axis-2 halos and the 3+3 axis-0
//           halo planes go to shared memory (coalesced; exchanged halo planes
//           or boundary ghosts through fetch());
//   walks:  warps 0-3 walk the 16-node lines along the brick's second axis,
//           warps 4-7 those along its third (concurrently, one window fill
//           per 16 nodes), storing p_avg_a = 0.5*(L+R) and the dissipation
//           term d_a = (alpha_a*0.5)*(R_a-L_a) per node;
//   fused:  thread (y,x) then walks its 8-node column along the first axis
//           and, per node, sums d = ((0 + d_0) + d_1) + d_2 in the
//           reference's axis order (term.py:84-86), evaluates H(x, p_avg),
//           delta = d - H (term.py:113), the stage update
//           (integrator.py:93-103), the optional tube mask
//           (reachability.py:249), the non-finite flags, and stores the node
//           (coalesced across x; its global stage inputs fetched one node
//           ahead).
// AO = 1 (4-D grids): the brick covers axes (1, 2, 3) of one axis-0 slice;
// a pre-pass (k_axis0_walk) has already walked axis 0 and left p_avg0 and
// d0 in scratch, so the fused walk starts the dissipation sum from d0 and H
// receives four costates.
// The line walkers (hj_weno_line.cuh / hj_eno_line.cuh) are rolled loops with
// a register window that compute every face quantity of their line once.
#pragma once
#include "hj_eno_line.cuh"
#include "hj_kernels.cuh"
#include "hj_weno_line.cuh"

namespace hj {

#ifndef HJ_ZWALK_UNROLL
#define HJ_ZWALK_UNROLL 1
#endif
constexpr int BZ = 8;                  // brick depth along its first axis
constexpr int BYX = 16;                // brick edge along its other two axes
constexpr int SEG = 8;                 // nodes per first-axis walk (= BZ)
constexpr int LSEG = 16;               // nodes per second / third-axis walk (= BYX)
constexpr int HB = 3;                  // ghost width held in shared memory (WENO5/ENO3 need 3)
constexpr int SVP = BYX + 2 * HB + 1;  // 23: odd pitch (conflict-free LDS.64 across y-lanes)
constexpr int SVR = BYX + 2 * HB;      // 22 rows per plane
constexpr int PLANE = SVR * SVP;       // doubles per plane of v
constexpr int NODES = BZ * BYX * BYX;  // 2048 nodes per brick
constexpr int BRICK_THREADS = 256;
static_assert(SEG == BZ && LSEG == BYX, "each walk covers its whole brick edge");
static_assert(BZ * BYX == BRICK_THREADS / 2, "half the CTA walks the second axis, half the third");

struct BrickSmem {
  double v[BZ * PLANE];           // brick planes with halos of the second / third axis
  double zh[2 * HB * BYX * BYX];  // first-axis halo planes: 3 below, 3 above (interior)
  double p1[NODES];               // p_avg of the second / third brick axis (swizzled node index)
  double p2[NODES];
  double t1[NODES];               // dissipation terms (alpha_a*0.5)*(R_a-L_a) of those axes
  double t2[NODES];
  // ham_eval inputs of the brick: node coordinates along its three axes
  // [BZ | BYX | BYX], then the Hamiltonian's two tables along its third axis
  double crd[BZ + 4 * BYX];
  // y0 of the combination stages for the fused first-axis walk: a two-node
  // ring per thread, filled by cp.async two nodes ahead (slot (i & 1) holds
  // node i).  Register slots filled by plain loads stalled ~8 % of the
  // kernel's samples: the consuming move waited on the scoreboard of the
  // youngest refill load, issued just before it (ncu source page, r01).
  double qy[2 * BRICK_THREADS];
};
constexpr int CRD_Y = BZ, CRD_X = BZ + BYX, CRD_T0 = BZ + 2 * BYX, CRD_T1 = BZ + 3 * BYX;

// node (z, y, x) of the brick -> slot in the per-node arrays; the XOR keeps
// LDS/STS conflict-free whether the lanes of a warp vary x or y
__device__ __forceinline__ int swz(int z, int y, int x) { return (z * BYX + y) * BYX + (x ^ y); }

// UNR flags (A/B variants): the fused first-axis walk unrolled by 2; the 4-D
// pre-pass reading its columns from global memory through a register queue
// (32-node segments) instead of staging them in shared memory
constexpr int UNR_Z2 = 16, UNR_PREREG = 32;

// UNR: unroll of the WENO walk (the window rotates with period 4).  The walk
// covers the brick edge N but stops after the first nv nodes (nv < N on the
// partial bricks of the far faces: 121 = 7*16 + 9 nodes, the 4-D grid of
// C4, leaves 7 of the last brick's 16 nodes outside the domain -- their
// steps would only occupy the FP64 pipe).  The bound is warp-uniform: lanes
// of a walk warp share the walk axis' brick extent.
template <int SCHEME, int UNR, int N, class Load, class Emit>
__device__ __forceinline__ void line_walk(const Load& ld, const Spacing& sp, const Emit& emit, int nv) {
  if constexpr (SCHEME == HJ_WENO5) {
    weno5_line<UNR, N>(ld, nv, weno_divisors(sp.h), emit);
  } else if constexpr (SCHEME == HJ_WENO5_FMA) {
    weno5_fma_line<UNR, N>(ld, nv, sp.rh, emit);
  } else if constexpr (SCHEME == HJ_ENO3) {
    eno3_line(ld, min(nv, N), eno_divisors(sp), emit);
  } else if constexpr (SCHEME == HJ_ENO2) {
    eno2_line(ld, min(nv, N), eno_divisors(sp), emit);
  } else {
    first_line(ld, min(nv, N), eno_divisors(sp), emit);
  }
}

// The three grid axes a brick spans (AO, AO+1, AO+2) and its slice base.
template <int AO>
struct BrickView {
  int n0, n1, n2;
  long long s0, s1;
  int slices;   // independent 3-D slices: batch (x the launch's axis-0 planes when AO = 1)
  RowSet zr, zp;
  __device__ __forceinline__ explicit BrickView(const StageArgs& P) {
    const GridArgs& G = P.g;
    n0 = G.n[AO];
    n1 = G.n[AO + 1];
    n2 = G.n[AO + 2];
    s0 = G.stride[AO];
    s1 = G.stride[AO + 1];
    zr = P.zr;
    zp = P.zp;
    slices = AO ? G.batch * zp.cnt : G.batch;
  }
  // element offset of slice b from problem 0's first owned node
  __device__ __forceinline__ long long slice_base(const GridArgs& G, int b) const {
    if (AO == 0) return (long long)b * G.batch_stride;
    const int pb = b / zp.cnt, i0 = zp.map(b % zp.cnt);
    return (long long)pb * G.batch_stride + (long long)i0 * G.stride[0];
  }
};

struct BrickCoord {
  int z0, y0, x0, b;
};

template <int AO>
__device__ __forceinline__ BrickCoord brick_coord(const BrickView<AO>& V, int lin) {
  // AO = 0: the launch's brick rows along the first axis (V.zr); AO = 1: every row
  const int nbx = (V.n2 + BYX - 1) / BYX, nby = (V.n1 + BYX - 1) / BYX;
  const int nbz = AO ? (V.n0 + BZ - 1) / BZ : V.zr.cnt;
  BrickCoord c;
  c.x0 = (lin % nbx) * BYX;
  lin /= nbx;
  c.y0 = (lin % nby) * BYX;
  lin /= nby;
  c.z0 = (AO ? (lin % nbz) : V.zr.map(lin % nbz)) * BZ;
  c.b = lin / nbz;
  return c;
}

// L2 prefetch of a brick's rows, issued while the current brick computes:
// the stage input with its halos, and the per-node inputs of the fused
// first-axis walk (y0 of the combination stages, the tube mask's previous
// snapshot, the 4-D pre-pass scratch), which would otherwise be HBM misses
// inside the walk
template <int AO>
__device__ __forceinline__ void prefetch_brick(const StageArgs& P, const GridArgs& G, const BrickView<AO>& V,
                                               const BrickCoord& c, int t) {
  const long long sb = V.slice_base(G, c.b);
  const double* vb = P.y_in + sb;
  for (int r = t; r < (BZ + 2 * HB) * SVR; r += BRICK_THREADS) {
    const int z = r / SVR - HB, yy = r % SVR - HB;
    const int gz = c.z0 + z, gy = c.y0 + yy;
    if (gz < 0 || gz >= V.n0 || gy < 0 || gy >= V.n1) continue;
    const int gx = max(c.x0 - HB, 0);
    const double* p = vb + gz * V.s0 + gy * V.s1 + gx;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 16));
  }
  // per-node streams of the fused walk: one brick row (16 nodes) per thread and stream
  const int z = t / BYX, yy = t % BYX;   // BZ x BYX = 128 rows per stream
  const int gz = c.z0 + (z & (BZ - 1)), gy = c.y0 + yy;
  if (gz >= V.n0 || gy >= V.n1) return;
  const long long off = sb + (long long)gz * V.s0 + (long long)gy * V.s1 + c.x0;
  if (z < BZ) {   // threads 0-127: y0, then the 4-D pairs; 128-255: the mask's previous snapshot
    if (P.stage >= HJ_STAGE_RK2_AVG && P.y0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(P.y0 + off));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(P.y0 + off + 15));
    }
    if (AO && P.aux0) {   // 16 (p_avg0, d0) pairs = 256 B
      const double* p = P.aux0 + 2 * off;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 16));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 31));
    }
  } else if (P.mask != HJ_MASK_NONE && P.mask_prev) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(P.mask_prev + off));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(P.mask_prev + off + 15));
  }
}

// 8-byte global -> shared asynchronous copy (LDGSTS) and its completion wait
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <int SCHEME, int HAM, int MINB, int AO, int UNR>
__device__ __forceinline__ void stage_brick(const StageArgs& P, const BrickView<AO>& V, BrickSmem& S,
                                            const BrickCoord c, unsigned& flags, const BrickCoord* next,
                                            bool load);

template <int SCHEME, int HAM, int MINB, int AO, int UNR>
__global__ void __launch_bounds__(BRICK_THREADS, MINB) k_stage_brick(const StageArgs P, int nbricks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BrickSmem& S = *reinterpret_cast<BrickSmem*>(smem_raw);
  const BrickView<AO> V(P);
  unsigned flags = 0u;
  // persistent CTAs: bricks blockIdx.x, +gridDim.x, ... (neighbouring CTAs take
  // neighbouring bricks, so halo rows are shared through L2)
  for (int lin = blockIdx.x; lin < nbricks; lin += gridDim.x) {
    const BrickCoord c = brick_coord(V, lin);
    const int nxt = lin + gridDim.x;
    BrickCoord cn;
    if (nxt < nbricks) cn = brick_coord(V, nxt);
    stage_brick<SCHEME, HAM, MINB, AO, UNR>(P, V, S, c, flags, (nxt < nbricks && !P.no_prefetch) ? &cn : nullptr,
                                            !P.skip_loads || lin == (int)blockIdx.x);
    __syncthreads();   // shared memory is reused by the next brick
  }
  if (P.stats) {
    long long dummy[1] = {0};
    reduce_stats<1>(P.stats, flags, P.tag, false, dummy, dummy);
  }
}

template <int SCHEME, int HAM, int MINB, int AO, int UNR>
__device__ __forceinline__ void stage_brick(const StageArgs& P, const BrickView<AO>& V, BrickSmem& S,
                                            const BrickCoord c, unsigned& flags, const BrickCoord* next,
                                            bool load) {
  constexpr int WALK_UNROLL = UNR & 15;   // WENO walk unroll (removes window rotation moves)
  // the fused first-axis walk carries the whole per-node update in its body:
  // kept rolled, so the hot loops fit the instruction cache (ncu: 8 % of the
  // samples were no_instructions with both walks unrolled)
  constexpr int ZWALK_UNROLL = (UNR & UNR_Z2) ? 2 : HJ_ZWALK_UNROLL;
  const GridArgs& G = P.g;
  const AxisView& A0 = G.ax[AO];
  const AxisView& A1 = G.ax[AO + 1];
  const AxisView& A2 = G.ax[AO + 2];
  const int n0 = V.n0, n1 = V.n1, n2 = V.n2;
  const int z0 = c.z0, y0 = c.y0, x0 = c.x0;
  const long long base = V.slice_base(G, c.b);
  const double* __restrict__ vin = P.y_in + base;
  const long long s0 = V.s0, s1 = V.s1;
  const int t = threadIdx.x;

  const bool zin = (z0 >= HB || A0.halo_lo) && (z0 + BZ + HB <= n0 || A0.halo_hi);
  const bool interior = zin && z0 + BZ <= n0 && y0 >= HB && y0 + BYX + HB <= n1 && x0 >= HB && x0 + BYX + HB <= n2;
  // ---- load.  Warp w owns brick plane z = w: it walks the plane's 22 rows
  // (second-axis halo rows included) with one incrementing row pointer, lane
  // = third-axis position (halo columns included); plane corners are never
  // read and skipped.  Values in memory go global -> shared with cp.async
  // (8 B, no register staging, all in flight at once); on boundary bricks the
  // extrapolated / dirichlet ghosts are then synthesised from the landed edge
  // nodes (no synchronous global loads on the load path).
  if (load) {
    static_assert(BZ == BRICK_THREADS / 32, "one warp per brick plane");
    const int lane = t & 31, warp = t >> 5;
    const int z = warp, gz = z0 + z;
    const int gx = x0 - HB + lane;
    const bool xin = lane >= HB && lane < HB + BYX;
    const bool lane_on = lane < SVR;
    const bool gx_in = gx >= 0 && gx < n2;
    double* srow = &S.v[z * PLANE + lane];
    if (interior) {
      const double* grow = vin + (gz * s0 + (y0 - HB) * s1 + gx);
#pragma unroll 2
      for (int yy = 0; yy < SVR; ++yy, grow += s1, srow += SVP) {
        const bool yin = yy >= HB && yy < HB + BYX;
        if (lane_on && (yin || xin)) { HJ_CHK(P, in, grow, 8); cp_async8(srow, grow); }
      }
    } else {
      // boundary brick, phase 1: every value that lives in memory (in-domain,
      // periodic wrap, exchanged halo planes) goes through cp.async; the
      // extrapolated / dirichlet ghosts wait for their edge nodes (phase 2)
      // (slots no walk reads -- outside the domain on both walk axes, planes
      // beyond the exchanged halos -- are left untouched)
      const int jx = gx_in ? gx : ghost_index(A2, gx);   // this lane's column: in memory or GI_SYNTH
      const int jz = ghost_index(A0, gz);
      const bool xmem = lane_on && jx != GI_SYNTH;
      const int r_lo = max(0, HB - y0), r_hi = min(SVR, n1 - y0 + HB);   // rows with gy in the domain
      if (gz < n0) {
        if (xmem) {
          // in-domain rows: one incrementing row pointer, as on interior bricks
          const double* grow = vin + ((long long)gz * s0 + (long long)(y0 - HB + r_lo) * s1 + jx);
          double* dst = &S.v[z * PLANE + r_lo * SVP + lane];
          for (int yy = r_lo; yy < r_hi; ++yy, grow += s1, dst += SVP)
            if (xin || (yy >= HB && yy < HB + BYX)) { HJ_CHK(P, in, grow, 8); cp_async8(dst, grow); }
          // ghost rows of a periodic second axis (their images live in memory),
          // read by the second-axis walk at the brick's own columns only
          if (A1.bc == HJ_BC_PERIODIC && xin && (r_lo > 0 || r_hi < SVR)) {
            for (int yy = 0; yy < SVR; ++yy) {
              if (yy >= r_lo && yy < r_hi) continue;
              const int jy = ghost_index(A1, y0 + yy - HB);
              const double* src = vin + ((long long)gz * s0 + (long long)jy * s1 + jx);
              HJ_CHK(P, in, src, 8);
              cp_async8(&S.v[z * PLANE + yy * SVP + lane], src);
            }
          }
        }
      } else if (jz != GI_SYNTH && jz != GI_ZERO && xin && gx_in) {
        // beyond the last plane of a partial brick, a plane that lives in memory
        // (periodic image / exchanged halo): the first-axis walk's columns
        const int ya = max(r_lo, HB), yb = min(r_hi, HB + BYX);
        const double* grow = vin + ((long long)jz * s0 + (long long)(y0 - HB + ya) * s1 + gx);
        double* dst = &S.v[z * PLANE + ya * SVP + lane];
        for (int yy = ya; yy < yb; ++yy, grow += s1, dst += SVP) {
          HJ_CHK(P, in, grow, 8);
          cp_async8(dst, grow);
        }
      }
      // first-axis halo planes (interior rows and columns of the brick only)
      const int half = lane >> 4, xl = lane & (BYX - 1);
#pragma unroll
      for (int r2 = warp; r2 < HB * BYX; r2 += BRICK_THREADS / 32) {
        const int row = 2 * r2 + half;
        const int k = row / BYX, y = row % BYX;
        const int e = (k < HB) ? (z0 - HB + k) : (z0 + BZ + k - HB);
        const int je = ghost_index(A0, e);
        const int gy = y0 + y, gxx = x0 + xl;
        double* dst = &S.zh[row * BYX + xl];
        if (gy >= n1 || gxx >= n2 || je == GI_ZERO) *dst = 0.0;
        else if (je != GI_SYNTH) {
          HJ_CHK(P, in, vin + ((long long)je * s0 + gy * s1 + gxx), 8);
          cp_async8(dst, vin + ((long long)je * s0 + gy * s1 + gxx));
        }
      }
      cp_async_wait_all();
      __syncthreads();
      // phase 2: synthesise the remaining ghosts from the landed edge nodes
      // plane value at relative first-axis index r (-HB..BZ+HB-1) for an
      // interior (y, x) of the brick, from S.v or the zh planes
      auto pz = [&](int r, int y, int x) -> double {
        if (r < 0) return S.zh[((r + HB) * BYX + y) * BYX + x];
        if (r >= BZ) return S.zh[((r - BZ + HB) * BYX + y) * BYX + x];
        return S.v[r * PLANE + (y + HB) * SVP + (x + HB)];
      };
      // (CTA-uniform / warp-uniform skips: which ghosts of this brick and plane
      // are synthesised at all -- periodic and exchanged ones are already loaded)
      const bool syn_y = (y0 < HB || y0 + BYX + HB > n1) && A1.bc != HJ_BC_PERIODIC;
      const bool syn_x = (x0 < HB || x0 + BYX + HB > n2) && A2.bc != HJ_BC_PERIODIC;
      const bool syn_zp = gz >= n0 && jz == GI_SYNTH;                       // this warp's plane
      const bool syn_zh = ghost_index(A0, z0 - 1) == GI_SYNTH || ghost_index(A0, z0 + BZ) == GI_SYNTH ||
                          ghost_index(A0, z0 + BZ + HB - 1) == GI_SYNTH;
      // Only the ghost slots some walk reads are visited: a second-axis ghost
      // row at the brick's in-domain columns, a third-axis ghost column at its
      // in-domain rows, a first-axis ghost plane at its in-domain (y, x); each
      // reads only in-domain slots that phase 1 loaded (never another ghost).
      if (gz < n0 && lane_on) {
        double* colp = &S.v[z * PLANE + lane];
        if (syn_y && xin && gx_in) {
          const int lo_end = min(SVR, HB - y0);        // rows with gy < 0
          const int hi_beg = max(0, n1 - y0 + HB);     // rows with gy >= n1
          if (lo_end > 0) {
            const double e = colp[(HB - y0) * SVP], in = colp[(HB - y0 + 1) * SVP];
            for (int yy = 0; yy < lo_end; ++yy) colp[yy * SVP] = ghost_synth(A1, y0 + yy - HB, e, in);
          }
          if (hi_beg < SVR) {
            const double e = colp[(n1 - 1 - y0 + HB) * SVP], in = colp[(n1 - 2 - y0 + HB) * SVP];
            for (int yy = hi_beg; yy < SVR; ++yy) colp[yy * SVP] = ghost_synth(A1, y0 + yy - HB, e, in);
          }
        }
        if (syn_x && !gx_in) {                          // this lane is a third-axis ghost column
          const int xe = (gx < 0 ? 0 : n2 - 1) - x0 + HB, xi = (gx < 0 ? 1 : n2 - 2) - x0 + HB;
          const int rows = min(BYX, n1 - y0);
          double* row = &S.v[z * PLANE + HB * SVP];
          for (int yy = 0; yy < rows; ++yy, row += SVP) row[lane] = ghost_synth(A2, gx, row[xe], row[xi]);
        }
      } else if (syn_zp && xin && gx_in) {              // this warp's plane lies beyond the last one
        const int re = n0 - 1 - z0, ri = n0 - 2 - z0;   // re in [0, BZ), ri >= -1
        const int rows = min(BYX, n1 - y0);
        for (int y = 0; y < rows; ++y) {
          const double edge = S.v[re * PLANE + (y + HB) * SVP + lane];
          const double inner = ri >= 0 ? S.v[ri * PLANE + (y + HB) * SVP + lane] : pz(ri, y, lane - HB);
          S.v[z * PLANE + (y + HB) * SVP + lane] = ghost_synth(A0, gz, edge, inner);
        }
      }
#pragma unroll
      for (int r2 = warp; r2 < HB * BYX && syn_zh; r2 += BRICK_THREADS / 32) {
        const int row = 2 * r2 + half;
        const int k = row / BYX, y = row % BYX;
        const int e = (k < HB) ? (z0 - HB + k) : (z0 + BZ + k - HB);
        if (y0 + y >= n1 || x0 + xl >= n2 || ghost_index(A0, e) != GI_SYNTH) continue;
        const int re = (e < 0 ? 0 : n0 - 1) - z0, ri = (e < 0 ? 1 : n0 - 2) - z0;
        S.zh[row * BYX + xl] = ghost_synth(A0, e, pz(re, y, xl), pz(ri, y, xl));
      }
    }
    // first-axis halo planes of an interior brick: 6 x 16 rows of 16, two rows per warp instruction
    if (interior) {
      const int half = lane >> 4, xl = lane & (BYX - 1);
#pragma unroll
      for (int r2 = warp; r2 < HB * BYX; r2 += BRICK_THREADS / 32) {
        const int row = 2 * r2 + half;
        const int k = row / BYX, y = row % BYX;
        const int e = (k < HB) ? (z0 - HB + k) : (z0 + BZ + k - HB);
        HJ_CHK(P, in, vin + e * s0 + (y0 + y) * s1 + (x0 + xl), 8);
        cp_async8(&S.zh[row * BYX + xl], vin + e * s0 + (y0 + y) * s1 + (x0 + xl));
      }
    }
    cp_async_wait_all();
  }
  // the Hamiltonian's node-table inputs for this brick (global loads once per
  // brick instead of per node)
  // (3-D only: the 4-D pair's inputs are constant along the fused walk)
  if (AO == 0 && HAM != HJ_HAM_ADVECTION && t < BZ + 4 * BYX) {
    double val = 0.0;
    if (t < CRD_Y) {
      if (z0 + t < n0) val = G.nodes[AO][z0 + t];
    } else if (t < CRD_X) {
      if (y0 + t - CRD_Y < n1) val = G.nodes[AO + 1][y0 + t - CRD_Y];
    } else if (t < CRD_T0) {
      if (x0 + t - CRD_X < n2) val = G.nodes[AO + 2][x0 + t - CRD_X];
    } else {
      const int w = (t - CRD_T0) / BYX, k = (t - CRD_T0) % BYX;
      if (P.ham.tab[w] && x0 + k < n2) val = P.ham.tab[w][x0 + k];
    }
    S.crd[t] = val;
  }
  __syncthreads();
  if (next) prefetch_brick<AO>(P, G, V, *next, t);

  // the first-axis walk's y0 inputs (RK2/RK3 combination stages) go through
  // the per-thread shared ring S.qy, two nodes ahead; the first two copies are
  // issued here so that their latency hides behind the second/third-axis
  // walks.  One cp.async group per node: at node i, wait_group 1 completes
  // exactly node i's copy (node i+1's may stay in flight).
  const int cy = t / BYX, cx = t % BYX;
  const bool col_on = y0 + cy < n1 && x0 + cx < n2;
  const long long coff0 = (long long)z0 * s0 + (long long)(y0 + cy) * s1 + (x0 + cx);
  const double* __restrict__ y0p = P.y0 ? P.y0 + base : nullptr;
  const bool need_y0 = P.stage >= HJ_STAGE_RK2_AVG;
  const int zmax = n0 - z0;   // nodes of this column inside the domain (may exceed BZ)
  if (need_y0) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (col_on && k < zmax) {
        HJ_CHK(P, y0, y0p + coff0 + (long long)k * s0, 8);
        cp_async8(&S.qy[k * BRICK_THREADS + t], y0p + coff0 + (long long)k * s0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }

  // ---- second and third brick axes together: warps 0-3 walk the BZ x BYX
  // lines along y, warps 4-7 the lines along x, each a whole 16-node edge;
  // they leave p_avg and the dissipation term of their axis per node
  // (lines whose nodes all lie outside the domain -- the partial bricks at
  // the far faces -- are skipped: nothing reads their p_avg / dissipation,
  // and the FP64 pipe they would occupy is shared with the SM's other warps)
  // 4-D: one code path serves both walks (line stride, output arrays and the
  // swizzled slot are runtime selects), so the two walk loops share one copy
  // in the instruction cache; each warp is wholly a y- or an x-walk warp
  // (measured: +3.7 % on 121^4; the 3-D kernel keeps two specialised copies,
  // -1.6 % there from the extra registers)
  if constexpr (AO == 1) {
    const bool yw = t < BRICK_THREADS / 2;
    const int tt = yw ? t : t - BRICK_THREADS / 2;
    const int c = tt % BYX, z = tt / BYX;   // c: the line's x (y-walk) or y (x-walk)
    if (z0 + z < n0 && (yw ? x0 + c < n2 : y0 + c < n1)) {
      const double* line = yw ? &S.v[z * PLANE + HB * SVP + (c + HB)] : &S.v[z * PLANE + (c + HB) * SVP + HB];
      const int step = yw ? SVP : 1;
      const double ah = P.alpha_half[AO + (yw ? 1 : 2)];
      double* pa = yw ? S.p1 : S.p2;
      double* ta = yw ? S.t1 : S.t2;
      const int row = z * BYX * BYX;
      auto ld = [&](int k) -> double { return line[k * step]; };
      auto emit = [&](int i, double L, double R) {
        // swz(z, i, c) for the y-walk, swz(z, c, i) for the x-walk
        const int s = row + (yw ? i * BYX + (c ^ i) : c * BYX + (i ^ c));
        pa[s] = 0.5 * (L + R);                               // term.py:101
        ta[s] = ah * (R - L);                                // term.py:85-86
      };
      line_walk<SCHEME, WALK_UNROLL, LSEG>(ld, G.sp[AO + (yw ? 1 : 2)], emit, yw ? n1 - y0 : n2 - x0);
    }
  } else if (t < BRICK_THREADS / 2) {
    const int x = t % BYX, z = t / BYX;
    if (z0 + z < n0 && x0 + x < n2) {
      const double* line = &S.v[z * PLANE + HB * SVP + (x + HB)];
      const double ah = P.alpha_half[AO + 1];
      auto ld = [&](int k) -> double { return line[k * SVP]; };
      auto emit = [&](int i, double L, double R) {
        const int s = swz(z, i, x);
        S.p1[s] = 0.5 * (L + R);                               // term.py:101
        S.t1[s] = ah * (R - L);                                // term.py:85-86
      };
      line_walk<SCHEME, WALK_UNROLL, LSEG>(ld, G.sp[AO + 1], emit, n1 - y0);
    }
  } else {
    const int y = t % BYX, z = (t - BRICK_THREADS / 2) / BYX;
    if (z0 + z < n0 && y0 + y < n1) {
      const double* line = &S.v[z * PLANE + (y + HB) * SVP + HB];
      const double ah = P.alpha_half[AO + 2];
      const int row = (z * BYX + y) * BYX;
      auto ld = [&](int k) -> double { return line[k]; };
      auto emit = [&](int i, double L, double R) {
        const int s = row + (i ^ y);
        S.p2[s] = 0.5 * (L + R);
        S.t2[s] = ah * (R - L);
      };
      line_walk<SCHEME, WALK_UNROLL, LSEG>(ld, G.sp[AO + 2], emit, n2 - x0);
    }
  }
  __syncthreads();

  // ---- first brick axis fused with the per-node update: thread (y, x) walks
  // its column (zh planes below / above) and, per node, forms
  //   d = ((prev + t_first) + t_second) + t_third     (term.py:84-86 axis order)
  //   H(x, p_avg), delta = d - H (term.py:113), the stage update
  //   (integrator.py:93-103), the optional tube mask (reachability.py:249),
  // the non-finite flags, and stores the node (coalesced across x).
  {
    const int y = cy, x = cx;
    if (col_on) {
      const double* col = &S.v[(y + HB) * SVP + (x + HB)];
      const double* zlo = &S.zh[HB * BYX * BYX + y * BYX + x];          // plane k+3, k in [-3,-1]
      const double* zhi = &S.zh[(HB - BZ) * BYX * BYX + y * BYX + x];   // plane k-BZ+3, k >= BZ
      const double ah = P.alpha_half[AO];
      const int s00 = swz(0, y, x);
      const long long off0 = coff0;
      const int slice0 = AO ? V.zp.map(c.b % V.zp.cnt) : 0;   // 4-D: the slice's axis-0 index
      const double* __restrict__ mp = P.mask_prev ? P.mask_prev + base : nullptr;
      double* __restrict__ out = P.y_out + base;
      const bool need_m = P.mask != HJ_MASK_NONE;
      // other global inputs of the node being emitted, fetched one node ahead
      double nz_m = 0.0, nz_p0 = 0.0, nz_d0 = 0.0;
      auto fetch_node = [&](int i) {
        const long long off = off0 + (long long)i * s0;
        if (need_m) HJ_CHK(P, mask, mp + off, 8);
        nz_m = need_m ? mp[off] : 0.0;
        if (AO) {
          HJ_CHK(P, aux, reinterpret_cast<const double2*>(P.aux0) + (base + off), 16);
          const double2 pd = __ldg(reinterpret_cast<const double2*>(P.aux0) + (base + off));
          nz_p0 = pd.x;
          nz_d0 = pd.y;
        }
      };
      fetch_node(0);
      auto ld = [&](int k) -> double {
        if (k < 0) return zlo[k * (BYX * BYX)];
        if (k < BZ) return col[k * PLANE];
        return zhi[k * (BYX * BYX)];
      };
      auto emit = [&](int i, double L, double R) {
        if (i >= zmax) return;
        double yz = 0.0;
        double* qslot = &S.qy[(i & 1) * BRICK_THREADS + t];
        if (need_y0) {
          asm volatile("cp.async.wait_group 1;" ::: "memory");   // node i's copy has landed
          yz = *qslot;
        }
        const double pv = nz_m, a0 = nz_p0, d0 = nz_d0;
        if (i + 1 < zmax && i + 1 < BZ) fetch_node(i + 1);
        const int s = s00 + i * (BYX * BYX);
        double p[3 + AO];
        if (AO) p[0] = a0;
        p[AO] = 0.5 * (L + R);                                   // term.py:101
        p[AO + 1] = S.p1[s];
        p[AO + 2] = S.p2[s];
        // derivative / p_avg finiteness, as ScalarField(p_avg) checks it (term.py:101):
        // a non-finite one-sided derivative always makes its p_avg non-finite
        // (tested below together with the node's other values: one compare on the
        // largest exponent field, the per-class flags only on the rare failure)
        // AO = 1: the dissipation continues from the axis-0 pre-pass
        const double dsum = (((AO ? d0 : 0.0) + ah * (R - L)) + S.t1[s]) + S.t2[s];
        // ham_eval inputs (hj_ham.cuh): 3-D Hamiltonians take the axis-0/1 nodes
        // and the axis-2 tables (staged per brick); the 4-D pair takes the
        // axis-2/3 nodes, constant along this walk
        double cin[4] = {0.0, 0.0, 0.0, 0.0};
        if (AO == 0) {
          cin[0] = S.crd[i];
          cin[1] = S.crd[CRD_Y + y];
          cin[2] = S.crd[CRD_T0 + x];
          cin[3] = S.crd[CRD_T1 + x];
        } else {
          int ix[4] = {slice0, z0 + i, y0 + y, x0 + x};
          ham_inputs<HAM, 4>(P.ham, G.nodes, ix, cin);
        }
        const double H = ham_eval<HAM, 3 + AO>(P.ham, cin, p);
        if (P.want_hnz && H != 0.0) flags |= HJ_FLAG_HAM_NONZERO;
        const double delta = dsum - H;                           // term.py:113
        const double yv = col[i * PLANE];
        double o = stage_update(P.stage, P.dt, yv, yz, delta);
        if (P.mask == HJ_MASK_MIN) o = (pv < o) ? pv : o;
        else if (P.mask == HJ_MASK_MAX) o = (pv > o) ? pv : o;
        HJ_CHK(P, out, out + off0 + (long long)i * s0, 8);
        out[off0 + (long long)i * s0] = o;
        if (need_y0) {
          // refill the slot just read with node i+2 (issued after the store of
          // o, which consumed yz: the slot's read has completed)
          if (i + 2 < zmax && i + 2 < BZ) {
            HJ_CHK(P, y0, y0p + (off0 + (long long)(i + 2) * s0), 8);
            cp_async8(qslot, y0p + (off0 + (long long)(i + 2) * s0));
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // non-finite flags: finite(x) <=> |hi(x)| < 0x7FF00000
        unsigned big = max(max(abs_hi(H), abs_hi(delta)), max(abs_hi(yv), abs_hi(o)));
#pragma unroll
        for (int a = 0; a < 3 + AO; ++a) big = max(big, abs_hi(p[a]));
        if (big >= 0x7FF00000u) {
          unsigned nf = 0u;
#pragma unroll
          for (int a = 0; a < 3 + AO; ++a) nf |= (abs_hi(p[a]) >= 0x7FF00000u) ? 1u : 0u;
          if (nf) flags |= HJ_NF_DERIV;
          if (!finite(H)) flags |= HJ_NF_HAM;
          if (!finite(delta)) flags |= HJ_NF_DELTA;
          if (!finite(yv)) flags |= HJ_NF_INPUT;
          if (!finite(o)) flags |= HJ_NF_OUTPUT;
        }
      };
      line_walk<SCHEME, ZWALK_UNROLL, SEG>(ld, G.sp[AO], emit, zmax);
    }
  }
}

// ---- 4-D pre-pass: the axis-0 walks (one thread per column segment, coalesced
// across the last axis); p_avg0 and d0 = 0 + (alpha0*0.5)*(R0-L0) to scratch.
// A segment covers up to PR consecutive 8-plane rows of the launch's row set
// (zr: rows lo..lo+split-1, then hs..): longer segments amortise the walk's
// window fill (5 faces + 3 centres) over more nodes.
constexpr int PRE_ROWS = 2;

template <int PR>
__host__ __device__ __forceinline__ int pre_segments(const RowSet& r) {
  return (r.split + PR - 1) / PR + (r.cnt - r.split + PR - 1) / PR;
}

template <int SCHEME, int PR>
__global__ void __launch_bounds__(256) k_axis0_walk(const StageArgs P) {
  const GridArgs& G = P.g;
  const long long plane = G.stride[0];
  const long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= plane) return;
  const RowSet& R = P.zr;
  const int nseg = pre_segments<PR>(R);
  const int sidx = blockIdx.y % nseg, pb = blockIdx.y / nseg;
  const int na = (R.split + PR - 1) / PR;
  int row, rows;   // first row of the segment and its row count
  if (sidx < na) {
    row = R.lo + sidx * PR;
    rows = min(PR, R.split - sidx * PR);
  } else {
    const int k = sidx - na;
    row = R.hs + k * PR;
    rows = min(PR, (R.cnt - R.split) - k * PR);
  }
  const int z0 = row * SEG;
  const long long base = (long long)pb * G.batch_stride + pos;
  const double* col = P.y_in + base;
  const AxisView A0 = G.ax[0];
  const double ah = P.alpha_half[0];
  const int zmax = min(rows * SEG, G.n[0] - z0);
  // a segment whose stencils stay inside the owned planes loads directly;
  // the walk reads k = -3..2 for its window, then k = 3, 4, ... one per step:
  // those arrive through a two-deep register queue (the load of node k+2 is
  // issued when node k is consumed, a whole walk step before it is needed)
  const bool inner = z0 >= 3 && z0 + zmax + 3 <= G.n[0];
  const double* cz = col + (long long)z0 * plane;
  const int kmax = zmax + 2;   // last index the walk reads
  double q0 = 0.0, q1 = 0.0;
  if (inner) {
    HJ_CHK(P, in, cz + 3 * plane, 8);
    HJ_CHK(P, in, cz + 4 * plane, 8);
    q0 = cz[3 * plane];
    q1 = (4 <= kmax) ? cz[4 * plane] : 0.0;
  }
  auto ld = [&](int k) -> double {
    if (!inner) return fetch(col, A0, z0 + k);
    if (k < 3) {
      HJ_CHK(P, in, cz + (long long)k * plane, 8);
      return cz[(long long)k * plane];
    }
    const double v = q0;
    q0 = q1;
    if (k + 2 <= kmax) {
      HJ_CHK(P, in, cz + (long long)(k + 2) * plane, 8);
      q1 = cz[(long long)(k + 2) * plane];
    }
    return v;
  };
  auto emit = [&](int i, double L, double R2) {
    if (i < zmax) {
      const long long o = base + (long long)(z0 + i) * plane;
      // (p_avg0, d0): term.py:101, and the dissipation sum's first term (term.py:84-86)
      HJ_CHK(P, aux, reinterpret_cast<double2*>(P.aux0) + o, 16);
      reinterpret_cast<double2*>(P.aux0)[o] = make_double2(0.5 * (L + R2), 0.0 + ah * (R2 - L));
    }
  };
  line_walk<SCHEME, 1, PR * SEG>(ld, G.sp[0], emit, zmax);
}

// Stage positions k = -3 .. zmax+2 (relative to node z0) of one line of axis
// view A starting at `line` into dst[(k + 3) * pitch].  Every value that lives
// in memory (in-domain nodes, a periodic axis' wrapped images) goes through
// cp.async -- all in flight, nothing waits per position; dirichlet ghosts are
// the constant; extrapolated ghosts are marked and synthesised by
// ghost_fill() once the copies have landed (they need the edge nodes).  Same
// values as fetch() (grid.py:203-225), bit for bit.
__device__ __forceinline__ void stage_line(const double* line, const AxisView& A, int z0, int zmax, double* dst,
                                           int pitch) {
  for (int k = -3; k < zmax + 3; ++k) {
    const int e = z0 + k;
    double* d = dst + (k + 3) * pitch;
    if (e >= 0 && e < A.n) {
      cp_async8(d, line + (long long)e * A.stride);
    } else if ((e < 0 && A.halo_lo) || (e >= A.n && A.halo_hi)) {
      // exchanged halo planes (multi-GPU slabs); beyond them nothing in the domain reads
      const bool in_halo = e < 0 ? e >= -A.halo_n : e < A.n + A.halo_n;
      if (in_halo) cp_async8(d, line + (long long)e * A.stride);
      else *d = 0.0;
    } else if (A.bc == HJ_BC_PERIODIC) {
      const int j = e < 0 ? ((e % A.n) + A.n) % A.n : e % A.n;
      cp_async8(d, line + (long long)j * A.stride);
    } else if (A.bc == HJ_BC_DIRICHLET) {
      *d = A.bcv;
    }
  }
}

// The extrapolated ghosts of a line staged by stage_line (after the copies
// of this thread -- or, for cooperative staging, of the CTA -- have landed).
__device__ __forceinline__ void ghost_fill(const AxisView& A, int z0, int zmax, double* dst, int pitch) {
  if (A.bc != HJ_BC_EXTRAPOLATE) return;
  if (z0 < 3 && !A.halo_lo) {
    const double v0 = dst[(0 - z0 + 3) * pitch], v1 = dst[(1 - z0 + 3) * pitch];
    for (int e = z0 - 3; e < 0; ++e) dst[(e - z0 + 3) * pitch] = v0 + (double)(-e) * (v0 - v1);   // grid.py:220,222
  }
  if (z0 + zmax + 3 > A.n && !A.halo_hi) {
    const double vn = dst[(A.n - 1 - z0 + 3) * pitch], vm = dst[(A.n - 2 - z0 + 3) * pitch];
    for (int e = A.n; e < z0 + zmax + 3; ++e)
      dst[(e - z0 + 3) * pitch] = vn + (double)(e - A.n + 1) * (vn - vm);                           // grid.py:221,223
  }
}

// The same pre-pass with the CTA's 256 column segments staged in shared
// memory first: rows k = -3 .. zmax+2 of the segment (at most 22), 256
// consecutive plane positions each, all in flight at once (cp.async for
// segments inside the owned planes, fetch() ghosts otherwise); every thread
// then walks its column from shared memory.  The global-load version above
// waits on one dependent load per walk step (long_scoreboard 35 % of its
// stall samples in r01).
constexpr int PRE_SROWS = PRE_ROWS * SEG + 6;   // 22

template <int SCHEME>
__global__ void __launch_bounds__(256, 2) k_axis0_walk_smem(const StageArgs P) {
  __shared__ double col_s[PRE_SROWS * 256];
  const GridArgs& G = P.g;
  const long long plane = G.stride[0];
  const long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool on = pos < plane;
  const RowSet& R = P.zr;
  const int nseg = pre_segments<PRE_ROWS>(R);
  const int sidx = blockIdx.y % nseg, pb = blockIdx.y / nseg;
  const int na = (R.split + PRE_ROWS - 1) / PRE_ROWS;
  int row, rows;
  if (sidx < na) {
    row = R.lo + sidx * PRE_ROWS;
    rows = min(PRE_ROWS, R.split - sidx * PRE_ROWS);
  } else {
    const int k = sidx - na;
    row = R.hs + k * PRE_ROWS;
    rows = min(PRE_ROWS, (R.cnt - R.split) - k * PRE_ROWS);
  }
  const int z0 = row * SEG;
  const long long base = (long long)pb * G.batch_stride + pos;
  const double* col = P.y_in + base;
  const AxisView A0 = G.ax[0];
  const double ah = P.alpha_half[0];
  const int zmax = min(rows * SEG, G.n[0] - z0);
  const bool inner = z0 >= 3 && z0 + zmax + 3 <= G.n[0];   // CTA-uniform
  const int t = threadIdx.x;
  if (on) {
    if (inner) {
      for (int k = -3; k < zmax + 3; ++k) {
        HJ_CHK(P, in, col + (long long)(z0 + k) * plane, 8);
        cp_async8(&col_s[(k + 3) * 256 + t], col + (long long)(z0 + k) * plane);
      }
    } else {
      stage_line(col, A0, z0, zmax, col_s + t, 256);   // (ghosts without waiting per position)
    }
  }
  cp_async_wait_all();
  if (on && !inner) ghost_fill(A0, z0, zmax, col_s + t, 256);
  __syncthreads();
  if (!on) return;
  auto ld = [&](int k) -> double { return col_s[(k + 3) * 256 + t]; };
  auto emit = [&](int i, double L, double R2) {
    if (i < zmax) {
      const long long o = base + (long long)(z0 + i) * plane;
      // (p_avg0, d0): term.py:101, and the dissipation sum's first term (term.py:84-86)
      HJ_CHK(P, aux, reinterpret_cast<double2*>(P.aux0) + o, 16);
      reinterpret_cast<double2*>(P.aux0)[o] = make_double2(0.5 * (L + R2), 0.0 + ah * (R2 - L));
    }
  };
  line_walk<SCHEME, 1, PRE_ROWS * SEG>(ld, G.sp[0], emit, zmax);
}

template <int SCHEME, int HAM, int MINB, int AO, int UNR>
static cudaError_t launch_brick(const StageArgs& P, cudaStream_t s) {
  const size_t smem = sizeof(BrickSmem);
  static std::atomic<bool> configured[64];  // per instantiation and device (idempotent if raced)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_brick<SCHEME, HAM, MINB, AO, UNR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev].store(true, std::memory_order_release);
  }
  const GridArgs& G = P.g;
  const long long slices = AO ? (long long)G.batch * P.zp.cnt : G.batch;
  const long long nbricks = (long long)((G.n[AO + 2] + BYX - 1) / BYX) * ((G.n[AO + 1] + BYX - 1) / BYX) *
                            (AO ? (G.n[AO] + BZ - 1) / BZ : P.zr.cnt) * slices;
  if (nbricks == 0) return cudaSuccess;
  const int nsm = sm_count(dev);
  const long long ctas = nbricks < (long long)MINB * nsm ? nbricks : (long long)MINB * nsm;
  if (AO) {
    const long long plane = G.stride[0];
    if (UNR & UNR_PREREG) {   // A/B: columns from global memory, 32-node segments
      dim3 pg((unsigned)((plane + 255) / 256), (unsigned)(pre_segments<4>(P.zr) * G.batch));
      k_axis0_walk<SCHEME, 4><<<pg, 256, 0, s>>>(P);
    } else {
      dim3 pg((unsigned)((plane + 255) / 256), (unsigned)(pre_segments<PRE_ROWS>(P.zr) * G.batch));
      k_axis0_walk_smem<SCHEME><<<pg, 256, 0, s>>>(P);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_stage_brick<SCHEME, HAM, MINB, AO, UNR><<<(unsigned)ctas, BRICK_THREADS, smem, s>>>(P, (int)nbricks);
  return cudaGetLastError();
}

// UNR: walk unroll of the 3-D kernels; UNR4: of the 4-D kernels
template <int SCHEME, int MINB, int UNR = 1, int UNR4 = UNR>
static cudaError_t launch_brick_ham(const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = true;
  if (P.g.dim == 4) {
    if (!P.aux0) { *handled = false; return cudaSuccess; }
    switch (P.ham.kind) {
      case HJ_HAM_ADVECTION: return launch_brick<SCHEME, HJ_HAM_ADVECTION, MINB, 1, UNR4>(P, s);
      case HJ_HAM_DI4: return launch_brick<SCHEME, HJ_HAM_DI4, MINB, 1, UNR4>(P, s);
      default: *handled = false; return cudaSuccess;
    }
  }
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: return launch_brick<SCHEME, HJ_HAM_ADVECTION, MINB, 0, UNR>(P, s);
    case HJ_HAM_ROCKETS: return launch_brick<SCHEME, HJ_HAM_ROCKETS, MINB, 0, UNR>(P, s);
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_brick<SCHEME, HJ_HAM_ROCKETS_EXTREMAL, MINB, 0, UNR>(P, s);
    case HJ_HAM_AIR3D: return launch_brick<SCHEME, HJ_HAM_AIR3D, MINB, 0, UNR>(P, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace hj
