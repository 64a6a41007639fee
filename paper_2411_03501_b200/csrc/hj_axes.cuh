// hj_axes.cuh -- the fused LF + TVD-RK stage as a pipeline of single-axis
// walks ("axes" path): one kernel per grid axis, each walking 16-node (the
// contiguous axis) or 32-node (the column axes, hj_axes_weno.cu) column
// segments of its axis from a shared-memory stage (all loads in flight at
// once), the last one fused with the node update.
//
// Why: the single-axis 4-D pre-pass (k_axis0_walk_smem, hj_brick.cuh) runs
// the WENO5 walk at 66.5 % of the FP64 pipe (ncu r02c), against 55-61 % for
// the walks inside the fused brick kernel, whose 115 KB of shared memory,
// barriers, 8-node fused walk (19 % window-fill overhead) and large hot loop
// cost issue efficiency.  Here every kernel is one small loop.
//
// Order of the dissipation sum (term.py:84-86: accumulated from zeros in axis
// order) and of the costates is preserved exactly: the contiguous axis X =
// dim-1 is walked FIRST but kept apart (PX, DX), then axes 0 .. dim-2 in
// order into a running sum D = ((0 + d0) + d1) ..., and the last kernel
// (axis dim-2) forms d = (D + d_{dim-2}) + DX, H(x, p0 .. p_{dim-1}), delta,
// the stage update, the mask and the flags -- the brick kernel's arithmetic,
// bit for bit.
//
// Scratch: field-sized arrays of 16-byte records (same node offsets as the
// field), so the last kernel's ring takes two streams with one copy each:
//   XR[n]   = (PX, DX)   costate / dissipation term of the contiguous axis
//   PD_a[n] = (P_a, D_a) costate of axis a, running dissipation sum over
//                        axes 0 .. a   (a = 0 .. dim-3)
#pragma once
#include "hj_brick.cuh"

namespace hj {

constexpr int AX_SEG = 16;                 // nodes per walk segment
constexpr int AX_ROWS = AX_SEG + 6;        // staged rows per segment (halo 3 + 3)
// 128-thread CTAs, 4 per SM (128 registers, 16 warps per SM as before): the
// CTAs' staging / walk / write-back phases desynchronise over twice as many
// CTAs (A/B against 256 x 2 on one B200: C2 +3.4 %, C4 +3.4 %, C5 +4.1 %,
// profiles/r02_raw/kernel_variant_ab.txt abb3)
constexpr int AX_THREADS = 128;
constexpr int AX_CTAS = 4;   // resident CTAs per SM the kernels are compiled for
constexpr int AX_PITCH = AX_THREADS + 1;   // odd pitch: transposed stores conflict-free

struct AxesScratch {
  double2* xr;
  double2* pd[HJ_MAX_DIM - 2];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// ---------------------------------------------------------------- contiguous axis (walked first)
// CTA = AX_THREADS rows x one 16-node segment along the row.  Rows are staged
// transposed (warp w loads rows 32w .. 32w+31, lanes along the row: 22
// consecutive doubles per load), thread t walks row t from shared memory, the
// (p, d) results are staged and written back row-wise (coalesced).
// WU: walk steps per loop iteration (2: the window state rolls through
// renamed registers instead of moves; hj_weno_line.cuh)
template <int SCHEME, int WU = 1>
__global__ void __launch_bounds__(AX_THREADS, AX_CTAS) k_axis_x(const StageArgs P, const AxesScratch S) {
  extern __shared__ __align__(16) double axs[];
  double* stg = axs;                                  // [AX_ROWS][AX_PITCH]
  double* sp = axs + AX_ROWS * AX_PITCH;              // [AX_SEG][AX_PITCH]
  double* sd = sp + AX_SEG * AX_PITCH;                // [AX_SEG][AX_PITCH]
  const GridArgs& G = P.g;
  const int X = G.dim - 1;
  const int nx = G.n[X];
  const AxisView AX = G.ax[X];
  const long long rows = (long long)G.batch * (G.cells / nx);
  const int x0 = blockIdx.y * AX_SEG;
  const int zmax = min(AX_SEG, nx - x0);
  const long long r0 = (long long)blockIdx.x * AX_THREADS;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool inner = x0 >= 3 && x0 + zmax + 3 <= nx;   // CTA-uniform
  // stage: warp w, rows 32w + j
  for (int j = 0; j < 32; ++j) {
    const int tr = warp * 32 + j;
    const long long r = r0 + tr;
    if (r >= rows || lane >= zmax + 6) continue;
    const double* row = P.y_in + r * nx;   // batches are contiguous: row r starts at r * nx
    const int e = x0 - 3 + lane;
    double* dst = &stg[lane * AX_PITCH + tr];
    if (inner || (e >= 0 && e < nx)) {
      HJ_CHK(P, in, row + e, 8);
      cp_async8(dst, row + e);
    } else if (AX.bc == HJ_BC_PERIODIC) {
      const int w = e < 0 ? ((e % nx) + nx) % nx : e % nx;
      cp_async8(dst, row + w);
    } else if (AX.bc == HJ_BC_DIRICHLET) {
      *dst = AX.bcv;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (!inner && r0 + t < rows) ghost_fill(AX, x0, zmax, stg + t, AX_PITCH);   // thread t: row t's extrapolated ghosts
  __syncthreads();
  const long long r = r0 + t;
  if (r < rows) {
    const double ah = P.alpha_half[X];
    auto ld = [&](int k) -> double { return stg[(k + 3) * AX_PITCH + t]; };
    auto emit = [&](int i, double L, double R) {
      if (i < zmax) {
        sp[i * AX_PITCH + t] = 0.5 * (L + R);   // term.py:101
        sd[i * AX_PITCH + t] = ah * (R - L);    // term.py:85-86 (added last: axis X is the last axis)
      }
    };
    line_walk<SCHEME, WU, AX_SEG>(ld, G.sp[X], emit, zmax);
  }
  __syncthreads();
  // write back row-wise: half-warps per row, lanes along the segment
  const int half = lane >> 4, xl = lane & 15;
  for (int j = 0; j < 16; ++j) {
    const int tr = warp * 32 + 2 * j + half;
    const long long rr = r0 + tr;
    if (rr >= rows || xl >= zmax) continue;
    const long long o = rr * nx + x0 + xl;
    HJ_CHK(P, aux, S.xr + o, 16);
    S.xr[o] = make_double2(sp[xl * AX_PITCH + tr], sd[xl * AX_PITCH + tr]);
  }
}

// ---------------------------------------------------------------- axes 0 .. dim-2
// MODE 0: first (D = 0 + d_a), 1: accumulate (D = D + d_a), 2: last, fused
// with the node update.  Columns: position p = o * inner + i (inner = the
// axis' stride, o = everything before the axis, batch included); a CTA takes
// AX_THREADS consecutive positions (coalesced) and one 16-node segment.  Per-node
// global inputs never sit on the walk's critical path: mode 1 stages the
// segment's D with the column (cp.async), mode 2 streams the node's scratch /
// y0 / mask values through a two-node cp.async ring filled two nodes ahead.
template <int DIM>
struct AxisColSmem {
  // ring doubles per node: XR and PD_{dim-3} records, P_0 (4-D), y0, mask
  static constexpr int NS = DIM + 3;
  // shared memory of a column kernel with SEGC-node segments: the staged
  // column rows, then the two-node ring (mode 1: D; mode 2: NS streams)
  static constexpr size_t bytes(int mode, int segc) {
    return sizeof(double) * (size_t)AX_THREADS *
           ((segc + 6) + (mode == 1 ? 2 : 0) + (mode == 2 ? 2 * NS : 0));
  }
};

template <int SCHEME, int HAM, int DIM, int AXIS, int SEGC, int WU = 1, int MINB = AX_CTAS>
__global__ void __launch_bounds__(AX_THREADS, MINB) k_axis_col(const StageArgs P, const AxesScratch S) {
  constexpr int axis = AXIS;
  constexpr int MODE = (AXIS == DIM - 2) ? 2 : (AXIS == 0 ? 0 : 1);
  constexpr int NS = AxisColSmem<DIM>::NS;
  constexpr int ROWS = SEGC + 6;
  extern __shared__ __align__(16) double cs[];   // [ROWS][AX_THREADS] column, then the ring (modes 1, 2)
  double* const extra = cs + ROWS * AX_THREADS;
  const GridArgs& G = P.g;
  const long long inner = G.stride[axis];
  const int na = G.n[axis];
  const long long total = (long long)G.batch * G.cells;
  const long long ncol = total / na;
  const long long p = (long long)blockIdx.x * AX_THREADS + threadIdx.x;
  const bool on = p < ncol;
  const long long o = p / inner, i = p - o * inner;
  const long long colbase = o * (na * inner) + i;   // field offset of node 0 of this column
  const double* col = P.y_in + colbase;
  const AxisView A = G.ax[axis];
  const int z0 = blockIdx.y * SEGC;
  const int zmax = min(SEGC, na - z0);
  const bool innerseg = z0 >= 3 && z0 + zmax + 3 <= na;   // CTA-uniform
  const int t = threadIdx.x;
  if (on) {
    if (innerseg) {
      for (int k = -3; k < zmax + 3; ++k) {
        HJ_CHK(P, in, col + (long long)(z0 + k) * inner, 8);
        cp_async8(&cs[(k + 3) * AX_THREADS + t], col + (long long)(z0 + k) * inner);
      }
    } else {
      stage_line(col, A, z0, zmax, cs + t, AX_THREADS);
    }
  }
  cp_async_wait_all();
  if (on && !innerseg) ghost_fill(A, z0, zmax, cs + t, AX_THREADS);   // own column: no barrier needed
  __syncthreads();
  const double ah = P.alpha_half[axis];
  auto ld = [&](int k) -> double { return cs[(k + 3) * AX_THREADS + t]; };
  if constexpr (MODE == 0) {
    auto emit = [&](int j, double L, double R) {
      if (j < zmax) {
        const long long off = colbase + (long long)(z0 + j) * inner;
        HJ_CHK(P, aux, S.pd[0] + off, 16);
        S.pd[0][off] = make_double2(0.5 * (L + R),         // term.py:101
                                    0.0 + ah * (R - L));   // term.py:84-86
      }
    };
    if (on) line_walk<SCHEME, WU, SEGC>(ld, G.sp[axis], emit, zmax);
  } else if constexpr (MODE == 1) {
    // the running sum's D of node j through a two-node cp.async ring
    auto issue = [&](int j) {
      if (on && j < zmax) {
        const long long off = colbase + (long long)(z0 + j) * inner;
        HJ_CHK(P, aux, &S.pd[axis - 1][off].y, 8);
        cp_async8(extra + (j & 1) * AX_THREADS + t, &S.pd[axis - 1][off].y);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    issue(1);
    auto emit = [&](int j, double L, double R) {
      if (j >= zmax) return;
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      const long long off = colbase + (long long)(z0 + j) * inner;
      HJ_CHK(P, aux, S.pd[axis] + off, 16);
      S.pd[axis][off] = make_double2(0.5 * (L + R),                                    // term.py:101
                                     extra[(j & 1) * AX_THREADS + t] + ah * (R - L));  // term.py:84-86
      issue(j + 2);   // (the slot's value is consumed by the store above)
    };
    if (on) line_walk<SCHEME, WU, SEGC>(ld, G.sp[axis], emit, zmax);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // node indices of this column (axis `axis` varies along the walk)
    int ix[HJ_MAX_DIM] = {0, 0, 0, 0, 0};
    {
      long long rem = colbase % G.cells;   // offset within the problem
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        ix[a] = (int)(rem / G.stride[a]);
        rem -= (long long)ix[a] * G.stride[a];
      }
    }
    double cin[4] = {0.0, 0.0, 0.0, 0.0};
    if (on) {
      ix[axis] = z0;
      ham_inputs<HAM, DIM>(P.ham, G.nodes, ix, cin);
    }
    const double* __restrict__ mp = P.mask_prev;
    const bool need_y0 = P.stage >= HJ_STAGE_RK2_AVG;
    const bool need_m = P.mask != HJ_MASK_NONE;
    unsigned flags = 0u;
    // ring slot (j & 1) at extra + (j & 1) * NS * T doubles (T = AX_THREADS):
    // thread t's XR record at [2t], its PD_{dim-3} record at [2T + 2t], then
    // 8-byte streams P_0 (4-D) at [4T + t], y0 at [(DIM + 1) T + t], mask at [(DIM + 2) T + t]
    auto issue = [&](int j) {
      if (on && j < zmax) {
        const long long off = colbase + (long long)(z0 + j) * inner;
        double* slot = extra + (j & 1) * NS * AX_THREADS;
        HJ_CHK(P, aux, S.xr + off, 16);
        HJ_CHK(P, aux, S.pd[DIM - 3] + off, 16);
        cp_async16(slot + 2 * t, S.xr + off);                          // (PX, DX)
        cp_async16(slot + 2 * AX_THREADS + 2 * t, S.pd[DIM - 3] + off);  // (P_{dim-3}, D)
        if constexpr (DIM == 4) {
          HJ_CHK(P, aux, &S.pd[0][off].x, 8);
          cp_async8(slot + 4 * AX_THREADS + t, &S.pd[0][off].x);       // P_0
        }
        if (need_y0) {
          HJ_CHK(P, y0, P.y0 + off, 8);
          cp_async8(slot + (DIM + 1) * AX_THREADS + t, P.y0 + off);
        }
        if (need_m) {
          HJ_CHK(P, mask, mp + off, 8);
          cp_async8(slot + (DIM + 2) * AX_THREADS + t, mp + off);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    issue(1);
    auto emit = [&](int j, double L, double R) {
      if (j >= zmax) return;
      asm volatile("cp.async.wait_group 1;" ::: "memory");   // node j's copies have landed
      const double* slot = extra + (j & 1) * NS * AX_THREADS + t;
      const double2 xr = reinterpret_cast<const double2*>(extra + (j & 1) * NS * AX_THREADS)[t];
      const double2 pd = reinterpret_cast<const double2*>(extra + (j & 1) * NS * AX_THREADS + 2 * AX_THREADS)[t];
      const long long off = colbase + (long long)(z0 + j) * inner;
      // H's node-table inputs: the column's constant ones were read once
      // (cin below); only the walk axis' coordinate changes per node
      if constexpr (HAM == HJ_HAM_AIR3D && axis == 1) cin[1] = G.nodes[1][z0 + j];
      if constexpr ((HAM == HJ_HAM_ROCKETS || HAM == HJ_HAM_ROCKETS_EXTREMAL) && axis == 0) cin[0] = G.nodes[0][z0 + j];
      if constexpr (HAM == HJ_HAM_DI4 && axis == 2) cin[0] = G.nodes[2][z0 + j];
      double pv[DIM];
      if constexpr (DIM == 4) pv[0] = slot[4 * AX_THREADS];
      pv[DIM - 3] = pd.x;
      pv[DIM - 2] = 0.5 * (L + R);                                           // term.py:101
      pv[DIM - 1] = xr.x;
      // term.py:84-86 order: (((0 + d0) + ...) + d_{dim-2}) + d_{dim-1}
      const double dsum = (pd.y + ah * (R - L)) + xr.y;
      const double H = ham_eval<HAM, DIM>(P.ham, cin, pv);
      if (P.want_hnz && H != 0.0) flags |= HJ_FLAG_HAM_NONZERO;
      const double delta = dsum - H;                                         // term.py:113
      const double yv = ld(j);
      const double yz = need_y0 ? slot[(DIM + 1) * AX_THREADS] : 0.0;
      double out = stage_update(P.stage, P.dt, yv, yz, delta);
      if (P.mask == HJ_MASK_MIN) {
        const double m = slot[(DIM + 2) * AX_THREADS];
        out = (m < out) ? m : out;
      } else if (P.mask == HJ_MASK_MAX) {
        const double m = slot[(DIM + 2) * AX_THREADS];
        out = (m > out) ? m : out;
      }
      HJ_CHK(P, out, P.y_out + off, 8);
      P.y_out[off] = out;
      // the slot's values are consumed (out depends on every one of them)
      issue(j + 2);
      unsigned big = max(max(abs_hi(H), abs_hi(delta)), max(abs_hi(yv), abs_hi(out)));
#pragma unroll
      for (int a = 0; a < DIM; ++a) big = max(big, abs_hi(pv[a]));
      if (big >= 0x7FF00000u) {
        unsigned nf = 0u;
#pragma unroll
        for (int a = 0; a < DIM; ++a) nf |= (abs_hi(pv[a]) >= 0x7FF00000u) ? 1u : 0u;
        if (nf) flags |= HJ_NF_DERIV;
        if (!finite(H)) flags |= HJ_NF_HAM;
        if (!finite(delta)) flags |= HJ_NF_DELTA;
        if (!finite(yv)) flags |= HJ_NF_INPUT;
        if (!finite(out)) flags |= HJ_NF_OUTPUT;
      }
    };
    if (on) line_walk<SCHEME, WU, SEGC>(ld, G.sp[axis], emit, zmax);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (P.stats) {   // every thread of the CTA (warp-synchronous reduction)
      long long dmy[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) dmy[a] = 0;
      reduce_stats<DIM>(P.stats, flags, P.tag, false, dmy, dmy);
    }
  }
}

// The pipeline of one stage.  Covers whole-grid launches (every axis-0 plane,
// no exchanged halos) of dims 3 and 4; *handled = false otherwise.
// parts: bit 0 the contiguous-axis kernel, bit 1 the column kernels (a slab
// stage launches them on either side of its halo exchange, hj_dd_stage)
// WU: walk two steps per loop iteration in the contiguous-axis kernel (bit 0),
// the last-axis kernel (bit 1), the axis-0 / middle-axis column kernels (bit
// 2); bit 3: column kernels compiled for 3 CTAs per SM (measured with
// 256-thread CTAs: 80 registers, spills, -32 .. -40 %; not instantiated);
// bit 4: the last-axis kernel on 2 SEGC-node segments.  Default: bit 2 only
// (A/B on one B200, profiles/r02_raw/kernel_variant_ab.txt: C2 +1.9 %, C4
// +1.9 %, C5 +-0; the unrolled contiguous-axis walk: C2 +2.0 %, C4 -4.7 %,
// C5 -0.6 %; the unrolled last-axis walk -0.4 .. -1.2 %)
template <int SCHEME, int HAM, int DIM, int SEGC = AX_SEG, int WU = 4>
static cudaError_t launch_axes_t(const StageArgs& P, cudaStream_t s, double* scratch, int parts = 3) {
  constexpr int XU = (WU & 1) ? 2 : 1, LU = (WU & 2) ? 2 : 1, CU = (WU & 4) ? 2 : 1, MB = (WU & 8) ? 3 : AX_CTAS;
  constexpr int LSEG = (WU & 16) ? 2 * SEGC : SEGC;   // bit 4: the last-axis kernel walks 2 SEGC-node segments
  const GridArgs& G = P.g;
  const long long span = (long long)G.batch_stride * (G.batch - 1) + G.cells;
  AxesScratch S{};
  S.xr = reinterpret_cast<double2*>(scratch);
  for (int a = 0; a < DIM - 2; ++a) S.pd[a] = reinterpret_cast<double2*>(scratch + 2 * (1 + a) * span);
  const size_t xsmem = (size_t)(AX_ROWS + 2 * AX_SEG) * AX_PITCH * sizeof(double);
  using CS = AxisColSmem<DIM>;
  static std::atomic<bool> configured[64];
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaSuccess;
  if (dev < 0 || dev >= 64 || !configured[dev].load(std::memory_order_acquire)) {
    e = cudaFuncSetAttribute(k_axis_x<SCHEME, XU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_axis_col<SCHEME, HAM, DIM, 0, SEGC, CU, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)CS::bytes(0, SEGC));
    if (e == cudaSuccess && DIM == 4)
      e = cudaFuncSetAttribute(k_axis_col<SCHEME, HAM, DIM, 1, SEGC, CU, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)CS::bytes(1, SEGC));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_axis_col<SCHEME, HAM, DIM, DIM - 2, LSEG, LU, MB>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CS::bytes(2, LSEG));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev].store(true, std::memory_order_release);
  }
  // the scratch is this path's "aux" extent (bounds-checking build)
  StageArgs Q = P;
  Q.bc.aux = Extent{scratch, scratch + axes_scratch_doubles(DIM, (size_t)span)};
  const int X = DIM - 1;
  const long long rows = (long long)G.batch * (G.cells / G.n[X]);
  if (parts & 1) {
    k_axis_x<SCHEME, XU><<<dim3((unsigned)((rows + AX_THREADS - 1) / AX_THREADS),
                            (unsigned)((G.n[X] + AX_SEG - 1) / AX_SEG)),
                       AX_THREADS, xsmem, s>>>(Q, S);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (!(parts & 2)) return cudaSuccess;
  auto grid_of = [&](int a, int seg) {
    const long long ncol = (long long)G.batch * G.cells / G.n[a];
    return dim3((unsigned)((ncol + AX_THREADS - 1) / AX_THREADS), (unsigned)((G.n[a] + seg - 1) / seg));
  };
  k_axis_col<SCHEME, HAM, DIM, 0, SEGC, CU, MB><<<grid_of(0, SEGC), AX_THREADS, CS::bytes(0, SEGC), s>>>(Q, S);
  if constexpr (DIM == 4) k_axis_col<SCHEME, HAM, DIM, 1, SEGC, CU, MB><<<grid_of(1, SEGC), AX_THREADS, CS::bytes(1, SEGC), s>>>(Q, S);
  k_axis_col<SCHEME, HAM, DIM, DIM - 2, LSEG, LU, MB><<<grid_of(DIM - 2, LSEG), AX_THREADS, CS::bytes(2, LSEG), s>>>(Q, S);
  return cudaGetLastError();
}

}  // namespace hj
