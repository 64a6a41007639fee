// hj_brick.cuh -- the fused LF + TVD-RK stage on 3-D grids, brick-tiled,
// templated on the upwind scheme and the device Hamiltonian.
//
// One CTA (256 threads, ~100 KB shared memory, 2 CTAs per SM) owns an
// 8 x 16 x 16 brick (axes 0, 1, 2).  Per stage and brick:
//   axis 0: thread (y,x) walks its 8-node column straight from global memory
//           (coalesced over x; exchanged halo planes / boundary ghosts via
//           fetch) and parks the values in shared memory;
//   axis 1: thread (z, segment, x) walks 8 nodes along y in shared memory;
//   axis 2: thread (z, segment, y) walks 8 nodes along x in shared memory;
//   every walk stores p_avg_a = 0.5*(L+R) and accumulates the dissipation
//   d = (0 + d0) + d1 + d2 with d_a = (alpha_a*0.5)*(R_a-L_a) in the
//   reference's axis order (term.py:84-86);
//   out:    coalesced pass per node -- H(x, p_avg), delta = d - H
//           (term.py:113), stage update (integrator.py:93-103), optional
//           tube mask (reachability.py:249), non-finite flags, store.
// The three axis walks run through ONE inlined copy of the line walker (a
// runtime-configured loop over the axes), keeping the kernel's instruction
// footprint small; the walker itself is a rolled loop with a register window
// (hj_weno_line.cuh / hj_eno_line.cuh) that computes each face quantity once.
#pragma once
#include "hj_eno_line.cuh"
#include "hj_kernels.cuh"
#include "hj_weno_line.cuh"

namespace hj {

constexpr int BZ = 8;                  // brick depth along axis 0
constexpr int BYX = 16;                // brick edge along axes 1 and 2
constexpr int SEG = 8;                 // nodes per thread walk along axes 1 and 2
constexpr int HB = 3;                  // ghost width held in shared memory (WENO5/ENO3 need 3)
constexpr int SVP = BYX + 2 * HB + 1;  // 23: odd pitch (conflict-free LDS.64 across y-lanes)
constexpr int SVR = BYX + 2 * HB;      // 22 rows per plane
constexpr int SAP = BYX + 1;           // 17: odd pitch of the per-node arrays
constexpr int BRICK_THREADS = 256;

struct BrickSmem {
  double v[BZ][SVR][SVP];    // brick values with axis-1/axis-2 halos
  double p0[BZ][BYX][SAP];   // p_avg per axis
  double p1[BZ][BYX][SAP];
  double p2[BZ][BYX][SAP];
  double d[BZ][BYX][SAP];    // running dissipation
};

template <int SCHEME, class Load, class Emit>
__device__ __forceinline__ void line_walk(const Load& ld, int n, const Spacing& sp, const Emit& emit) {
  if constexpr (SCHEME == HJ_WENO5) {
    weno5_line(ld, n, weno_divisors(sp.h), emit);
  } else if constexpr (SCHEME == HJ_ENO3) {
    eno3_line(ld, n, eno_divisors(sp), emit);
  } else if constexpr (SCHEME == HJ_ENO2) {
    eno2_line(ld, n, eno_divisors(sp), emit);
  } else {
    first_line(ld, n, eno_divisors(sp), emit);
  }
}

template <int SCHEME, int HAM, int MINB>
__global__ void __launch_bounds__(BRICK_THREADS, MINB) k_stage_brick(const StageArgs P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BrickSmem& S = *reinterpret_cast<BrickSmem*>(smem_raw);
  const GridArgs& G = P.g;
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];
  const int nbz = (n0 + BZ - 1) / BZ;
  const int bz = blockIdx.z % nbz, b = blockIdx.z / nbz;
  const int z0 = bz * BZ, y0 = blockIdx.y * BYX, x0 = blockIdx.x * BYX;
  const long long base = (long long)b * G.batch_stride;
  const double* __restrict__ vin = P.y_in + base;
  const int t = threadIdx.x;
  unsigned flags = 0u;

  // ---- axis-1 / axis-2 halos of the brick's planes (ghost rules via fetch)
  for (int q = t; q < BZ * 12 * BYX; q += BRICK_THREADS) {
    const int z = q / (12 * BYX), r = q % (12 * BYX);
    const int gz = z0 + z;
    if (r < 6 * BYX) {           // rows y in {-3..-1, 16..18}, x interior
      const int k = r / BYX, x = r % BYX;
      const int y = (k < 3) ? (k - 3) : (BYX + k - 3);
      const int gx = x0 + x;
      double val = 0.0;
      if (gz < n0 && gx < n2) val = fetch(vin + (long long)gz * G.stride[0] + gx, G.ax[1], y0 + y);
      S.v[z][y + HB][x + HB] = val;
    } else {                     // columns x in {-3..-1, 16..18}, y interior
      const int rr = r - 6 * BYX;
      const int k = rr / BYX, y = rr % BYX;
      const int x = (k < 3) ? (k - 3) : (BYX + k - 3);
      const int gy = y0 + y;
      double val = 0.0;
      if (gz < n0 && gy < n1)
        val = fetch(vin + (long long)gz * G.stride[0] + (long long)gy * G.stride[1], G.ax[2], x0 + x);
      S.v[z][y + HB][x + HB] = val;
    }
  }
  {
    // in-brick columns past the domain edge of a partial brick: valid nodes
    // read them as ghosts of axis 1 (gy >= n1) or axis 2 (gx >= n2)
    const int y = t / BYX, x = t % BYX;
    const int gy = y0 + y, gx = x0 + x;
    if (gy >= n1 || gx >= n2) {
      for (int k = 0; k < BZ; ++k) {
        const int gz = z0 + k;
        double val = 0.0;
        if (gz < n0 && gx < n2) val = fetch(vin + (long long)gz * G.stride[0] + gx, G.ax[1], gy);
        else if (gz < n0 && gy < n1)
          val = fetch(vin + (long long)gz * G.stride[0] + (long long)gy * G.stride[1], G.ax[2], gx);
        S.v[k][y + HB][x + HB] = val;
      }
    }
  }

  // ---- the three axis walks through one copy of the line walker
#pragma unroll 1
  for (int ax = 0; ax < 3; ++ax) {
    const double* src;          // line start (relative node 0)
    long long sstride;          // element stride along the line
    bool from_global;
    int e0 = 0;                 // global index of relative node 0 (axis-0 walk)
    double* op;                 // p_avg output, node 0
    double* od;                 // dissipation, node 0
    int ostride;
    int nvalid;                 // nodes [0, nvalid) are inside the domain
    int len;
    double* park = nullptr;
    if (ax == 0) {
      const int y = t / BYX, x = t % BYX;
      const int gy = y0 + y, gx = x0 + x;
      src = vin + (long long)gy * G.stride[1] + gx;
      sstride = 0;
      from_global = true;
      e0 = z0;
      park = &S.v[0][y + HB][x + HB];
      op = &S.p0[0][y][x];
      od = &S.d[0][y][x];
      ostride = BYX * SAP;
      len = BZ;
      nvalid = (gy < n1 && gx < n2) ? min(BZ, n0 - z0) : -1;
    } else if (ax == 1) {
      const int x = t % BYX, seg = (t / BYX) % (BYX / SEG), z = t / (BYX * (BYX / SEG));
      src = &S.v[z][HB + seg * SEG][x + HB];
      sstride = SVP;
      from_global = false;
      op = &S.p1[z][seg * SEG][x];
      od = &S.d[z][seg * SEG][x];
      ostride = SAP;
      len = SEG;
      nvalid = (z0 + z < n0 && x0 + x < n2) ? min(SEG, n1 - (y0 + seg * SEG)) : 0;
    } else {
      const int y = t % BYX, seg = (t / BYX) % (BYX / SEG), z = t / (BYX * (BYX / SEG));
      src = &S.v[z][y + HB][HB + seg * SEG];
      sstride = 1;
      from_global = false;
      op = &S.p2[z][y][seg * SEG];
      od = &S.d[z][y][seg * SEG];
      ostride = 1;
      len = SEG;
      nvalid = (z0 + z < n0 && y0 + y < n1) ? min(SEG, n2 - (x0 + seg * SEG)) : 0;
    }
    if (nvalid >= 0) {   // axis-0 walks skip columns outside the domain
      const AxisView A0 = G.ax[0];
      const double ah = P.alpha_half[ax];
      const bool first = ax == 0;
      auto ld = [&](int k) -> double {
        if (from_global) {
          const double val = fetch(src, A0, e0 + k);
          if (k >= 0 && k < BZ) park[k * (SVR * SVP)] = val;
          return val;
        }
        return src[k * sstride];
      };
      auto emit = [&](int i, double L, double R) {
        if (i < nvalid && (!finite(L) || !finite(R))) flags |= HJ_NF_DERIV;
        op[i * ostride] = 0.5 * (L + R);                     // term.py:101
        const double prev = first ? 0.0 : od[i * ostride];   // term.py:84 zeros
        od[i * ostride] = prev + ah * (R - L);               // term.py:85-86
      };
      line_walk<SCHEME>(ld, len, G.sp[ax], emit);
    }
    __syncthreads();
  }

  // ---- per node: H, delta, stage update, mask, store (coalesced over axis 2)
  {
    const double* __restrict__ y0p = P.y0 ? P.y0 + base : nullptr;
    const double* __restrict__ mp = P.mask_prev ? P.mask_prev + base : nullptr;
    double* __restrict__ out = P.y_out + base;
#pragma unroll 2
    for (int q = t; q < BZ * BYX * BYX; q += BRICK_THREADS) {
      const int z = q / (BYX * BYX), y = (q / BYX) % BYX, x = q % BYX;
      const int gz = z0 + z, gy = y0 + y, gx = x0 + x;
      if (gz >= n0 || gy >= n1 || gx >= n2) continue;
      const long long off = (long long)gz * G.stride[0] + (long long)gy * G.stride[1] + gx;
      double p[3];
      p[0] = S.p0[z][y][x];
      p[1] = S.p1[z][y][x];
      p[2] = S.p2[z][y][x];
      const int ix[3] = {gz, gy, gx};
      const double H = hamiltonian<HAM, 3>(P.ham, G.nodes, ix, p);
      if (!finite(H)) flags |= HJ_NF_HAM;
      if (P.want_hnz && H != 0.0) flags |= HJ_FLAG_HAM_NONZERO;
      const double delta = S.d[z][y][x] - H;                // term.py:113
      if (!finite(delta)) flags |= HJ_NF_DELTA;
      const double yv = S.v[z][y + HB][x + HB];
      if (!finite(yv)) flags |= HJ_NF_INPUT;
      const double yz = (P.stage >= HJ_STAGE_RK2_AVG) ? y0p[off] : 0.0;
      double o = stage_update(P.stage, P.dt, yv, yz, delta);
      if (P.mask == HJ_MASK_MIN) {
        const double pv = mp[off];
        o = (pv < o) ? pv : o;
      } else if (P.mask == HJ_MASK_MAX) {
        const double pv = mp[off];
        o = (pv > o) ? pv : o;
      }
      if (!finite(o)) flags |= HJ_NF_OUTPUT;
      out[off] = o;
    }
  }
  if (P.stats) {
    long long dummy[1] = {0};
    reduce_stats<1>(P.stats, flags, P.tag, false, dummy, dummy);
  }
}

template <int SCHEME, int HAM, int MINB>
static cudaError_t launch_brick(const StageArgs& P, cudaStream_t s) {
  const size_t smem = sizeof(BrickSmem);
  static bool configured[64] = {};  // per instantiation and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_brick<SCHEME, HAM, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev] = true;
  }
  const GridArgs& G = P.g;
  dim3 grid((G.n[2] + BYX - 1) / BYX, (G.n[1] + BYX - 1) / BYX, ((G.n[0] + BZ - 1) / BZ) * G.batch);
  k_stage_brick<SCHEME, HAM, MINB><<<grid, BRICK_THREADS, smem, s>>>(P);
  return cudaGetLastError();
}

template <int SCHEME, int MINB>
static cudaError_t launch_brick_ham(const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: return launch_brick<SCHEME, HJ_HAM_ADVECTION, MINB>(P, s);
    case HJ_HAM_ROCKETS: return launch_brick<SCHEME, HJ_HAM_ROCKETS, MINB>(P, s);
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_brick<SCHEME, HJ_HAM_ROCKETS_EXTREMAL, MINB>(P, s);
    case HJ_HAM_AIR3D: return launch_brick<SCHEME, HJ_HAM_AIR3D, MINB>(P, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace hj
