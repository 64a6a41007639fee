// hj_fast.cu -- the fused WENO5 + LF + TVD-RK stage on 3-D grids, brick-tiled.
//
// One CTA owns a BZ x BY x BX brick (16^3).  Per stage and brick:
//   phase Z  (axis 0): thread (y,x) walks its z-column from global memory
//            (coalesced across x, halo planes / boundary ghosts synthesised),
//            parks the brick's values in shared memory and stores p_avg0 and
//            d0 = (alpha0*0.5)*(R0-L0) per node;
//   phase Y  (axis 1): thread (z,x) walks y through shared memory,
//            p_avg1 and the running dissipation (0 + d0) + d1;
//   phase X  (axis 2): thread (z,y) walks x, finishes the dissipation
//            (term.py:84-86 order), evaluates H(x, p_avg) and stores delta;
//   phase O: coalesced pass -- stage update (integrator.py:93-103), optional
//            tube mask, non-finite flags, store.
// Every line walk uses hj_weno_line.cuh: each face quantity once per face.
#include "hj_kernels.cuh"
#include "hj_weno_line.cuh"

namespace hj {

constexpr int BB = 16;                 // brick edge
constexpr int HB = 3;                  // WENO5 ghost width
constexpr int SVP = BB + 2 * HB + 1;   // 23: odd pitch (conflict-free LDS.64 across y-lanes)
constexpr int SVR = BB + 2 * HB;       // 22 rows per plane
constexpr int SAP = BB + 1;            // 17: odd pitch of the per-node arrays
constexpr int THREADS = BB * BB;       // 256

struct FastSmem {
  double v[BB][SVR][SVP];    // brick values with x/y halos
  double p0[BB][BB][SAP];    // p_avg axis 0, later delta
  double p1[BB][BB][SAP];    // p_avg axis 1
  double d[BB][BB][SAP];     // running dissipation
};

template <int HAM>
__global__ void __launch_bounds__(THREADS, 1) k_stage_brick_weno(const StageArgs P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem& S = *reinterpret_cast<FastSmem*>(smem_raw);
  const GridArgs& G = P.g;
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];
  const int bx = blockIdx.x, by = blockIdx.y;
  const int nbz = (n0 + BB - 1) / BB;
  const int bz = blockIdx.z % nbz, b = blockIdx.z / nbz;
  const int z0 = bz * BB, y0 = by * BB, x0 = bx * BB;
  const long long base = (long long)b * G.batch_stride;
  const double* __restrict__ vin = P.y_in + base;
  const int t = threadIdx.x;
  unsigned flags = 0u;

  // ---- halo rows / columns of the x and y axes for the brick's planes
  for (int q = t; q < BB * (6 * BB + 6 * BB); q += THREADS) {
    const int z = q / (12 * BB), r = q % (12 * BB);
    const int gz = z0 + z;
    if (r < 6 * BB) {            // y halo rows: y in {-3..-1, 16..18}, x interior
      const int k = r / BB, x = r % BB;
      const int y = (k < 3) ? (k - 3) : (BB + k - 3);
      const int gx = x0 + x;
      double val = 0.0;
      if (gz < n0 && gx < n2) {
        const double* line = vin + (long long)gz * G.stride[0] + gx;
        val = fetch(line, G.ax[1], y0 + y);
      }
      S.v[z][y + HB][x + HB] = val;
    } else {                     // x halo columns: x in {-3..-1, 16..18}, y interior
      const int rr = r - 6 * BB;
      const int k = rr / BB, y = rr % BB;
      const int x = (k < 3) ? (k - 3) : (BB + k - 3);
      const int gy = y0 + y;
      double val = 0.0;
      if (gz < n0 && gy < n1) {
        const double* line = vin + (long long)gz * G.stride[0] + (long long)gy * G.stride[1];
        val = fetch(line, G.ax[2], x0 + x);
      }
      S.v[z][y + HB][x + HB] = val;
    }
  }

  // ---- phase Z: column walks (axis 0)
  {
    const int y = t / BB, x = t % BB;
    const int gy = y0 + y, gx = x0 + x;
    const bool col_ok = gy < n1 && gx < n2;
    const double* col = vin + (long long)gy * G.stride[1] + gx;
    const AxisView A0 = G.ax[0];
    const double ah = P.alpha_half[0];
    if (col_ok) {
      auto ld = [&](int k) -> double {
        const int e = z0 + k;
        const double val = fetch(col, A0, e);
        if (k >= 0 && k < BB) S.v[k][y + HB][x + HB] = val;
        return val;
      };
      auto emit = [&](int i, double L, double R) {
        if (z0 + i < n0 && (!finite(L) || !finite(R))) flags |= HJ_NF_DERIV;
        S.p0[i][y][x] = 0.5 * (L + R);
        S.d[i][y][x] = 0.0 + ah * (R - L);
      };
      weno5_line<BB>(ld, weno_divisors(G.sp[0].h), emit);
    } else {
#pragma unroll 1
      for (int k = 0; k < BB; ++k) S.v[k][y + HB][x + HB] = 0.0;
    }
  }
  __syncthreads();

  // ---- phase Y: walks along axis 1 in shared memory
  {
    const int z = t / BB, x = t % BB;
    const double ah = P.alpha_half[1];
    const bool ok = (z0 + z < n0) && (x0 + x < n2);
    auto ld = [&](int k) -> double { return S.v[z][k + HB][x + HB]; };
    auto emit = [&](int i, double L, double R) {
      if (ok && y0 + i < n1 && (!finite(L) || !finite(R))) flags |= HJ_NF_DERIV;
      S.p1[z][i][x] = 0.5 * (L + R);
      S.d[z][i][x] = S.d[z][i][x] + ah * (R - L);
    };
    weno5_line<BB>(ld, weno_divisors(G.sp[1].h), emit);
  }
  __syncthreads();

  // ---- phase X: walks along axis 2, then H and delta
  {
    const int z = t / BB, y = t % BB;
    const int gz = z0 + z, gy = y0 + y;
    const double ah = P.alpha_half[2];
    const bool ok = gz < n0 && gy < n1;
    auto ld = [&](int k) -> double { return S.v[z][y + HB][k + HB]; };
    auto emit = [&](int i, double L, double R) {
      const int gx = x0 + i;
      const bool valid = ok && gx < n2;
      if (valid && (!finite(L) || !finite(R))) flags |= HJ_NF_DERIV;
      double p[3];
      p[0] = S.p0[z][y][i];
      p[1] = S.p1[z][y][i];
      p[2] = 0.5 * (L + R);
      const double diss = S.d[z][y][i] + ah * (R - L);
      double H = 0.0;
      if (valid) {
        const int ix[3] = {gz, gy, gx};
        H = hamiltonian<HAM, 3>(P.ham, G.nodes, ix, p);
        if (!finite(H)) flags |= HJ_NF_HAM;
        if (P.want_hnz && H != 0.0) flags |= HJ_FLAG_HAM_NONZERO;
      }
      const double delta = diss - H;
      if (valid && !finite(delta)) flags |= HJ_NF_DELTA;
      S.p0[z][y][i] = delta;
    };
    weno5_line<BB>(ld, weno_divisors(G.sp[2].h), emit);
  }
  __syncthreads();

  // ---- phase O: stage update + mask, coalesced over x
  {
    const double* __restrict__ y0p = P.y0 ? P.y0 + base : nullptr;
    const double* __restrict__ mp = P.mask_prev ? P.mask_prev + base : nullptr;
    double* __restrict__ out = P.y_out + base;
#pragma unroll 4
    for (int q = t; q < BB * BB * BB; q += THREADS) {
      const int z = q / (BB * BB), y = (q / BB) % BB, x = q % BB;
      const int gz = z0 + z, gy = y0 + y, gx = x0 + x;
      if (gz >= n0 || gy >= n1 || gx >= n2) continue;
      const long long off = (long long)gz * G.stride[0] + (long long)gy * G.stride[1] + gx;
      const double yv = S.v[z][y + HB][x + HB];
      if (!finite(yv)) flags |= HJ_NF_INPUT;
      const double yz = (P.stage >= HJ_STAGE_RK2_AVG) ? y0p[off] : 0.0;
      double o = stage_update(P.stage, P.dt, yv, yz, S.p0[z][y][x]);
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

template <int HAM>
static cudaError_t launch_brick(const StageArgs& P, cudaStream_t s) {
  const size_t smem = sizeof(FastSmem);
  static bool configured[64] = {};  // per instantiation and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_brick_weno<HAM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev] = true;
  }
  const GridArgs& G = P.g;
  dim3 grid((G.n[2] + BB - 1) / BB, (G.n[1] + BB - 1) / BB, ((G.n[0] + BB - 1) / BB) * G.batch);
  k_stage_brick_weno<HAM><<<grid, THREADS, smem, s>>>(P);
  return cudaGetLastError();
}

// Claims 3-D WENO5 stages without range statistics; everything else falls
// back to the generic per-node kernel (hj_stage_generic.cuh).
cudaError_t launch_stage_fast(int scheme, const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = false;
  if (scheme != HJ_WENO5 || P.g.dim != 3 || P.want_ranges) return cudaSuccess;
  if (P.g.n[0] >= 65535 * BB || P.g.n[1] > 65535 * BB) return cudaSuccess;
  if (((P.g.n[0] + BB - 1) / BB) * (long long)P.g.batch > 65535) return cudaSuccess;
  *handled = true;
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: return launch_brick<HJ_HAM_ADVECTION>(P, s);
    case HJ_HAM_ROCKETS: return launch_brick<HJ_HAM_ROCKETS>(P, s);
    case HJ_HAM_ROCKETS_EXTREMAL: return launch_brick<HJ_HAM_ROCKETS_EXTREMAL>(P, s);
    case HJ_HAM_AIR3D: return launch_brick<HJ_HAM_AIR3D>(P, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace hj
