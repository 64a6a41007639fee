// hj_misc.cu -- ghost extension, implicit-surface init, CSG, tube mask,
// sublevel count and the host-Hamiltonian bridge kernels.
#include "hj_kernels.cuh"

namespace hj {

// ------------------------------------------------------------------ extend_with_ghost_cells
// Value of E_K(...E_0(v)) at extended coordinates e (grid.py:238-242: axes
// extended in order, so a corner ghost is the composition of per-axis rules).
template <int K>
__device__ double ext_val(const GridArgs& G, const double* __restrict__ v, int* e) {
  if constexpr (K < 0) {
    long long off = 0;
    for (int a = 0; a < G.dim; ++a) off += (long long)e[a] * G.stride[a];
    return v[off];
  } else {
    if (K >= G.dim) return ext_val<K - 1>(G, v, e);
    const int ek = e[K], n = G.n[K];
    if (ek >= 0 && ek < n) return ext_val<K - 1>(G, v, e);
    const AxisView& A = G.ax[K];
    double r;
    if (A.bc == HJ_BC_PERIODIC) {
      e[K] = ((ek % n) + n) % n;
      r = ext_val<K - 1>(G, v, e);
    } else if (A.bc == HJ_BC_DIRICHLET) {
      r = A.bcv;
    } else if (ek < 0) {
      e[K] = 0;
      const double v0 = ext_val<K - 1>(G, v, e);
      e[K] = 1;
      const double v1 = ext_val<K - 1>(G, v, e);
      r = v0 + (double)(-ek) * (v0 - v1);
    } else {
      e[K] = n - 1;
      const double vn = ext_val<K - 1>(G, v, e);
      e[K] = n - 2;
      const double vm = ext_val<K - 1>(G, v, e);
      r = vn + (double)(ek - n + 1) * (vn - vm);
    }
    e[K] = ek;
    return r;
  }
}

__global__ void k_extend(const GridArgs G, int w, const double* __restrict__ v, double* __restrict__ ext,
                         long long total) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int e[HJ_MAX_DIM];
  long long rem = idx;
  for (int a = G.dim - 1; a >= 0; --a) {
    const int ne = G.n[a] + 2 * w;
    const long long q = rem / ne;
    e[a] = (int)(rem - q * ne) - w;
    rem = q;
  }
  ext[idx] = ext_val<HJ_MAX_DIM - 1>(G, v, e);
}

// ------------------------------------------------------------------ shapes (shapes.py:24-83)
struct ShapeParams {
  double v[16];
};

__global__ void k_shape(const GridArgs G, int kind, const ShapeParams P, double* __restrict__ out) {
  const double* prm = P.v;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= G.cells * G.batch) return;
  int ix[HJ_MAX_DIM];
  const long long off = locate(G, idx, ix);
  const int d = G.dim;
  double r;
  if (kind == HJ_SHAPE_SPHERE || kind == HJ_SHAPE_CYLINDER) {
    // d2 = zeros; d2 += (x_a - c_a)**2 ; sqrt(d2) - radius   (shapes.py:29-32, 43-49)
    const unsigned ignore = (kind == HJ_SHAPE_CYLINDER) ? (unsigned)prm[d + 1] : 0u;
    double d2 = 0.0;
    for (int a = 0; a < d; ++a) {
      if (ignore & (1u << a)) continue;
      const double t = G.nodes[a][ix[a]] - prm[a];
      d2 = d2 + t * t;
    }
    r = sqrt(d2) - prm[d];
  } else if (kind == HJ_SHAPE_ELLIPSOID) {
    // e = zeros; e += w_a * x_a**2 ; e - radius   (shapes.py:61-66)
    double e = 0.0;
    for (int a = 0; a < d; ++a) {
      const double x = G.nodes[a][ix[a]];
      e = e + prm[a] * (x * x);
    }
    r = e - prm[d];
  } else {
    // hyper_rectangle (shapes.py:69-83): q_a = max(lo-x, x-hi);
    // outside = sqrt(0 + sum max(q_a,0)**2); inside = min(max_a q_a, 0)
    double s = 0.0, qmax = -INFINITY;
    for (int a = 0; a < d; ++a) {
      const double x = G.nodes[a][ix[a]];
      const double q1 = prm[a] - x, q2 = x - prm[d + a];
      const double q = (q1 >= q2) ? q1 : q2;
      const double qp = (q >= 0.0) ? q : 0.0;
      s = s + qp * qp;
      qmax = (a == 0 || q > qmax) ? q : qmax;
    }
    const double inside = (qmax <= 0.0) ? qmax : 0.0;
    r = sqrt(s) + inside;
  }
  out[off] = r;
}

// ------------------------------------------------------------------ elementwise helpers
__global__ void k_csg(int op, long long n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i];
  double r;
  switch (op) {
    case HJ_CSG_UNION: { const double y = b[i]; r = (y < x) ? y : x; } break;       // np.minimum
    case HJ_CSG_INTERSECT: { const double y = b[i]; r = (y > x) ? y : x; } break;   // np.maximum
    case HJ_CSG_COMPLEMENT: r = -x; break;                                          // negate
    default: { const double y = -b[i]; r = (y > x) ? y : x; } break;                // max(a, -b)
  }
  out[i] = r;
}

__global__ void k_mask(long long n, const double* __restrict__ prev, double* __restrict__ v, int mask) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = v[i], p = prev[i];
  v[i] = (mask == HJ_MASK_MIN) ? ((p < x) ? p : x) : ((p > x) ? p : x);
}

__global__ void k_count_below(long long n, const double* __restrict__ v, double level,
                              unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += (v[i] < level) ? 1ull : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// Tube acceptance checks on the device (reference: test_reachability.py:218-285
// over the mask of reachability.py:249), so a solve can verify its own tube
// without copying fields to the host.  out[0] nesting violations (v above
// prev for the min mask / below for the max mask), out[1] target-containment
// violations (v above / below the target), out[2] #{v < level}, out[3]
// #{prev >= level and v < level} (nodes captured during the interval).
__global__ void k_tube_check(long long n, const double* __restrict__ prev, const double* __restrict__ v,
                             const double* __restrict__ target, int mask_min, double level,
                             unsigned long long* __restrict__ out) {
  unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = prev[i], b = v[i], g = target[i];
    c0 += (mask_min ? (b > a) : (b < a)) ? 1ull : 0ull;
    c1 += (mask_min ? (b > g) : (b < g)) ? 1ull : 0ull;
    c2 += (b < level) ? 1ull : 0ull;
    c3 += (!(a < level) && b < level) ? 1ull : 0ull;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    c3 += __shfl_xor_sync(0xffffffffu, c3, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (c0) atomicAdd(&out[0], c0);
    if (c1) atomicAdd(&out[1], c1);
    if (c2) atomicAdd(&out[2], c2);
    if (c3) atomicAdd(&out[3], c3);
  }
}

__global__ void k_stats_reset(hj_stats* st) {
  const int t = threadIdx.x;
  if (t < HJ_MAX_DIM) {
    st->lo_key[t] = KEY_POS_INF;
    st->hi_key[t] = KEY_NEG_INF;
  }
  if (t == 0) {
    st->nonfinite = 0u;
    st->first_bad_tag = 0x7fffffff;
  }
}

// ------------------------------------------------------------------ host-Hamiltonian bridge
struct PtrSet {
  const double* l[HJ_MAX_DIM];
  const double* r[HJ_MAX_DIM];
  double* p[HJ_MAX_DIM];
};

template <int DIM>
__global__ void __launch_bounds__(256) k_costates(const GridArgs G, const PtrSet S, hj_stats* st) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = G.cells * G.batch;
  long long lo[DIM], hi[DIM];
  unsigned flags = 0u;
#pragma unroll
  for (int a = 0; a < DIM; ++a) { lo[a] = KEY_POS_INF; hi[a] = KEY_NEG_INF; }
  if (idx < total) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double l = S.l[a][idx], r = S.r[a][idx];
      if (!finite(l) || !finite(r)) flags |= HJ_NF_DERIV;
      S.p[a][idx] = 0.5 * (l + r);                       // term.py:101
      lo[a] = min(order_key(l), order_key(r));           // term.py:71-77
      hi[a] = max(order_key(l), order_key(r));
    }
  }
  if (st) reduce_stats<DIM>(st, flags, 0, true, lo, hi);
}

template <int DIM>
__global__ void __launch_bounds__(256) k_glf_delta(const GridArgs G, const PtrSet S, const double* ahalf_dev,
                                                   double a0, double a1, double a2, double a3,
                                                   const double* __restrict__ ham, double* __restrict__ diss_out,
                                                   double* __restrict__ delta, hj_stats* st) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = G.cells * G.batch;
  unsigned flags = 0u;
  long long dummy[1] = {0};
  if (idx < total) {
    const double ah[4] = {a0, a1, a2, a3};
    double diss = 0.0;                                   // term.py:84
#pragma unroll
    for (int a = 0; a < DIM; ++a) diss = diss + ah[a] * (S.r[a][idx] - S.l[a][idx]);  // term.py:85-86
    if (diss_out) diss_out[idx] = diss;
    const double d = diss - ham[idx];                    // term.py:113
    if (!finite(d)) flags |= HJ_NF_DELTA;
    delta[idx] = d;
  }
  if (st) reduce_stats<1>(st, flags, 0, false, dummy, dummy);
}

__global__ void k_rk_combine(long long n, int stage, double dt, const double* __restrict__ y,
                             const double* __restrict__ y0, const double* __restrict__ delta,
                             double* __restrict__ out, hj_stats* st, int tag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned flags = 0u;
  long long dummy[1] = {0};
  if (i < n) {
    const double d = delta[i];
    if (!finite(d)) flags |= HJ_NF_DELTA;
    const double o = stage_update(stage, dt, y[i], (stage >= HJ_STAGE_RK2_AVG) ? y0[i] : 0.0, d);
    if (!finite(o)) flags |= HJ_NF_OUTPUT;
    out[i] = o;
  }
  if (st) reduce_stats<1>(st, flags, tag, false, dummy, dummy);
}

// ------------------------------------------------------------------ launchers
static inline unsigned nblocks(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

cudaError_t launch_extend(const GridArgs& G, int w, const double* v, double* ext, cudaStream_t s) {
  long long total = 1;
  for (int a = 0; a < G.dim; ++a) total *= (G.n[a] + 2 * w);
  k_extend<<<nblocks(total, 256), 256, 0, s>>>(G, w, v, ext, total);
  return cudaGetLastError();
}

cudaError_t launch_shape(const GridArgs& G, int kind, const double* prm, int nprm, double* out, cudaStream_t s) {
  ShapeParams P{};
  for (int i = 0; i < nprm && i < 16; ++i) P.v[i] = prm[i];
  k_shape<<<nblocks(G.cells * G.batch, 256), 256, 0, s>>>(G, kind, P, out);
  return cudaGetLastError();
}

cudaError_t launch_csg(int op, long long n, const double* a, const double* b, double* out, cudaStream_t s) {
  k_csg<<<nblocks(n, 256), 256, 0, s>>>(op, n, a, b, out);
  return cudaGetLastError();
}

cudaError_t launch_mask(long long n, const double* prev, double* v, int mask, cudaStream_t s) {
  k_mask<<<nblocks(n, 256), 256, 0, s>>>(n, prev, v, mask);
  return cudaGetLastError();
}

cudaError_t launch_count_below(long long n, const double* v, double level, unsigned long long* c,
                               cudaStream_t s) {
  long long b = nblocks(n, 256);
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  k_count_below<<<(unsigned)b, 256, 0, s>>>(n, v, level, c);
  return cudaGetLastError();
}

cudaError_t launch_tube_check(long long n, const double* prev, const double* v, const double* target, int mask_min,
                              double level, unsigned long long* out, cudaStream_t s) {
  long long b = nblocks(n, 256);
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  k_tube_check<<<(unsigned)b, 256, 0, s>>>(n, prev, v, target, mask_min, level, out);
  return cudaGetLastError();
}

cudaError_t launch_stats_reset(hj_stats* st, cudaStream_t s) {
  k_stats_reset<<<1, 32, 0, s>>>(st);
  return cudaGetLastError();
}

cudaError_t launch_costates(const GridArgs& G, const double* const* l, const double* const* r,
                            double* const* p, hj_stats* st, cudaStream_t s) {
  PtrSet S{};
  for (int a = 0; a < G.dim; ++a) { S.l[a] = l[a]; S.r[a] = r[a]; S.p[a] = p[a]; }
  const unsigned b = nblocks(G.cells * G.batch, 256);
  switch (G.dim) {
    case 1: k_costates<1><<<b, 256, 0, s>>>(G, S, st); break;
    case 2: k_costates<2><<<b, 256, 0, s>>>(G, S, st); break;
    case 3: k_costates<3><<<b, 256, 0, s>>>(G, S, st); break;
    default: k_costates<4><<<b, 256, 0, s>>>(G, S, st); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_glf_delta(const GridArgs& G, const double* ahalf, const double* const* l,
                             const double* const* r, const double* ham, double* diss, double* delta,
                             hj_stats* st, cudaStream_t s) {
  PtrSet S{};
  for (int a = 0; a < G.dim; ++a) { S.l[a] = l[a]; S.r[a] = r[a]; }
  const unsigned b = nblocks(G.cells * G.batch, 256);
  double a4[4] = {0, 0, 0, 0};
  for (int a = 0; a < G.dim && a < 4; ++a) a4[a] = ahalf[a];
  switch (G.dim) {
    case 1: k_glf_delta<1><<<b, 256, 0, s>>>(G, S, nullptr, a4[0], a4[1], a4[2], a4[3], ham, diss, delta, st); break;
    case 2: k_glf_delta<2><<<b, 256, 0, s>>>(G, S, nullptr, a4[0], a4[1], a4[2], a4[3], ham, diss, delta, st); break;
    case 3: k_glf_delta<3><<<b, 256, 0, s>>>(G, S, nullptr, a4[0], a4[1], a4[2], a4[3], ham, diss, delta, st); break;
    default: k_glf_delta<4><<<b, 256, 0, s>>>(G, S, nullptr, a4[0], a4[1], a4[2], a4[3], ham, diss, delta, st); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_rk_combine(long long n, int stage, double dt, const double* y, const double* y0,
                              const double* delta, double* out, hj_stats* st, int tag, cudaStream_t s) {
  k_rk_combine<<<nblocks(n, 256), 256, 0, s>>>(n, stage, dt, y, y0, delta, out, st, tag);
  return cudaGetLastError();
}

}  // namespace hj
