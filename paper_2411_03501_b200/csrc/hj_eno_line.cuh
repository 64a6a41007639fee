// hj_eno_line.cuh -- first-order / ENO2 / ENO3 upwind pairs along one line,
// every divided difference computed once (rolling window), divisions by the
// line constants h, 2h, 3h with hoisted reciprocals (div_by, bit-identical to
// '/').  Operation order: spatial.py:119-179.
//
//   D1f(j) = (v[j+1]-v[j])/h           face between j and j+1
//   D2c(j) = (D1f(j)-D1f(j-1))/(2h)    node j
//   D3f(j) = (D2c(j+1)-D2c(j))/(3h)    face between j and j+1
#pragma once
#include "hj_math.cuh"

namespace hj {

struct EnoDivisors {
  Recip h, h2, h3;
  double hv;
};

__device__ __forceinline__ EnoDivisors eno_divisors(const Spacing& s) {
  EnoDivisors K;
  K.h = make_recip(s.h);
  K.h2 = make_recip(s.h2);
  K.h3 = make_recip(s.h3);
  K.hv = s.h;
  return K;
}

// ld(k) for k in [-1, n]; emit(i, left, right)
template <class Load, class Emit>
__device__ __forceinline__ void first_line(const Load& ld, int n, const EnoDivisors& K, const Emit& emit) {
  double u = ld(-1);
  double un = ld(0);
  double dm = div_by(un - u, K.h);  // D1f(i-1)
  u = un;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    un = ld(i + 1);
    const double d0 = div_by(un - u, K.h);  // D1f(i)
    u = un;
    emit(i, dm, d0);
    dm = d0;
  }
}

// ld(k) for k in [-2, n+1]
template <class Load, class Emit>
__device__ __forceinline__ void eno2_line(const Load& ld, int n, const EnoDivisors& K, const Emit& emit) {
  double u = ld(-2), un;
  un = ld(-1); const double fm2 = div_by(un - u, K.h); u = un;   // D1f(-2)
  un = ld(0);  double fm1 = div_by(un - u, K.h); u = un;         // D1f(-1)
  un = ld(1);  double f0 = div_by(un - u, K.h); u = un;          // D1f(0)
  double cm1 = div_by(fm1 - fm2, K.h2);                          // D2c(-1)
  double c0 = div_by(f0 - fm1, K.h2);                            // D2c(0)
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    un = ld(i + 2);
    const double fp1 = div_by(un - u, K.h);                      // D1f(i+1)
    u = un;
    const double cp1 = div_by(fp1 - f0, K.h2);                   // D2c(i+1)
    const double L = fm1 + pick_smaller(cm1, c0) * K.hv;         // spatial.py:137
    const double R = f0 - pick_smaller(c0, cp1) * K.hv;          // spatial.py:140
    emit(i, L, R);
    fm1 = f0; f0 = fp1;
    cm1 = c0; c0 = cp1;
  }
}

// ld(k) for k in [-3, n+2]
template <class Load, class Emit>
__device__ __forceinline__ void eno3_line(const Load& ld, int n, const EnoDivisors& K, const Emit& emit) {
  double f[5];
  double u = ld(-3), un;
#pragma unroll
  for (int k = 0; k < 5; ++k) {           // D1f(-3) .. D1f(1)
    un = ld(k - 2);
    f[k] = div_by(un - u, K.h);
    u = un;
  }
  double c[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k] = div_by(f[k + 1] - f[k], K.h2);   // D2c(-2) .. D2c(1)
  double tm2 = div_by(c[1] - c[0], K.h3);  // D3f(-2)
  double tm1 = div_by(c[2] - c[1], K.h3);  // D3f(-1)
  double t0 = div_by(c[3] - c[2], K.h3);   // D3f(0)
  double fm1 = f[2], f0 = f[3], fp1 = f[4];      // D1f(i-1), D1f(i), D1f(i+1)
  double cm1 = c[1], c0 = c[2], cp1 = c[3];      // D2c(i-1), D2c(i), D2c(i+1)
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    un = ld(i + 3);
    const double fp2 = div_by(un - u, K.h);              // D1f(i+2)
    u = un;
    const double cp2 = div_by(fp2 - fp1, K.h2);          // D2c(i+2)
    const double tp1 = div_by(cp2 - cp1, K.h3);          // D3f(i+1)
    const bool lc = fabs(cm1) <= fabs(c0);
    const bool rc = fabs(c0) <= fabs(cp1);
    const double l2 = fm1 + (lc ? cm1 : c0) * K.hv;
    const double r2 = f0 - (rc ? c0 : cp1) * K.hv;
    double first = lc ? tm2 : tm1, second = lc ? tm1 : t0, mult = lc ? 2.0 : -1.0;
    const double L = l2 + ((pick_smaller(first, second) * mult) * K.hv) * K.hv;   // spatial.py:173
    first = rc ? tm1 : t0;
    second = rc ? t0 : tp1;
    mult = rc ? -1.0 : 2.0;
    const double R = r2 + ((pick_smaller(first, second) * mult) * K.hv) * K.hv;   // spatial.py:178
    emit(i, L, R);
    fm1 = f0; f0 = fp1; fp1 = fp2;
    cm1 = c0; c0 = cp1; cp1 = cp2;
    tm2 = tm1; tm1 = t0; t0 = tp1;
  }
}

}  // namespace hj
