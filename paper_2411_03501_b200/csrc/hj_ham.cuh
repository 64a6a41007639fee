// hj_ham.cuh -- registered device Hamiltonians (TermConfig.hamiltonian,
// term.py:29).  Each evaluates H(x, p_avg) at one node with the reference's
// (or the pinned builder fixture's) left-to-right operation order.  Trig
// values come from host tables (np.cos/np.sin), never recomputed here.
#pragma once
#include "hj_math.cuh"

namespace hj {

// H in two parts: the node-table inputs c[0..3] of the node, then H of
// (c, p_avg).  Inputs per Hamiltonian:
//   ROCKETS / EXTREMAL: c0 = x (axis-0 node), c2 = cos th, c3 = sin th (axis-2 tables)
//   AIR3D:              c0 = x, c1 = y (axis-1 node), c2 = v_b cos psi, c3 = v_b sin psi
//   DI4:                c0 = w_x (axis-2 node), c1 = w_y (axis-3 node)
//   ADVECTION:          none
// ix[a] = index along axis a of the (owned) grid, nodes[a] = device copy of
// g.axis_nodes[a] for that slab.  The brick kernel stages the inputs of a
// whole brick in shared memory and calls ham_eval directly.
template <int HAM, int DIM>
__device__ __forceinline__ void ham_inputs(const hj_ham& H, const double* const* nodes, const int* ix, double* c) {
  if (HAM == HJ_HAM_ROCKETS || HAM == HJ_HAM_ROCKETS_EXTREMAL) {
    c[0] = nodes[0][ix[0]];
    c[2] = H.tab[0][ix[2]];
    c[3] = H.tab[1][ix[2]];
  } else if (HAM == HJ_HAM_AIR3D) {
    c[0] = nodes[0][ix[0]];
    c[1] = nodes[1][ix[1]];
    c[2] = H.tab[0][ix[2]];
    c[3] = H.tab[1][ix[2]];
  } else if (HAM == HJ_HAM_DI4) {
    c[0] = nodes[2][ix[2]];
    c[1] = nodes[3][ix[3]];
  }
}

template <int HAM, int DIM>
__device__ __forceinline__ double ham_eval(const hj_ham& H, const double* c, const double* p) {
  if (HAM == HJ_HAM_ADVECTION) {
    // term.py:136-140: out = zeros; out += c_i * p_i (axis order)
    double out = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) out = out + H.p[a] * p[a];
    return out;
  } else if (HAM == HJ_HAM_ROCKETS) {
    // reachability.py:70-80
    const double a = H.p[0], grav = H.p[1], u_min = H.p[2], u_max = H.p[3];
    const double x = c[0], ct = c[2], st = c[3];
    const double p1 = p[0], p2 = p[1], p3 = p[2];
    const double t1 = ((-a) * p1) * ct;
    const double t2 = p2 * ((grav - a) - a * st);
    const double t3 = u_max * fabs(p1 * x + p3);
    const double t4 = u_min * fabs(p2 * x + p3);
    return ((t1 - t2) - t3) + t4;
  } else if (HAM == HJ_HAM_ROCKETS_EXTREMAL) {
    // reachability.py:101-115; p[4] = mid, p[5] = half precomputed on the host
    const double a = H.p[0], grav = H.p[1], mid = H.p[4], half = H.p[5];
    const double x = c[0], ct = c[2], st = c[3];
    const double p1 = p[0], p2 = p[1], p3 = p[2];
    const double c1 = p1 * x - p3;
    const double c2 = p2 * x + p3;
    const double t1 = ((-a) * p1) * ct;
    const double t2 = p2 * ((grav - a) - a * st);
    return (((t1 + t2) - mid * (c1 + c2)) - half * fabs(c1)) + half * fabs(c2);
  } else if (HAM == HJ_HAM_AIR3D) {
    // builder fixture (paper_2411_03501_b200/problems.py air3d_hamiltonian):
    // H = -((((-va*p1 + vbcos*p1) + vbsin*p2) + a*|(y*p1 - x*p2) - p3|) - b*|p3|)
    const double va = H.p[0], a_in = H.p[2], b_in = H.p[3];
    const double x = c[0], y = c[1], vbc = c[2], vbs = c[3];
    const double p1 = p[0], p2 = p[1], p3 = p[2];
    const double s = (((-va) * p1 + vbc * p1) + vbs * p2) + a_in * fabs((y * p1 - x * p2) - p3);
    return -(s - b_in * fabs(p3));
  } else {
    // HJ_HAM_DI4 builder fixture (problems.py di4_hamiltonian):
    // H = -((p1*wx + p2*wy) + (d_bar - u_bar)*(|p3| + |p4|)); p[2] = d_bar - u_bar
    const double k = H.p[2];
    const double wx = c[0], wy = c[1];
    return -((p[0] * wx + p[1] * wy) + k * (fabs(p[2]) + fabs(p[3])));
  }
}

template <int HAM, int DIM>
__device__ __forceinline__ double hamiltonian(const hj_ham& H, const double* const* nodes,
                                              const int* ix, const double* p) {
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  ham_inputs<HAM, DIM>(H, nodes, ix, c);
  return ham_eval<HAM, DIM>(H, c, p);
}

}  // namespace hj
