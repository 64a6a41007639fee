"""Builder-supplied Hamiltonians for the benchmark configurations.

Air3D and the 4-D relative double integrator are not in the reference
("no formulas given").  They plug into the reference's own
TermConfig contract; the operation order is pinned here and mirrored by the
device functors (csrc/hj_ham.cuh) and by tests/golden/make_golden.py, which
ran them through the reference's term / integrator / solve_brt to make the
golden vectors.

Air3D (Mitchell's toolbox constants): relative state (x, y, psi), psi periodic,
    H = -( -v_a p1 + v_b cos(psi) p1 + v_b sin(psi) p2
           + a |y p1 - x p2 - p3| - b |p3| )
    alpha = (max|-v_a + v_b cos psi| + a max|y|, max|v_b sin psi| + a max|x|, a + b)

Relative double integrator pair: (p_x, p_y, w_x, w_y), p' = w, w' = d - u,
|u|_inf <= u_bar, |d|_inf <= d_bar,
    H = -( p1 w_x + p2 w_y + (d_bar - u_bar)(|p3| + |p4|) )
    alpha = (max|w_x|, max|w_y|, u_bar + d_bar, u_bar + d_bar)
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .grid import Grid, ScalarField, create_grid
from .term import DeviceHamiltonian, RangeFreePartials, TermConfig


@dataclass(frozen=True)
class Air3DParams:
    v_a: float = 5.0
    v_b: float = 5.0
    a_in: float = 1.0      # evader turn-rate bound
    b_in: float = 1.0      # pursuer turn-rate bound
    radius: float = 5.0    # capture radius of the target cylinder


AIR3D_BOUNDS = ((-6.0, -10.0, 0.0), (20.0, 10.0, 2 * math.pi))


def air3d_tables(g: Grid, p: Air3DParams):
    psi = g.axis_nodes[2]
    return p.v_b * np.cos(psi), p.v_b * np.sin(psi)


class Air3DHamiltonian(DeviceHamiltonian):
    kind = _lib.HAM_AIR3D
    dim = 3

    def __init__(self, params: Air3DParams):
        self.p = params

    def params(self):
        return (self.p.v_a, self.p.v_b, self.p.a_in, self.p.b_in)

    def tables(self, g):
        return air3d_tables(g, self.p)


class Air3DPartials(RangeFreePartials):
    def __init__(self, params: Air3DParams):
        self.p = params

    def alphas(self, t, g):
        vbc, vbs = air3d_tables(g, self.p)
        x, y = g.axis_nodes[0], g.axis_nodes[1]
        return np.array([
            float(np.max(np.abs(-self.p.v_a + vbc))) + self.p.a_in * float(np.max(np.abs(y))),
            float(np.max(np.abs(vbs))) + self.p.a_in * float(np.max(np.abs(x))),
            self.p.a_in + self.p.b_in,
        ])


def air3d_term_config(params: Air3DParams | None = None, scheme: str = "weno5") -> TermConfig:
    params = params or Air3DParams()
    return TermConfig(hamiltonian=Air3DHamiltonian(params), partials=Air3DPartials(params),
                      derivative_scheme=scheme)


def air3d_grid(n: int | tuple[int, int, int]) -> Grid:
    counts = (n, n, n) if isinstance(n, int) else tuple(n)
    return create_grid(AIR3D_BOUNDS[0], AIR3D_BOUNDS[1], counts, periodic_axes={2})


@dataclass(frozen=True)
class DI4Params:
    u_bar: float = 1.0
    d_bar: float = 0.5
    radius: float = 2.0


DI4_BOUNDS = ((-8.0, -8.0, -4.0, -4.0), (8.0, 8.0, 4.0, 4.0))


class DI4Hamiltonian(DeviceHamiltonian):
    kind = _lib.HAM_DI4
    dim = 4

    def __init__(self, params: DI4Params):
        self.p = params

    def params(self):
        return (self.p.u_bar, self.p.d_bar)


class DI4Partials(RangeFreePartials):
    def __init__(self, params: DI4Params):
        self.p = params

    def alphas(self, t, g):
        s = self.p.u_bar + self.p.d_bar
        return np.array([float(np.max(np.abs(g.axis_nodes[2]))), float(np.max(np.abs(g.axis_nodes[3]))), s, s])


def di4_term_config(params: DI4Params | None = None, scheme: str = "weno5") -> TermConfig:
    params = params or DI4Params()
    return TermConfig(hamiltonian=DI4Hamiltonian(params), partials=DI4Partials(params), derivative_scheme=scheme)


def di4_grid(n: int | tuple[int, int, int, int]) -> Grid:
    counts = (n,) * 4 if isinstance(n, int) else tuple(n)
    return create_grid(DI4_BOUNDS[0], DI4_BOUNDS[1], counts)


def di4_target(g: Grid, params: DI4Params | None = None) -> ScalarField:
    """sqrt(p_x^2 + p_y^2) - radius: a cylinder ignoring both velocity axes."""
    from .shapes import cylinder_mask

    params = params or DI4Params()
    return cylinder_mask(g, (0b1100), (0.0, 0.0, 0.0, 0.0), params.radius)
