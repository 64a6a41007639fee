"""Upwind one-sided derivatives -- drop-in for hjls.spatial, computed on the GPU.

Each function returns the (left, right) pair along one axis
(spatial.py:1-24 for the conventions).  The arithmetic runs in the sm_100a
kernels of libhjb200.so (hj_derivs, hj_weno5_workspace,
hj_divided_differences); results equal the reference value for value.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device as dev
from .grid import Grid, ScalarField

GHOST_WIDTH = {"first": 1, "eno2": 2, "eno3": 3, "weno5": 3}   # spatial.py:27
# Schemes beyond the reference's registry: "weno5_fma" is WENO5 evaluated in
# tolerance mode (FMA, reciprocal multiplies, one division per side; within
# the north-star 1e-9 contract instead of bit-exact -- hjb200.h HJ_WENO5_FMA).
TOLERANCE_SCHEMES = {"weno5_fma": 3}
SCHEME_WIDTH = {**GHOST_WIDTH, **TOLERANCE_SCHEMES}


@dataclass(frozen=True)
class DerivativePair:
    """Left/backward and right/forward derivative fields along one axis."""

    left: ScalarField
    right: ScalarField
    axis: int


@dataclass(frozen=True)
class DividedDifferenceTable:
    """Divided differences over the ghost extension of one axis, axis last
    (spatial.py:42-56).  ``d2``/``d3`` are None when not requested."""

    d0: np.ndarray
    d1: np.ndarray
    d2: np.ndarray | None
    d3: np.ndarray | None
    spacing: float


@dataclass(frozen=True)
class WenoWorkspace:
    """Per-node WENO diagnostics of one side, working axis last (spatial.py:58-71)."""

    sigma1: np.ndarray
    sigma2: np.ndarray
    sigma3: np.ndarray
    alpha1: np.ndarray
    alpha2: np.ndarray
    alpha3: np.ndarray
    eps: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray


def _validate(g: Grid, f: ScalarField, axis: int) -> None:
    # spatial.py:76-79
    if not 0 <= axis < g.dim:
        raise ValueError(f"axis {axis} out of range for dim {g.dim}")
    if not f.matches(g):
        raise ValueError(f"field shape {f.grid_shape} does not match grid {g.counts}")


def _pair(g: Grid, f: ScalarField, axis: int, scheme: str, eps_mode: str = "squared") -> DerivativePair:
    _validate(g, f, axis)
    dg = dev.device_grid(g)
    L, R = dev.derivs_dev(dg, dev.to_dev(f.values), axis, scheme, eps_mode)
    return DerivativePair(left=ScalarField(dev.to_host(L)), right=ScalarField(dev.to_host(R)), axis=axis)


def upwind_first_first(g: Grid, f: ScalarField, axis: int) -> DerivativePair:
    """First-order pair: backward / forward differences (spatial.py:119-126)."""
    return _pair(g, f, axis, "first")


def upwind_first_eno2(g: Grid, f: ScalarField, axis: int) -> DerivativePair:
    """Second-order ENO pair (spatial.py:147-153)."""
    return _pair(g, f, axis, "eno2")


def upwind_first_eno3(g: Grid, f: ScalarField, axis: int) -> DerivativePair:
    """Third-order ENO pair (spatial.py:156-179)."""
    return _pair(g, f, axis, "eno3")


def _eps_mode(eps_mode: str) -> str:
    if eps_mode not in ("squared", "raw"):
        raise ValueError(f"eps_mode must be 'squared' or 'raw', got {eps_mode!r}")
    return eps_mode


def upwind_first_weno5(g: Grid, f: ScalarField, axis: int, eps_mode: str = "squared") -> DerivativePair:
    """Fifth-order WENO pair, Jiang-Peng weights (spatial.py:239-247)."""
    return _pair(g, f, axis, "weno5", _eps_mode(eps_mode))


def upwind_first_weno5_fma(g: Grid, f: ScalarField, axis: int) -> DerivativePair:
    """WENO5 pair in tolerance mode (same scheme as upwind_first_weno5, "squared"
    epsilon; agrees with it to rounding, not bitwise -- hjb200.h HJ_WENO5_FMA)."""
    return _pair(g, f, axis, "weno5_fma")


def weno5_workspace(g: Grid, f: ScalarField, axis: int, side: str = "left",
                    eps_mode: str = "squared") -> WenoWorkspace:
    """WENO smoothness / weight internals of one side (spatial.py:250-257)."""
    _validate(g, f, axis)
    if side not in ("left", "right"):
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    _eps_mode(eps_mode)
    ws = dev.to_host(dev.weno5_workspace_dev(dev.device_grid(g), dev.to_dev(f.values), axis, side, eps_mode))
    # the reference leaves the working axis last
    fields = [np.ascontiguousarray(np.moveaxis(ws[k], axis, -1)) for k in range(10)]
    return WenoWorkspace(*fields)


def divided_differences(g: Grid, f: ScalarField, axis: int, order: int = 3,
                        width: int | None = None) -> DividedDifferenceTable:
    """Divided-difference table over the ghost extension (spatial.py:99-106)."""
    if not 1 <= order <= 3:
        raise ValueError(f"order must be 1..3, got {order}")
    w = order if width is None else width
    _validate(g, f, axis)
    d0, d1, d2, d3 = dev.divided_differences_dev(dev.device_grid(g), dev.to_dev(f.values), axis, order, w)
    host = lambda t: None if t is None else dev.to_host(t)  # noqa: E731
    return DividedDifferenceTable(d0=host(d0), d1=host(d1), d2=host(d2), d3=host(d3),
                                  spacing=float(g.spacings[axis]))


_SCHEMES = {
    "first": upwind_first_first,
    "eno2": upwind_first_eno2,
    "eno3": upwind_first_eno3,
    "weno5": upwind_first_weno5,
    "weno5_fma": upwind_first_weno5_fma,
}


def derivative_pair(g: Grid, f: ScalarField, axis: int, scheme: str) -> DerivativePair:
    """Dispatch by scheme name (spatial.py:268-276)."""
    if scheme not in _SCHEMES:
        raise ValueError(f"unknown derivative scheme {scheme!r}; pick from {sorted(_SCHEMES)}")
    return _SCHEMES[scheme](g, f, axis)
