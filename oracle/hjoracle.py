"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the HJ grid-update path.

Python face of oracle/hjoracle.c (a C restatement of the reference,
/root/reference/pkg/src/hjls, -ffp-contract=off) plus the host loops of the
reference integrator and tube driver restated over it.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module; the product package never does.

Pinning: tests/test_oracle_golden.py compares every entry point with golden
vectors that tests/golden/make_golden.py produced by running the reference
itself.

Grids are duck-typed: anything with the reference Grid's attributes (dim,
counts, spacings, boundary[i].kind/.value, axis_nodes) works, so the same
oracle checks the reference's grids and the package's.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhjoracle.so")
MAXD = 5

SCHEMES = {"first": 0, "eno2": 1, "eno3": 2, "weno5": 3}
BCS = {"periodic": 0, "extrapolate": 1, "dirichlet": 2}
HAMS = {"advection": 0, "rockets": 1, "rockets_extremal": 2, "air3d": 3, "di4": 4}


class OrGrid(ctypes.Structure):
    _fields_ = [
        ("dim", c_int),
        ("n", c_int64 * MAXD),
        ("h", c_double * MAXD),
        ("bc", c_int * MAXD),
        ("bcv", c_double * MAXD),
        ("nodes", c_void_p * MAXD),
    ]


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc; no reference build system)."""
    r = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = POINTER(OrGrid)
        L.or_derivs.argtypes = [P, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]
        L.or_weno_workspace.argtypes = [P, c_int, c_int, c_int, c_void_p, c_void_p]
        L.or_extend_ghost.argtypes = [P, c_int, c_void_p, c_void_p]
        L.or_hamiltonian.argtypes = [P, c_int, c_void_p, c_void_p, c_void_p, c_void_p]
        L.or_term.argtypes = [P, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p]
        L.or_term.restype = c_int
        L.or_stage.argtypes = [c_int64, c_int, c_double, c_void_p, c_void_p, c_void_p, c_void_p]
        L.or_mask.argtypes = [c_int64, c_void_p, c_void_p, c_int]
        L.or_shape.argtypes = [P, c_int, c_void_p, c_void_p]
        L.or_set_threads.argtypes = [c_int]
        L.or_get_threads.restype = c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class _G:
    """Keeps the numpy buffers alive while the C struct points at them."""

    def __init__(self, g):
        self.s = OrGrid()
        self.s.dim = int(g.dim)
        self.keep = []
        for a in range(g.dim):
            self.s.n[a] = int(g.counts[a])
            self.s.h[a] = float(g.spacings[a])
            self.s.bc[a] = BCS[g.boundary[a].kind]
            self.s.bcv[a] = float(g.boundary[a].value)
            nodes = np.ascontiguousarray(g.axis_nodes[a], dtype=np.float64)
            self.keep.append(nodes)
            self.s.nodes[a] = _ptr(nodes)

    @property
    def ref(self):
        return ctypes.byref(self.s)


def _f64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64))


# ---------------------------------------------------------------- spatial
def derivs(g, v, axis: int, scheme: str, eps_mode: str = "squared"):
    """derivative_pair / upwind_first_* (spatial.py:119-276) -> (left, right)."""
    v = _f64(v).reshape(tuple(g.counts))
    L, R = np.empty_like(v), np.empty_like(v)
    G = _G(g)
    lib().or_derivs(G.ref, SCHEMES[scheme], axis, 1 if eps_mode == "raw" else 0, _ptr(v), _ptr(L), _ptr(R))
    return L, R


def weno5_workspace(g, v, axis: int, side: str = "left", eps_mode: str = "squared") -> dict:
    """weno5_workspace (spatial.py:250-257) -> dict of the 10 diagnostic fields."""
    v = _f64(v).reshape(tuple(g.counts))
    ws = np.empty((10,) + v.shape)
    G = _G(g)
    lib().or_weno_workspace(G.ref, axis, 0 if side == "left" else 1, 1 if eps_mode == "raw" else 0, _ptr(v),
                            _ptr(ws))
    names = ("sigma1", "sigma2", "sigma3", "alpha1", "alpha2", "alpha3", "eps", "w1", "w2", "w3")
    # the reference leaves the working axis last (spatial.py:250-257 never restores it)
    return {k: np.ascontiguousarray(np.moveaxis(ws[i], axis, -1)) for i, k in enumerate(names)}


def extend_ghost(g, v, width: int) -> np.ndarray:
    """extend_with_ghost_cells (grid.py:228-243)."""
    v = _f64(v).reshape(tuple(g.counts))
    out = np.empty(tuple(n + 2 * width for n in g.counts))
    G = _G(g)
    lib().or_extend_ghost(G.ref, width, _ptr(v), _ptr(out))
    return out


def divided_differences(g, v, axis: int, order: int = 3, width: int | None = None):
    """divided_differences (spatial.py:99-106) as plain numpy over the oracle's
    single-axis ghost extension -> (d0, d1, d2|None, d3|None), axis last."""
    w = order if width is None else width
    ext = _extend_one_axis(g, v, axis, w)
    h = float(g.spacings[axis])
    d1 = np.diff(ext, axis=-1) / h
    d2 = np.diff(d1, axis=-1) / (2.0 * h) if order >= 2 else None
    d3 = np.diff(d2, axis=-1) / (3.0 * h) if order >= 3 else None
    return ext, d1, d2, d3


def _extend_one_axis(g, v, axis, w):
    # grid.py:203-225, restated for one axis through the C line extender
    # (extend_ghost on a 1-axis view): move the axis last, extend every line.
    v = _f64(v).reshape(tuple(g.counts))
    work = np.moveaxis(v, axis, -1)
    n = work.shape[-1]
    lines = np.ascontiguousarray(work.reshape(-1, n))

    class _Line:
        dim = 1
        counts = (n,)
        spacings = np.array([float(g.spacings[axis])])
        boundary = (g.boundary[axis],)
        axis_nodes = (np.asarray(g.axis_nodes[axis], dtype=np.float64),)

    out = np.stack([extend_ghost(_Line, row, w) for row in lines]) if lines.shape[0] else np.empty((0, n + 2 * w))
    return out.reshape(work.shape[:-1] + (n + 2 * w,))


# ---------------------------------------------------------------- Hamiltonians
class Ham:
    """A registered Hamiltonian for the oracle: kind, constants, tables, alphas."""

    def __init__(self, kind: str, prm, tabs=(), alphas=None):
        self.kind = kind
        self.prm = np.zeros(16)
        self.prm[: len(prm)] = [float(x) for x in prm]
        self.tabs = [_f64(t) for t in tabs]
        self.alphas = None if alphas is None else _f64(alphas)

    def tab_array(self):
        arr = (c_void_p * 4)()
        for i, t in enumerate(self.tabs):
            arr[i] = _ptr(t)
        return arr


def hamiltonian(g, ham: Ham, p) -> np.ndarray:
    ps = [_f64(x).reshape(tuple(g.counts)) for x in p]
    out = np.empty(tuple(g.counts))
    parr = (c_void_p * MAXD)()
    for i, x in enumerate(ps):
        parr[i] = _ptr(x)
    G = _G(g)
    tabs = ham.tab_array()
    lib().or_hamiltonian(G.ref, HAMS[ham.kind], _ptr(ham.prm), ctypes.addressof(tabs), ctypes.addressof(parr),
                         _ptr(out))
    return out


def term(g, ham: Ham, scheme: str, v, alphas=None):
    """term_lax_friedrichs (term.py:90-126) for a range-free registered H.
    Returns (delta, step_bound, ranges, h_nonzero)."""
    v = _f64(v).reshape(tuple(g.counts))
    alphas = _f64(ham.alphas if alphas is None else alphas)
    delta = np.empty_like(v)
    lo, hi = np.empty(MAXD), np.empty(MAXD)
    G = _G(g)
    tabs = ham.tab_array()
    nz = lib().or_term(G.ref, SCHEMES[scheme], HAMS[ham.kind], _ptr(ham.prm), ctypes.addressof(tabs),
                       _ptr(alphas), _ptr(v), _ptr(delta), _ptr(lo), _ptr(hi))
    inv_bound = float(np.sum(alphas / np.asarray(g.spacings)))   # term.py:115
    bound = 1.0 / inv_bound if inv_bound > 0.0 else np.inf        # term.py:116-119
    ranges = tuple((float(lo[a]), float(hi[a])) for a in range(g.dim))
    return delta, bound, ranges, bool(nz)


def stage(kind: int, dt: float, y, y0, delta) -> np.ndarray:
    """integrator.py:93-103 combination (kind 1 Euler, 2 RK2 avg, 3 RK3 1/4, 4 RK3 1/3)."""
    y = _f64(y)
    out = np.empty_like(y)
    y0p = _ptr(_f64(y0)) if y0 is not None else None
    d = _f64(delta)
    y0a = _f64(y0) if y0 is not None else None
    lib().or_stage(y.size, kind, float(dt), _ptr(y), _ptr(y0a) if y0a is not None else None, _ptr(d), _ptr(out))
    return out


def shape(g, kind: int, params) -> np.ndarray:
    out = np.empty(tuple(g.counts))
    prm = _f64(params)
    G = _G(g)
    lib().or_shape(G.ref, kind, _ptr(prm), _ptr(out))
    return out


# ---------------------------------------------------------------- host loops
def integrate(g, ham: Ham, scheme: str, order: int, tspan, y0, cfl: float = 0.5, max_step=None,
              single_step: bool = False, mask_prev=None, mask_min: bool = True):
    """_integrate (integrator.py:69-126) over the oracle term; optional tube
    mask applied to the final state (reachability.py:249).
    Returns (t_final, y_final, steps, min_dt, max_dt)."""
    t0, t1 = float(tspan[0]), float(tspan[1])
    if t1 < t0:
        raise ValueError(f"tspan must be increasing, got [{t0}, {t1}]")
    t = t0
    y = _f64(y0).reshape(tuple(g.counts)).copy()
    steps = 0
    min_dt, max_dt = np.inf, 0.0
    while t < t1:
        d1, bound, _, _ = term(g, ham, scheme, y)
        dt = cfl * bound
        if max_step is not None:
            dt = min(dt, max_step)
        remaining = t1 - t
        last = dt >= remaining
        if last:
            dt = remaining
        if not (dt > 0.0 and np.isfinite(dt)):
            raise RuntimeError(f"step {steps}: no usable step size (dt={dt})")
        if order == 1:
            y_next = stage(1, dt, y, None, d1)
        elif order == 2:
            y1 = stage(1, dt, y, None, d1)
            d2 = term(g, ham, scheme, y1)[0]
            y_next = stage(2, dt, y1, y, d2)
        else:
            y1 = stage(1, dt, y, None, d1)
            d2 = term(g, ham, scheme, y1)[0]
            yh = stage(3, dt, y1, y, d2)
            d3 = term(g, ham, scheme, yh)[0]
            y_next = stage(4, dt, yh, y, d3)
        y = y_next.reshape(y.shape)
        t = t1 if last else t + dt
        steps += 1
        min_dt = min(min_dt, dt)
        max_dt = max(max_dt, dt)
        if single_step:
            break
    if steps == 0:
        min_dt = 0.0
    if mask_prev is not None:
        prev = _f64(mask_prev)
        lib().or_mask(y.size, _ptr(prev), _ptr(y), 1 if mask_min else 0)
    return t, y, steps, min_dt, max_dt


def solve_brt(g, ham: Ham, scheme: str, target, horizon: float, global_steps: int, order: int = 3,
              cfl: float = 0.5, max_step=None, over: bool = True):
    """solve_brt (reachability.py:218-254) generalised to any dim / RK order.
    Returns (snapshots, times, steps_per_interval)."""
    target = _f64(target).reshape(tuple(g.counts))
    if horizon == 0:
        return [target], [0.0], []
    snaps, times, steps = [target], [0.0], []
    v = target
    for k in range(1, global_steps + 1):
        t0 = times[-1]
        t1 = horizon * k / global_steps
        _, y, n, _, _ = integrate(g, ham, scheme, order, (t0, t1), v, cfl, max_step, mask_prev=snaps[-1],
                                  mask_min=over)
        v = y
        snaps.append(v)
        times.append(t1)
        steps.append(n)
    return snaps, times, steps
