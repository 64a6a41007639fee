"""Lax-Friedrichs right-hand side -- drop-in for hjls.term.

The evaluator contracts are the reference's (term.py:8-16):

    hamiltonian(t, grid, v, p_avg)      -> ScalarField (or array) of H(x, p)
    partials(t, grid, v, ranges, axis)  -> float bound on max |dH/dp_axis|

Two execution routes, both on the GPU:

* **registered device Hamiltonians** (:class:`DeviceHamiltonian`, built by
  :func:`advection_term_config`, ``rockets_term_config``, ``air3d_term_config``,
  ``di4_term_config``): the whole term -- ghosts, upwind derivatives, p_avg,
  H, GLF dissipation, delta -- is one fused sm_100a kernel (hj_term / hj_stage);
* **any other Python Hamiltonian** (the reference tests' lambdas): the
  derivatives, costate averages and ranges, dissipation and delta run in CUDA
  kernels, and only the user's own ``hamiltonian`` / ``partials`` callables run
  on the host between them (the host-Hamiltonian bridge).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _lib
from . import device as dev
from .grid import Grid, ScalarField
from .spatial import SCHEME_WIDTH, DerivativePair

Hamiltonian = Callable[[float, Grid, ScalarField, Sequence[ScalarField]], ScalarField]
Partials = Callable[[float, Grid, ScalarField, Sequence[tuple[float, float]], int], float]


# ---------------------------------------------------------------- registered device Hamiltonians
class DeviceHamiltonian:
    """A Hamiltonian with a device functor (hj_ham.cuh).  Calling it keeps the
    reference contract: H on the given costates, evaluated on the GPU."""

    kind: int = -1
    dim: int | None = None

    def params(self) -> tuple:
        raise NotImplementedError

    def tables(self, g: Grid) -> tuple:
        return ()

    def device(self, g: Grid) -> dev.DeviceHam:
        cache = self.__dict__.setdefault("_dev_cache", {})
        key = id(g)
        hit = cache.get(key)
        if hit is None or hit[0] is not g:
            hit = (g, dev.DeviceHam(self.kind, self.params(), self.tables(g)))
            cache[key] = hit
        return hit[1]

    def check_grid(self, g: Grid) -> None:
        if self.dim is not None and g.dim != self.dim:
            raise ValueError(f"expected {self.dim} costate fields, got {g.dim}")

    def __call__(self, t: float, g: Grid, v, p: Sequence[ScalarField]) -> ScalarField:
        if self.dim is not None and len(p) != self.dim:
            raise ValueError(f"expected {self.dim} costate fields, got {len(p)}")
        dg = dev.device_grid(g)
        out = dev.eval_hamiltonian_dev(dg, self.device(g), [dev.to_dev(x.values) for x in p])
        return ScalarField(dev.to_host(out))


class RangeFreePartials:
    """Dissipation bounds that ignore the costate ranges, so the fused solve
    needs no device->host round trip per stage."""

    def alphas(self, t: float, g: Grid) -> np.ndarray:
        raise NotImplementedError

    def __call__(self, t: float, g: Grid, v, ranges, axis: int) -> float:
        return float(self.alphas(t, g)[axis])


class AdvectionHamiltonian(DeviceHamiltonian):
    """H = sum_i c_i p_i accumulated from zero (term.py:136-140)."""

    kind = _lib.HAM_ADVECTION

    def __init__(self, speeds):
        self.c = np.asarray(speeds, dtype=np.float64).ravel()

    def params(self):
        return tuple(self.c)

    def check_grid(self, g: Grid) -> None:
        if g.dim > self.c.size:
            raise ValueError(f"advection needs {g.dim} speeds, got {self.c.size}")

    def __call__(self, t, g, v, p):
        if len(p) > self.c.size:
            raise ValueError(f"advection needs {len(p)} speeds, got {self.c.size}")
        return super().__call__(t, g, v, p)


class AdvectionPartials(RangeFreePartials):
    """alpha_i = |c_i| (term.py:142-143)."""

    def __init__(self, speeds):
        self.c = np.asarray(speeds, dtype=np.float64).ravel()

    def alphas(self, t, g):
        return np.array([abs(float(self.c[a])) for a in range(g.dim)])


# ---------------------------------------------------------------- configuration / outputs
@dataclass(frozen=True)
class TermConfig:
    """Evaluators plus scheme choices for one Hamiltonian term (term.py:33-52)."""

    hamiltonian: Hamiltonian
    partials: Partials
    derivative_scheme: str = "eno2"
    dissipation: str = "glf"
    approximation_sign: str = "over"

    def __post_init__(self) -> None:
        if self.derivative_scheme not in SCHEME_WIDTH:
            raise ValueError(f"unknown derivative scheme {self.derivative_scheme!r}; "
                             f"pick from {sorted(SCHEME_WIDTH)}")
        if self.dissipation != "glf":
            raise ValueError(f"only 'glf' dissipation is available, got {self.dissipation!r}")
        if self.approximation_sign not in ("over", "under"):
            raise ValueError("approximation_sign must be 'over' or 'under'")

    @property
    def on_device(self) -> bool:
        """True when the whole term can run as the fused kernel."""
        return isinstance(self.hamiltonian, DeviceHamiltonian)


@dataclass(frozen=True)
class TermOutput:
    """dv/dt field plus the inverse-CFL step bound (term.py:55-60)."""

    delta: ScalarField
    step_bound: float


# ---------------------------------------------------------------- shared host scalar logic
def validated_alphas(partials, t, g, v, ranges) -> np.ndarray:
    """alpha_i = partials(...) checked finite and >= 0 (term.py:78-83)."""
    if isinstance(partials, RangeFreePartials):
        raw = [float(x) for x in partials.alphas(t, g)]
    else:
        raw = [float(partials(t, g, v, ranges, i)) for i in range(g.dim)]
    alphas = np.empty(g.dim)
    for i, a in enumerate(raw):
        if not np.isfinite(a) or a < 0.0:
            raise ValueError(f"partials returned invalid bound {a} for axis {i}")
        alphas[i] = a
    return alphas


def step_bound(alphas: np.ndarray, g: Grid) -> float:
    """1 / sum_i(alpha_i / dx_i), or inf when every alpha is zero (term.py:115-119)."""
    inv = float(np.sum(alphas / g.spacings))
    return 1.0 / inv if inv > 0.0 else np.inf


def warn_zero_dissipation() -> None:
    warnings.warn(
        "all dissipation coefficients are zero while H is nonzero; "
        "CFL step bound is undefined (reported as infinite)",
        stacklevel=3,
    )


def raise_for_flags(flags: int) -> None:
    """Map device non-finite flags to the reference's ValueErrors."""
    if flags & _lib.NF_INPUT or flags & _lib.NF_DERIV:
        raise ValueError("field contains non-finite values")
    if flags & _lib.NF_HAM:
        raise ValueError("hamiltonian returned non-finite values")
    if flags & (_lib.NF_DELTA | _lib.NF_OUTPUT):
        raise ValueError("field contains non-finite values")


def device_alphas(cfg: TermConfig, t: float, g: Grid, dg, v_dev, v_host=None) -> np.ndarray:
    """alphas for a fused evaluation.  Range-free partials need nothing from the
    device; any other partials get the stage's costate ranges from a ranges-
    only pass of the fused kernel first (two-pass GLF, term.py:71-83)."""
    if isinstance(cfg.partials, RangeFreePartials):
        return validated_alphas(cfg.partials, t, g, None, None)
    st = dev.Stats().reset()
    dev.term_dev(dg, cfg.derivative_scheme, cfg.hamiltonian.device(g), [0.0] * g.dim, v_dev, st)
    s = st.read()
    raise_for_flags(s.nonfinite & (_lib.NF_INPUT | _lib.NF_DERIV | _lib.NF_HAM))
    ranges = dev.Stats.ranges(s, g.dim)
    v = v_host if v_host is not None else ScalarField(dev.to_host(v_dev))
    return validated_alphas(cfg.partials, t, g, v, ranges)


# ---------------------------------------------------------------- public API
def dissipation_glf(derivs: Sequence[DerivativePair], partials: Partials, t: float, v: ScalarField,
                    g: Grid) -> tuple[ScalarField, np.ndarray]:
    """Global LF dissipation sum_i alpha_i (p_i+ - p_i-)/2 and alpha (term.py:63-87)."""
    dg = dev.device_grid(g)
    Ls = [dev.to_dev(d.left.values) for d in derivs]
    Rs = [dev.to_dev(d.right.values) for d in derivs]
    st = dev.Stats().reset()
    dev.costates_dev(dg, Ls, Rs, st)
    ranges = dev.Stats.ranges(st.read(), len(derivs))
    alphas = validated_alphas(partials, t, g, v, ranges)
    zero = dev.to_dev(np.zeros(v.grid_shape))
    _, diss = dev.glf_delta_dev(dg, alphas, Ls, Rs, zero, True, None)
    return ScalarField(dev.to_host(diss)), alphas


def term_lax_friedrichs(t: float, v: ScalarField, cfg: TermConfig, g: Grid) -> TermOutput:
    """delta = -(H(x, p_avg) - dissipation) and the CFL bound (term.py:90-126)."""
    if not v.matches(g):
        raise ValueError(f"field shape {v.grid_shape} does not match grid {g.counts}")
    if cfg.on_device:
        return _term_fused(t, v, cfg, g)
    return _term_bridge(t, v, cfg, g)


def _term_fused(t: float, v: ScalarField, cfg: TermConfig, g: Grid) -> TermOutput:
    cfg.hamiltonian.check_grid(g)
    dg = dev.device_grid(g)
    v_dev = dev.to_dev(v.values)
    alphas = device_alphas(cfg, t, g, dg, v_dev, v)
    st = dev.Stats().reset()
    delta = dev.term_dev(dg, cfg.derivative_scheme, cfg.hamiltonian.device(g), alphas, v_dev, st)
    s = st.read()
    raise_for_flags(s.nonfinite)
    bound = step_bound(alphas, g)
    if bound == np.inf and s.nonfinite & _lib.FLAG_HAM_NONZERO:
        warn_zero_dissipation()
    return TermOutput(delta=ScalarField._from_device(dev.to_host(delta)), step_bound=bound)


def _term_bridge(t: float, v: ScalarField, cfg: TermConfig, g: Grid) -> TermOutput:
    dg = dev.device_grid(g)
    v_dev = dev.to_dev(v.values)
    Ls, Rs = [], []
    for axis in range(g.dim):
        L, R = dev.derivs_dev(dg, v_dev, axis, cfg.derivative_scheme)
        Ls.append(L)
        Rs.append(R)
    st = dev.Stats().reset()
    P = dev.costates_dev(dg, Ls, Rs, st)
    s = st.read()
    raise_for_flags(s.nonfinite & _lib.NF_DERIV)
    p_avg = [ScalarField(dev.to_host(p)) for p in P]
    ham = cfg.hamiltonian(t, g, v, p_avg)
    ham_values = ham.values if isinstance(ham, ScalarField) else np.asarray(ham, dtype=np.float64)
    if ham_values.shape != v.grid_shape:
        raise ValueError(f"hamiltonian returned shape {ham_values.shape}, expected {v.grid_shape}")
    if not np.isfinite(ham_values).all():
        raise ValueError("hamiltonian returned non-finite values")
    alphas = validated_alphas(cfg.partials, t, g, v, dev.Stats.ranges(s, g.dim))
    st2 = dev.Stats().reset()
    delta, _ = dev.glf_delta_dev(dg, alphas, Ls, Rs, dev.to_dev(ham_values), False, st2)
    raise_for_flags(st2.read().nonfinite)
    bound = step_bound(alphas, g)
    if bound == np.inf and np.any(ham_values != 0.0):
        warn_zero_dissipation()
    return TermOutput(delta=ScalarField(dev.to_host(delta)), step_bound=bound)


def advection_term_config(speeds: Sequence[float], scheme: str = "first") -> TermConfig:
    """Constant-coefficient advection H = sum_i c_i p_i, alpha_i = |c_i| (term.py:129-145)."""
    return TermConfig(hamiltonian=AdvectionHamiltonian(speeds), partials=AdvectionPartials(speeds),
                      derivative_scheme=scheme)
