"""Two-rocket game and the backward reachable tube -- drop-in for hjls.reachability.

``solve_brt`` keeps the reference's semantics (reachability.py:218-254): per
interval, integrate the Lax-Friedrichs term with TVD-RK3, then mask against
the previous snapshot (min for "over", max for "under").  With a registered
device Hamiltonian the tube lives in HBM for the whole solve; every RK stage
is one fused kernel and the mask is fused into the interval's last stage.
Snapshots are copied to the host once per interval (they are the result),
on a side stream that overlaps the next interval's compute (SnapshotPipe).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev
from .grid import Grid, ScalarField
from .integrator import IntegrationResult, IntegratorOptions, LaxFriedrichsRHS, ode_cfl_3
from .term import DeviceHamiltonian, RangeFreePartials, TermConfig


@dataclass(frozen=True)
class RocketParams:
    """Shared rocket constants, feet/second (reachability.py:33-47)."""

    a: float = 1.0
    grav: float = 32.0
    capture_radius: float = 1.5
    u_min: float = -1.0
    u_max: float = 1.0

    def __post_init__(self) -> None:
        if self.a <= 0 or self.grav <= 0 or self.capture_radius <= 0:
            raise ValueError("a, grav and capture_radius must be positive")
        if not self.u_min < self.u_max:
            raise ValueError(f"need u_min < u_max, got [{self.u_min}, {self.u_max}]")


def _theta_tables(g: Grid):
    # reachability.py:60-61: cos/sin of the heading nodes taken on the host with
    # the reference's own NumPy expression, so the device sees the same bits
    theta = g.axis_nodes[2].reshape(1, 1, -1)
    return np.cos(theta).ravel(), np.sin(theta).ravel()


class RocketsHamiltonian(DeviceHamiltonian):
    """Device functor for the published closed form (reachability.py:61-81) or
    the extremal-control form (reachability.py:84-116)."""

    dim = 3

    def __init__(self, params: RocketParams, route: str = "published"):
        if route not in ("published", "extremal"):
            raise ValueError(f"hamiltonian must be 'published' or 'extremal', got {route!r}")
        self.rp = params
        self.route = route
        self.kind = _lib.HAM_ROCKETS if route == "published" else _lib.HAM_ROCKETS_EXTREMAL

    def params(self):
        return (self.rp.a, self.rp.grav, self.rp.u_min, self.rp.u_max)

    def tables(self, g):
        return _theta_tables(g)

    def check_grid(self, g):
        if g.dim != 3:
            raise ValueError(f"expected 3 costate fields, got {g.dim}")


class RocketsPartials(RangeFreePartials):
    """rockets_partials as a range-free bound (reachability.py:139-157)."""

    def __init__(self, params: RocketParams):
        self.rp = params

    def alphas(self, t, g):
        return np.array([rockets_partials(t, g, None, None, a, self.rp) for a in range(3)])


def rockets_hamiltonian(t: float, g: Grid, v, p: Sequence[ScalarField], params: RocketParams) -> ScalarField:
    """H = -a p1 cos(th) - p2 (grav - a - a sin(th)) - u_max|p1 x + p3| + u_min|p2 x + p3|."""
    if len(p) != 3:
        raise ValueError(f"expected 3 costate fields, got {len(p)}")
    return RocketsHamiltonian(params, "published")(t, g, v, p)


def rockets_hamiltonian_extremal(t: float, g: Grid, v, p: Sequence[ScalarField],
                                 params: RocketParams) -> ScalarField:
    """Extremal-control Hamiltonian (reachability.py:84-116)."""
    if len(p) != 3:
        raise ValueError(f"expected 3 costate fields, got {len(p)}")
    return RocketsHamiltonian(params, "extremal")(t, g, v, p)


def rockets_hamiltonian_oracle(t: float, state: Sequence[float], p: Sequence[float],
                               params: RocketParams) -> float:
    """-max_{u_e} min_{u_p} p . f over the four control corners (reachability.py:119-136).

    A scalar test oracle of the reference, kept as plain host arithmetic (it
    is not part of the grid-update path)."""
    x, _, theta = (float(s) for s in state)
    p1, p2, p3 = (float(c) for c in p)
    a, g = params.a, params.grav
    best_e = -np.inf
    for u_e in (params.u_min, params.u_max):
        best_p = np.inf
        for u_p in (params.u_min, params.u_max):
            fx = a * np.cos(theta) + u_e * x
            fz = a * np.sin(theta) + a + u_p * x - g
            ft = u_p - u_e
            best_p = min(best_p, p1 * fx + p2 * fz + p3 * ft)
        best_e = max(best_e, best_p)
    return -best_e


def rockets_partials(t: float, g: Grid, v, ranges, axis: int, params: RocketParams) -> float:
    """Global |dH/dp_axis| bounds, independent of the ranges (reachability.py:139-157)."""
    a, grav = params.a, params.grav
    x_max = float(max(abs(g.mins[0]), abs(g.maxs[0])))
    if axis == 0:
        return a + abs(params.u_max) * x_max
    if axis == 1:
        return max(abs(grav), abs(grav - 2.0 * a)) + abs(params.u_min) * x_max
    if axis == 2:
        return abs(params.u_max) + abs(params.u_min)
    raise ValueError(f"axis {axis} out of range for the 3-state rockets game")


def rockets_term_config(params: RocketParams, scheme: str = "eno2", hamiltonian: str = "published") -> TermConfig:
    """Bundle a rockets Hamiltonian route with its bounds (reachability.py:160-183)."""
    if hamiltonian not in ("published", "extremal"):
        raise ValueError(f"hamiltonian must be 'published' or 'extremal', got {hamiltonian!r}")
    return TermConfig(hamiltonian=RocketsHamiltonian(params, hamiltonian), partials=RocketsPartials(params),
                      derivative_scheme=scheme)


@dataclass(frozen=True)
class ReachProblem:
    """Grid, target level function, term wiring, horizon (reachability.py:186-207)."""

    grid: Grid
    target: ScalarField
    params: RocketParams
    term_config: TermConfig
    horizon: float
    global_steps: int

    def __post_init__(self) -> None:
        if self.grid.dim != 3:
            raise ValueError(f"rockets game needs a 3-D grid, got dim {self.grid.dim}")
        if not self.grid.is_periodic(2):
            raise ValueError("the heading axis (axis 2) must be periodic")
        if not self.target.matches(self.grid):
            raise ValueError("target field does not match the grid")
        if self.horizon < 0:
            raise ValueError(f"horizon must be nonnegative, got {self.horizon}")
        if self.global_steps < 1:
            raise ValueError(f"need at least one global step, got {self.global_steps}")


@dataclass(frozen=True)
class BRTResult:
    """Tube snapshots, the first at lookback time 0 (reachability.py:210-215)."""

    snapshots: tuple[ScalarField, ...]
    times: tuple[float, ...]


class SnapshotPipe:
    """Overlaps each interval's snapshot copy with the next interval's compute.

    ``push`` records an event after the interval's kernels and hands the
    device->host copy to a worker thread, which waits for the event on a side
    stream and copies into a fresh host array (pageable: a snapshot is a
    retained result, and pinning fresh memory per snapshot costs more than
    the copy -- scripts/d2h_probe.py); the main thread meanwhile launches the
    next interval.  Then it completes the PREVIOUS interval: waits for its
    copy and calls ``deliver(k, t, array)``.  Snapshots are delivered in
    order, at most one interval behind the solve.  Small fields (C1's
    0.75 MB) go through pinned staging on the side stream instead.
    """

    def __init__(self, deliver):
        from concurrent.futures import ThreadPoolExecutor

        self.deliver = deliver
        self.copy = torch.cuda.Stream()
        self.pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="hj-snapshot")
        self.pending = None

    def _fetch(self, state: torch.Tensor, ready) -> np.ndarray:
        with torch.cuda.device(state.device), torch.cuda.stream(self.copy):
            self.copy.wait_event(ready)
            out = np.empty(tuple(state.shape), dtype=np.float64)
            torch.from_numpy(out).copy_(state)   # returns once the bytes are on the host
        return out

    SMALL = 4 << 20   # below this, pinned staging is cheap and a thread hand-off is not

    def push(self, k, t, state: torch.Tensor) -> None:
        if state.numel() * state.element_size() < self.SMALL:
            host = dev.host_empty(state.shape, state.dtype)
            self.copy.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.copy):
                host.copy_(state, non_blocking=True)
                done = torch.cuda.Event()
                done.record(self.copy)
            state.record_stream(self.copy)

            def result():
                done.synchronize()
                return host.numpy()
        else:
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream())
            result = self.pool.submit(self._fetch, state, ready).result
        self.drain()
        self.pending = (k, t, result)

    def drain(self) -> None:
        if self.pending is None:
            return
        k, t, result = self.pending
        self.pending = None
        self.deliver(k, t, result())

    def close(self) -> None:
        self.pool.shutdown(wait=True)


def solve_tube(g: Grid, target: ScalarField, cfg: TermConfig, horizon: float, global_steps: int, order: int = 3,
               opts: IntegratorOptions | None = None,
               progress: Callable[[int, float, ScalarField], None] | None = None,
               diagnostics: list | None = None, keep_snapshots: bool = True) -> BRTResult:
    """The tube driver of solve_brt for any dimension and RK order.

    ReachProblem insists on the 3-D rockets layout and solve_brt hard-wires
    RK3 (reachability.py:198-199, 246); this is the same loop with those two
    choices opened up (Air3D C1 runs RK2, the 4-D pair runs on 4 axes).

    ``diagnostics`` (a list, registered device Hamiltonians): the tube's
    acceptance checks (test_reachability.py:218-285) evaluated on the GPU per
    interval (hj_tube_check) and appended as dicts -- nesting and target
    containment violations, sublevel count and volume, nodes captured in the
    interval -- with no field copied to the host for them.
    ``keep_snapshots=False`` skips the per-interval snapshot copies: the
    result then holds the target and the final field only (times likewise).
    """
    if horizon == 0:
        return BRTResult(snapshots=(target,), times=(0.0,))
    if not keep_snapshots and (progress is not None or not cfg.on_device):
        raise ValueError("keep_snapshots=False needs a registered device Hamiltonian and no progress callback")
    opts = opts or IntegratorOptions()
    use_min = cfg.approximation_sign == "over"
    snaps = [target]
    times = [0.0]
    if cfg.on_device:
        from .engine import FusedIntegrator

        fi = FusedIntegrator(g, cfg)
        prev = dev.to_dev(target.values)
        target_dev = prev
        counters = (torch.zeros((global_steps, 4), dtype=torch.int64, device=prev.device)
                    if diagnostics is not None else None)

        def deliver(k, t, values):
            v = ScalarField._from_device(values)   # finiteness checked on the device
            snaps.append(v)
            times.append(t)
            if progress is not None:
                progress(k, t, v)

        pipe = SnapshotPipe(deliver)
        t0 = 0.0
        try:
            for k in range(1, global_steps + 1):
                t1 = horizon * k / global_steps
                try:
                    res = fi.integrate(order, (t0, t1), prev, opts, mask_prev=prev, use_min=use_min)
                except Exception as err:
                    pipe.drain()   # callbacks of the intervals that did finish
                    raise RuntimeError(f"tube interval {k} failed: {err}") from err
                if counters is not None:
                    dev.tube_check_dev(prev, res.y, target_dev, use_min, 0.0, counters[k - 1])
                prev = res.y
                # interval k's snapshot streams to the host while interval k+1
                # computes; interval k-1's is handed out meanwhile
                if keep_snapshots:
                    pipe.push(k, t1, prev)
                t0 = t1
            pipe.drain()
        finally:
            pipe.close()
        if counters is not None:
            cell = float(np.prod(g.spacings))
            for k, row in enumerate(counters.cpu().tolist(), start=1):
                diagnostics.append({"interval": k, "t": horizon * k / global_steps, "nesting_violations": row[0],
                                    "containment_violations": row[1], "sublevel_nodes": row[2],
                                    "volume": cell * row[2], "captured": row[3]})
        if not keep_snapshots:
            final = ScalarField._from_device(dev.to_host(prev))
            return BRTResult(snapshots=(target, final), times=(0.0, float(t0)))
        return BRTResult(snapshots=tuple(snaps), times=tuple(times))

    from .integrator import ode_cfl_1, ode_cfl_2

    integ = {1: ode_cfl_1, 2: ode_cfl_2, 3: ode_cfl_3}[order]
    rhs = LaxFriedrichsRHS(g)
    v = target
    for k in range(1, global_steps + 1):
        t0 = times[-1]
        t1 = horizon * k / global_steps
        try:
            res: IntegrationResult = integ(rhs, (t0, t1), v, opts, cfg)
        except Exception as err:
            raise RuntimeError(f"tube interval {k} failed: {err}") from err
        y = dev.to_dev(res.y_final.values)
        dev.mask_dev(y, dev.to_dev(snaps[-1].values), use_min)
        v = ScalarField(dev.to_host(y))
        snaps.append(v)
        times.append(t1)
        if progress is not None:
            progress(k, t1, v)
    return BRTResult(snapshots=tuple(snaps), times=tuple(times))


_BATCH: "weakref.WeakKeyDictionary" = None


def _batch_runner(g: Grid, cfg: TermConfig, batch: int):
    """(FusedIntegrator over the stacked batch, pinned staging, copy pool) of
    (grid, cfg, batch, device), reused across solve_tube_batch calls."""
    global _BATCH
    import weakref
    from concurrent.futures import ThreadPoolExecutor

    from .engine import FusedIntegrator

    if _BATCH is None:
        _BATCH = weakref.WeakKeyDictionary()
    per = _BATCH.setdefault(g, {})
    key = (id(cfg), batch, torch.cuda.current_device())
    hit = per.get(key)
    if hit is None or hit[0] is not cfg:
        fi = FusedIntegrator(g, cfg, dg=dev.DeviceGrid(g, batch=batch))
        staging = dev.host_empty((batch,) + tuple(g.counts), dev.F64)
        hit = (cfg, fi, staging, ThreadPoolExecutor(max_workers=8, thread_name_prefix="hj-batch"))
        per.clear()   # one batch shape per grid is kept
        per[key] = hit
    return hit[1], hit[2], hit[3]


def _stream_runner(g: Grid, cfg: TermConfig, batch: int):
    """(one FusedIntegrator per problem, one stream per problem, per-problem
    device inputs) of (grid, cfg, batch, device), reused across calls."""
    from .engine import FusedIntegrator

    fi, staging, pool = _batch_runner(g, cfg, batch)   # (the pinned staging and copy pool)
    key = ("streams", id(cfg), batch, torch.cuda.current_device())
    per = _BATCH.setdefault(g, {})
    hit = per.get(key)
    if hit is None or hit[0] is not cfg:
        fis = [FusedIntegrator(g, cfg) for _ in range(batch)]
        streams = [torch.cuda.Stream() for _ in range(batch)]
        ins = [torch.empty(tuple(g.counts), dtype=dev.F64, device=dev.device()) for _ in range(batch)]
        hit = (cfg, fis, streams, ins)
        per[key] = hit
    return hit[1], hit[2], hit[3], staging, pool


def _solve_batch_streamed(g: Grid, arrs, cfg: TermConfig, horizon: float, order: int, opts, use_min: bool):
    """One interval of every problem of the batch, final states only: problem b
    runs on its own stream -- host copy into pinned staging, H2D, the native
    integration (mask fused in the last stage), D2H -- so the copies of one
    problem overlap the stages of the others (the lockstep batch waits for
    the whole batch's input before its first stage and for its last stage
    before any output).  Errors are read from each problem's device flags
    after all streams finish: the reference's non-finite-input ValueError,
    or the interval's RuntimeError."""
    B = len(arrs)
    fis, streams, ins, staging, pool = _stream_runner(g, cfg, B)
    st = staging.numpy()
    # host copies into pinned staging problem by problem, each split across the
    # pool's threads, so problem 0's DMA can start after 1/B of the copying
    n0 = st.shape[1]
    parts = min(8, n0)
    bounds = [n0 * k // parts for k in range(parts + 1)]
    futs = [[pool.submit(np.copyto, st[b, bounds[k]:bounds[k + 1]], a[bounds[k]:bounds[k + 1]])
             for k in range(parts)] for b, a in enumerate(arrs)]
    out = dev.host_empty((B,) + tuple(g.counts), dev.F64)
    main = torch.cuda.current_stream()
    for b in range(B):
        s = streams[b]
        s.wait_stream(main)
        for f in futs[b]:
            f.result()
        with torch.cuda.stream(s):
            ins[b].copy_(staging[b], non_blocking=True)
            try:
                res = fis[b].integrate(order, (0.0, horizon), ins[b], opts, mask_prev=ins[b], use_min=use_min,
                                       check=False)
            except Exception as err:
                raise RuntimeError(f"tube interval 1 failed: {err}") from err
            out[b].copy_(res.y, non_blocking=True)
            res.y.record_stream(s)
    for s in streams:
        main.wait_stream(s)
    main.synchronize()
    for b in range(B):
        try:
            fis[b].raise_pending(order, 0.0, horizon, ins[b], opts)
        except ValueError as err:
            if str(err) == "field contains non-finite values":
                raise
            raise RuntimeError(f"tube interval 1 failed: {err}") from err
        except Exception as err:
            raise RuntimeError(f"tube interval 1 failed: {err}") from err
    return out.numpy()


def solve_tube_batch(g: Grid, targets, cfg: TermConfig, horizon: float, global_steps: int, order: int = 3,
                     opts: IntegratorOptions | None = None, keep_snapshots: bool = True):
    """A batch of independent tubes sharing grid and dynamics (BASELINE C5:
    the flock of Air3D problems).  Dissipation bounds and dt depend on the
    grid and Hamiltonian only, so the batch advances in lockstep: every stage
    of every problem is one kernel launch over the stacked (B, n0, ...)
    state.  Returns (snapshots (global_steps+1, B, *counts) | final (B, ...),
    times)."""
    if not cfg.on_device:
        raise TypeError("solve_tube_batch needs a registered device Hamiltonian")
    arrs = [np.asarray(t.values if isinstance(t, ScalarField) else t, dtype=np.float64) for t in targets]
    for a in arrs:
        if a.shape != tuple(g.counts):
            raise ValueError(f"targets have shape {a.shape}, grid needs {g.counts}")
    opts = opts or IntegratorOptions()
    if not keep_snapshots and global_steps == 1 and len(arrs) > 1 and horizon > 0.0:
        # final states of one interval: per-problem streams overlap the copies with the stages
        return _solve_batch_streamed(g, arrs, cfg, float(horizon), order, opts,
                                     cfg.approximation_sign == "over"), (0.0, horizon)
    fi, staging, pool = _batch_runner(g, cfg, len(arrs))
    # the targets go to pinned staging on host threads (NumPy copies release
    # the GIL), then one DMA; finiteness is checked on the device
    st = staging.numpy()
    for f in [pool.submit(np.copyto, st[b], a) for b, a in enumerate(arrs)]:
        f.result()
    prev = torch.empty(staging.shape, dtype=dev.F64, device=dev.device())
    prev.copy_(staging, non_blocking=True)
    if not bool(torch.isfinite(prev).all()):
        raise ValueError("field contains non-finite values")
    tgt = st.copy() if keep_snapshots else None
    snaps = [tgt] if keep_snapshots else []
    times = [0.0]
    use_min = cfg.approximation_sign == "over"
    pipe = SnapshotPipe(lambda k, t, values: snaps.append(values)) if keep_snapshots else None
    try:
        for k in range(1, global_steps + 1):
            t0, t1 = times[-1], horizon * k / global_steps
            try:
                res = fi.integrate(order, (t0, t1), prev, opts, mask_prev=prev, use_min=use_min)
            except Exception as err:
                raise RuntimeError(f"tube interval {k} failed: {err}") from err
            prev = res.y
            if pipe is not None:
                pipe.push(k, t1, prev)
            times.append(t1)
        if pipe is not None:
            pipe.drain()
    finally:
        if pipe is not None:
            pipe.close()
    return (np.stack(snaps) if keep_snapshots else dev.to_host(prev)), tuple(times)


def solve_brt(problem: ReachProblem, opts: IntegratorOptions | None = None,
              progress: Callable[[int, float, ScalarField], None] | None = None) -> BRTResult:
    """Grow the backward reachable tube over ``global_steps`` equal intervals
    with TVD-RK3 and per-interval masking (reachability.py:218-254)."""
    return solve_tube(problem.grid, problem.target, problem.term_config, problem.horizon, problem.global_steps,
                      order=3, opts=opts, progress=progress)


def sublevel_volume(g: Grid, f: ScalarField, level: float = 0.0) -> float:
    """Volume of {f < level}, one cell per node (reachability.py:257-260); the
    count runs on the GPU."""
    cell = float(np.prod(g.spacings))
    return cell * float(dev.count_below_dev(dev.to_dev(f.values), level))


__all__ = [
    "BRTResult", "ReachProblem", "RocketParams", "RocketsHamiltonian", "RocketsPartials", "rockets_hamiltonian",
    "rockets_hamiltonian_extremal", "rockets_hamiltonian_oracle", "rockets_partials", "rockets_term_config",
    "solve_brt", "solve_tube", "sublevel_volume",
]

_ = math
