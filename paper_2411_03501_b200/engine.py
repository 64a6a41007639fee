"""The device-resident integration loop (the hot path's runtime).

Host side: the scalar logic of the reference integrator, byte-for-byte
(_integrate, integrator.py:69-126: dt = cfl*bound, min(max_step), clip to the
remaining span, t = t1 on the last step).  Device side: one fused sm_100a
kernel per TVD-RK stage (hj_stage), state ping-ponging between three HBM
buffers, the tube mask fused into the final stage of an interval.

Because registered dissipation bounds are range-free, the whole stage
schedule is known on the host in advance: nothing waits on the device
inside an interval.  Non-finite values are flagged on the device per stage
(hj_stats.first_bad_tag) and turned into the reference's exceptions once,
when the interval completes.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dev
from .term import RangeFreePartials, TermConfig, device_alphas, raise_for_flags, step_bound, warn_zero_dissipation

_STAGES = {
    1: (_lib.STAGE_EULER,),
    2: (_lib.STAGE_EULER, _lib.STAGE_RK2_AVG),
    3: (_lib.STAGE_EULER, _lib.STAGE_RK3_QUARTER, _lib.STAGE_RK3_THIRD),
}


@dataclass
class DeviceIntegration:
    t_final: float
    y: torch.Tensor
    steps_taken: int
    min_dt: float
    max_dt: float


class FusedIntegrator:
    """Integrates v_t + H(x, grad v) = 0 with a registered device Hamiltonian.

    ``dg`` may be a batched or slab DeviceGrid; ``exchange`` (multi-GPU) is
    called on every stage input before the stage kernel runs.
    """

    def __init__(self, g, cfg: TermConfig, dg: dev.DeviceGrid | None = None, exchange=None):
        if not cfg.on_device:
            raise TypeError("FusedIntegrator needs a TermConfig with a registered device Hamiltonian")
        cfg.hamiltonian.check_grid(g)
        self.lib = dev.require()
        self.g = g
        self.cfg = cfg
        self.dg = dg or dev.device_grid(g)
        self.dh = cfg.hamiltonian.device(g)
        self.scheme = cfg.derivative_scheme
        self.range_free = isinstance(cfg.partials, RangeFreePartials)
        self.exchange = exchange
        self.stats = dev.Stats()
        self._bufs: list[torch.Tensor] = []
        self._alpha_cache = None
        self.launches = 0

    # ------------------------------------------------------------ helpers
    def _alphas(self, t: float, y: torch.Tensor) -> np.ndarray:
        if self.range_free:
            if self._alpha_cache is None:
                self._alpha_cache = device_alphas(self.cfg, t, self.g, self.dg, None)
            return self._alpha_cache
        return device_alphas(self.cfg, t, self.g, self.dg, y)

    def _alphas_at(self, t: float, y: torch.Tensor | None, step: int) -> np.ndarray:
        """_alphas inside the term evaluation of ``step``: an invalid bound (or a
        non-finite range pass) surfaces as the reference's _rhs error
        (integrator.py:59-63: RuntimeError 'term evaluation failed at step k')."""
        try:
            return self._alphas(t, y)
        except ValueError as err:
            raise RuntimeError(f"term evaluation failed at step {step} (t={t:g}): {err}") from err

    def _buffers(self, like: torch.Tensor) -> list[torch.Tensor]:
        if not self._bufs or self._bufs[0].shape != like.shape:
            self._bufs = [torch.empty_like(like) for _ in range(3)]
        return self._bufs

    def _stage(self, alphas_c, dt, kind, y_in, y0, y_out, mask_prev, mask, tag, strm):
        if self.exchange is not None:
            self.exchange(y_in)
        dev.stage_dev(self.dg, self.scheme, self.dh, alphas_c, dt, kind, y_in, y0, y_out, mask_prev, mask,
                      self.stats, tag, lib=self.lib, strm=strm)
        self.launches += 1

    # ------------------------------------------------------------ the loop
    def integrate(self, order: int, tspan, y: torch.Tensor, opts, mask_prev: torch.Tensor | None = None,
                  use_min: bool = True, check: bool = True) -> DeviceIntegration:
        """_integrate (integrator.py:69-126) on device state ``y`` (left intact)."""
        t0, t1 = float(tspan[0]), float(tspan[1])
        if t1 < t0:
            raise ValueError(f"tspan must be increasing, got [{t0}, {t1}]")
        kinds = _STAGES[order]
        mask = (_lib.MASK_MIN if use_min else _lib.MASK_MAX) if mask_prev is not None else _lib.MASK_NONE
        if self._native_ok(opts):
            return self._integrate_native(order, t0, t1, y, opts, mask_prev, mask, use_min, check)
        strm = dev.stream()
        self.stats.reset()
        bufs = self._buffers(y)
        times: dict[int, float] = {}
        t, cur, steps = t0, y, 0
        min_dt, max_dt = np.inf, 0.0
        zero_alpha = False
        while t < t1:
            alphas = self._alphas_at(t, cur, steps)
            bound = step_bound(alphas, self.g)
            zero_alpha = zero_alpha or bound == np.inf
            dt = opts.cfl_factor * bound
            if opts.max_step is not None:
                dt = min(dt, opts.max_step)
            remaining = t1 - t
            last = dt >= remaining
            if last:
                dt = remaining
            if not (dt > 0.0 and np.isfinite(dt)):
                if check:
                    self._raise_pending(times)
                raise RuntimeError(f"step {steps}: no usable step size (dt={dt})")
            t_next = t1 if last else t + dt
            final = last or opts.single_step or not (t_next < t1)
            alphas_c = _lib.doubles(alphas, _lib.HJ_MAX_DIM)
            outs = [b for b in bufs if b is not cur][:2]
            stage_t = (t, t + dt, t + 0.5 * dt)
            src, dst = cur, outs[0]
            for k, kind in enumerate(kinds):
                tag = steps * 4 + k
                times[tag] = stage_t[k] if order == 3 else (t, t + dt)[k]
                is_last = k == len(kinds) - 1
                if k > 0:
                    dst = outs[1] if src is outs[0] else outs[0]
                y0 = cur if kind != _lib.STAGE_EULER else None
                if k > 0 and not self.range_free:
                    # range-dependent partials: each stage's own costate ranges (term.py:71-83)
                    alphas_c = _lib.doubles(self._alphas_at(times[tag], src, steps), _lib.HJ_MAX_DIM)
                self._stage(alphas_c, dt, kind, src, y0, dst, mask_prev if (final and is_last) else None,
                            mask if (final and is_last) else _lib.MASK_NONE, tag, strm)
                src = dst
            # rotate so the three buffers keep their roles: new state = src
            cur = src
            t = t_next
            steps += 1
            min_dt = min(min_dt, dt)
            max_dt = max(max_dt, dt)
            if opts.collect_stats:
                print(f"step {steps}: t={t:.6g} dt={dt:.6g} min={cur.min().item():.6g} max={cur.max().item():.6g}",
                      file=sys.stderr)
            if opts.single_step:
                break
        if steps == 0:
            min_dt = 0.0
            cur = y.clone()
            if mask_prev is not None:
                dev.mask_dev(cur, mask_prev, use_min)
        elif cur is not y:
            # hand the caller a tensor that later calls will not overwrite
            cur = cur.clone()
        if check:
            self._raise_pending(times, warn=zero_alpha)
        return DeviceIntegration(t, cur, steps, min_dt, max_dt)

    # ------------------------------------------------------------ host -> host single step
    # A call that takes one step on a host field (ode_cfl_k(..., single_step) or a
    # span shorter than one CFL step) is copy-bound when run as H2D, stages,
    # D2H.  The pipeline cuts the field into axis-0 chunks: the H2D of chunk
    # k+1 (copy stream) overlaps the stages over the planes whose stencils are
    # complete (hj_stage_planes; stage s lags stage s-1 by the ghost width,
    # rounded to the kernels' 8-plane rows), and finished planes of the last
    # stage go back to pinned host memory on a third stream.  The node updates
    # are the same as one launch per stage, bit for bit.
    pipeline_min_cells = 1 << 22     # smaller fields: plain copies are cheap
    pipeline_chunk = 16              # planes per H2D chunk (multiple of 8; 16 measured best at 301^3, scripts/e2e_probe.py)
    pipeline_priority = True         # later RK stages on higher-priority streams (the D2H-feeding stage first)
    pipeline_first = 16              # planes of the first H2D chunk
    pipeline_drain = 16              # planes per stage launch once the whole input has arrived

    pipeline_ramp = 0                # row-sized H2D chunks after the first
    pipeline_tail = 0                # last planes delivered in row-sized H2D chunks

    def _plan(self, n0: int, stages: int):
        return pipeline_plan(n0, stages, int(self.pipeline_chunk), first=int(self.pipeline_first),
                             drain=int(self.pipeline_drain), ramp=int(self.pipeline_ramp),
                             tail=int(self.pipeline_tail))

    def _pipeline_ok(self, opts, y_host: np.ndarray) -> bool:
        # (a periodic first axis wraps the stencil of the first planes onto the
        # last ones, which arrive last: no pipeline)
        return (self._native_ok(opts) and self.dg.batch == 1 and y_host.size >= self.pipeline_min_cells
                and self.g.counts[0] >= 16 and not self.g.is_periodic(0))

    def integrate_host(self, order: int, tspan, y_host: np.ndarray, opts) -> tuple:
        """_integrate on a host field; returns (t_final, y_host_final, steps, min_dt, max_dt)."""
        t0, t1 = float(tspan[0]), float(tspan[1])
        one_step = False
        dt = 0.0
        if t1 > t0 and self._pipeline_ok(opts, y_host):
            bound = step_bound(self._alphas_at(t0, None, 0), self.g)
            dt = opts.cfl_factor * bound
            if opts.max_step is not None:
                dt = min(dt, opts.max_step)
            last = dt >= t1 - t0
            if last:
                dt = t1 - t0
            one_step = (opts.single_step or last) and dt > 0.0 and np.isfinite(dt)
        if not one_step:
            res = self.integrate(order, (t0, t1), dev.to_dev(y_host), opts)
            return res.t_final, dev.to_host(res.y), res.steps_taken, res.min_dt, res.max_dt
        t_next = t1 if dt >= t1 - t0 else t0 + dt
        y_out = self._pipelined_step(order, t0, dt, y_host)
        stage_t = (t0, t0 + dt, t0 + 0.5 * dt) if order == 3 else (t0, t0 + dt)
        self._raise_pending({k: stage_t[k] for k in range(order)}, warn=bound == np.inf)
        return t_next, y_out, 1, dt, dt

    def _pipelined_step(self, order: int, t0: float, dt: float, y_host: np.ndarray) -> np.ndarray:
        kinds = _STAGES[order]
        n0 = self.g.counts[0]
        shape = tuple(self.g.counts)
        prio = bool(self.pipeline_priority)
        if getattr(self, "_pipe", None) is None or self._pipe[0] != (shape, prio):
            mk = lambda: torch.empty(shape, dtype=dev.F64, device=dev.device())  # noqa: E731
            # stage k on priority -k: when launches of several stages are ready
            # the block scheduler serves the later stage first, so the last
            # stage (and its D2H) trails the input by as little as possible
            self._pipe = ((shape, prio), [mk() for _ in range(len(kinds) + 1)], torch.cuda.Stream(),
                          torch.cuda.Stream(), [torch.cuda.Stream(priority=-k if prio else 0)
                                                for k in range(len(kinds))])
        _, bufs, s_in, s_out, s_st = self._pipe
        y_dev = bufs[0]
        out_host = dev.host_empty(shape, dev.F64)
        src_host = torch.from_numpy(np.ascontiguousarray(y_host, dtype=np.float64))
        staged = None
        if not src_host.is_pinned():
            # a pageable input (a plain NumPy array, as a reference caller
            # passes it): host threads copy it chunk by chunk into pinned
            # staging memory, ahead of the DMA of the chunks before
            staged = self._stage_pageable(src_host)
            src_host = self._staging
        comp = torch.cuda.current_stream()
        alphas_c = _lib.doubles(self._alphas(t0, None), _lib.HJ_MAX_DIM)
        self.stats.reset()                           # on comp: ordered before every stage stream below
        for st in (s_in, s_out, *s_st):
            st.wait_stream(comp)                     # the buffers' previous users, and the reset
        # one stream per stage: a launch waits (events) for the latest launch of
        # the stage before it (or the latest input chunk), so launches of
        # different stages overlap and fill each other's partial last waves
        last_ev = [None] * (len(kinds) + 1)          # [0]: input chunks, [k+1]: stage k's latest launch
        for op, k, lo, hi in self._plan(n0, len(kinds)):
            if op == "h2d":
                if staged is not None:
                    for f in staged.pop(lo):
                        f.result()
                with torch.cuda.stream(s_in):
                    y_dev[lo:hi].copy_(src_host[lo:hi], non_blocking=True)
                    last_ev[0] = torch.cuda.Event()
                    last_ev[0].record(s_in)
            elif op == "stage":
                st = s_st[k]
                st.wait_event(last_ev[k])            # everything this launch reads has been produced
                kind = kinds[k]
                dev.stage_dev(self.dg, self.scheme, self.dh, alphas_c, dt, kind, bufs[k],
                              y_dev if kind != _lib.STAGE_EULER else None, bufs[k + 1], None, _lib.MASK_NONE,
                              self.stats, k, lib=self.lib, strm=st.cuda_stream, planes=(lo, hi))
                self.launches += 1
                last_ev[k + 1] = torch.cuda.Event()
                last_ev[k + 1].record(st)
            else:   # "d2h" of finished planes of the last stage
                s_out.wait_event(last_ev[-1])
                with torch.cuda.stream(s_out):
                    out_host[lo:hi].copy_(bufs[-1][lo:hi], non_blocking=True)
        s_out.synchronize()
        for st in (s_in, s_out, *s_st):
            comp.wait_stream(st)
        return out_host.numpy()

    staging_threads = 8          # host threads copying a pageable input into pinned memory

    def _stage_pageable(self, src: torch.Tensor) -> dict:
        """Queue the copies of ``src`` into the cached pinned staging buffer in
        the pipeline's H2D chunk order, split across host threads (NumPy copies
        release the GIL).  Returns {chunk start plane: [futures]}."""
        from concurrent.futures import ThreadPoolExecutor

        if getattr(self, "_staging", None) is None or self._staging.shape != src.shape:
            self._staging = dev.host_empty(src.shape, src.dtype)
        if getattr(self, "_stage_pool", None) is None:
            self._stage_pool = ThreadPoolExecutor(max_workers=int(self.staging_threads),
                                                  thread_name_prefix="hj-stage")
        dst, srcn = self._staging.numpy(), src.numpy()
        n0 = src.shape[0]
        out: dict[int, list] = {}
        for op, _, lo, hi in self._plan(n0, 1):
            if op != "h2d":
                continue
            step = max(1, -(-(hi - lo) // int(self.staging_threads)))
            out[lo] = [self._stage_pool.submit(np.copyto, dst[a:min(a + step, hi)], srcn[a:min(a + step, hi)])
                       for a in range(lo, hi, step)]
        return out

    # ------------------------------------------------------------ native loop
    def _native_ok(self, opts) -> bool:
        """hj_integrate runs the whole loop in C++ when nothing needs the host
        between stages: range-free bounds, no per-step stats printing, no
        halo exchange (multi-GPU slabs override _stage)."""
        return (self.range_free and not opts.collect_stats and self.exchange is None
                and type(self)._stage is FusedIntegrator._stage)

    def _integrate_native(self, order, t0, t1, y, opts, mask_prev, mask, use_min, check) -> DeviceIntegration:
        import ctypes

        alphas = self._alphas_at(t0, y, 0)
        bound = step_bound(alphas, self.g)
        bufs = self._buffers(y)
        info = (ctypes.c_double * 6)()
        yfin = ctypes.c_void_p()
        self.stats.reset()
        rc = self.lib.hj_integrate(self.dg.ref, _lib.SCHEME_CODES[self.scheme], self.dh.ref,
                                   _lib.doubles(alphas, _lib.HJ_MAX_DIM), int(order), t0, t1, float(opts.cfl_factor),
                                   float(opts.max_step) if opts.max_step is not None else -1.0,
                                   1 if opts.single_step else 0, float(bound), dev.ptr(y), dev.ptr(bufs[0]),
                                   dev.ptr(bufs[1]), dev.ptr(bufs[2]), dev.ptr(mask_prev), int(mask), self.stats.p,
                                   info, ctypes.byref(yfin), dev.stream())
        _lib.check(rc, "hj_integrate")
        t, steps, min_dt, max_dt = info[0], int(info[1]), info[2], info[3]
        self.launches += steps * len(_STAGES[order])
        if info[4]:
            if check:
                self._raise_pending(self._replay_times(order, t0, t1, bound, opts))
            raise RuntimeError(f"step {steps}: no usable step size (dt={info[5]})")
        if steps == 0:
            cur = y.clone()
            if mask_prev is not None:
                dev.mask_dev(cur, mask_prev, use_min)
        else:
            cur = next(b for b in bufs if b.data_ptr() == yfin.value).clone()
        if check:
            self._raise_pending(self._replay_times(order, t0, t1, bound, opts), warn=bound == np.inf)
        return DeviceIntegration(t, cur, steps, min_dt, max_dt)

    @staticmethod
    def _replay_times(order, t0, t1, bound, opts) -> dict[int, float]:
        """Stage start times per tag, from the same scalar dt logic (only read
        when an error has to be reported)."""

        class _Lazy(dict):
            def get(self, tag, default=None):
                t, steps = t0, 0
                while t < t1:
                    dt = opts.cfl_factor * bound
                    if opts.max_step is not None:
                        dt = min(dt, opts.max_step)
                    remaining = t1 - t
                    last = dt >= remaining
                    if last:
                        dt = remaining
                    if steps == tag // 4:
                        k = tag % 4
                        return (t, t + dt, t + 0.5 * dt)[k] if order == 3 else (t, t + dt)[min(k, 1)]
                    t = t1 if last else t + dt
                    steps += 1
                    if opts.single_step:
                        break
                return default

        return _Lazy()

    def step3(self, y: torch.Tensor, t: float, dt: float, events: list | None = None) -> torch.Tensor:
        """One TVD-RK3 step with a given dt on device state ``y`` (three fused
        stages, no host sync).  Used by the benchmark; ``events`` collects a
        (start, end) CUDA event pair per stage launch."""
        bufs = self._buffers(y)
        outs = [b for b in bufs if b is not y][:2]
        alphas_c = _lib.doubles(self._alphas(t, y), _lib.HJ_MAX_DIM)
        strm = dev.stream()
        src = y
        for k, (kind, dst) in enumerate(zip(_STAGES[3], (outs[0], outs[1], outs[0]))):
            if events is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            self._stage(alphas_c, dt, kind, src, y if k else None, dst, None, _lib.MASK_NONE, k, strm)
            if events is not None:
                e1.record()
                events.append((e0, e1))
            src = dst
        return src

    def _read_stats(self):
        return self.stats.read()

    def raise_pending(self, order: int, t0: float, t1: float, y: torch.Tensor, opts) -> None:
        """The error check integrate(check=True) does after a native run, for a
        caller that ran it with check=False on a stream of its own and has
        synchronised since (the device flags are still those of that run)."""
        bound = step_bound(self._alphas_at(t0, y, 0), self.g)
        self._raise_pending(self._replay_times(order, t0, t1, bound, opts), warn=bound == np.inf)

    def _raise_pending(self, times: dict[int, float], warn: bool = False) -> None:
        """Turn the device flags into the exception the reference raises first."""
        s = self._read_stats()
        if warn and s.nonfinite & _lib.FLAG_HAM_NONZERO:
            warn_zero_dissipation()
        if not s.nonfinite & _lib.NF_MASK:
            return
        key = int(s.first_bad_tag)
        tag, code = key >> 3, key & 7
        step = tag // 4
        t = times.get(tag, float("nan"))
        if code in (1, 5):
            # the reference's ScalarField(y) on a stage input / the final state
            raise ValueError("field contains non-finite values")
        try:
            raise_for_flags({2: _lib.NF_DERIV, 3: _lib.NF_HAM, 4: _lib.NF_DELTA}.get(code, _lib.NF_DELTA))
        except ValueError as err:
            # integrator.py:61-63
            raise RuntimeError(f"term evaluation failed at step {step} (t={t:g}): {err}") from err


def pipeline_plan(n0: int, stages: int, chunk: int, reach: int = 3, row: int = 8, first: int = 16,
                  drain: int = 16, ramp: int = 0, tail: int = 0) -> list[tuple[str, int, int, int]]:
    """Schedule of the pipelined host->host step over axis-0 planes [0, n0):
    ("h2d", -1, lo, hi) input chunks -- a first chunk of ``first`` planes,
    ``ramp`` chunks of ``row`` planes, ``chunk``-plane chunks, and the last
    ``tail`` planes again in ``row``-plane chunks (short chunks at both ends
    start the first output copy early and leave little work behind the last
    input copy) -- ("stage", k, lo, hi) launches of stage k over planes whose
    stencil inputs are complete -- ``reach`` planes behind the previous
    stage's front (or its end), rounded down to the kernels' ``row``-plane
    rows -- and ("d2h", -1, lo, hi) copies of the last stage's finished
    planes.  Once the whole input has arrived every stage advances by at most
    ``drain`` planes per round, so the final copies start early.  Pure host
    logic (tests/test_host_logic.py checks coverage and dependencies)."""
    chunk = max(row, (chunk // row) * row)
    drain = max(row, (drain // row) * row)
    first = max(1, min(first, n0))
    bounds = [first]
    for _ in range(ramp):
        if bounds[-1] < n0:
            bounds.append(min(n0, bounds[-1] + row))
    body_end = max(bounds[-1], n0 - max(0, tail))
    while bounds[-1] + chunk < body_end:
        bounds.append(bounds[-1] + chunk)
    while bounds[-1] < n0:
        bounds.append(min(n0, bounds[-1] + (row if bounds[-1] >= body_end else body_end - bounds[-1])))
    plan: list[tuple[str, int, int, int]] = []
    done = [0] * stages
    arrived, nxt = 0, 0
    while done[-1] < n0:
        if nxt < len(bounds):
            plan.append(("h2d", -1, arrived, bounds[nxt]))
            arrived = bounds[nxt]
            nxt += 1
        hi = arrived
        for k in range(stages):
            hi = n0 if hi == n0 else max(0, ((hi - reach) // row) * row)
            if arrived == n0:
                hi = min(hi, done[k] + drain)
            if hi > done[k]:
                plan.append(("stage", k, done[k], hi))
                if k == stages - 1:
                    plan.append(("d2h", -1, done[k], hi))
                done[k] = hi
            hi = done[k]
    return plan


def integrate_fused(g, cfg: TermConfig, order: int, tspan, y0_host: np.ndarray, opts) -> DeviceIntegration:
    fi = FusedIntegrator(g, cfg)
    return fi.integrate(order, tspan, dev.to_dev(y0_host), opts)
