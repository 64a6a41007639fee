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
            alphas = self._alphas(t, cur)
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
                    alphas_c = _lib.doubles(self._alphas(times[tag], src), _lib.HJ_MAX_DIM)
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

    # ------------------------------------------------------------ native loop
    def _native_ok(self, opts) -> bool:
        """hj_integrate runs the whole loop in C++ when nothing needs the host
        between stages: range-free bounds, no per-step stats printing, no
        halo exchange (multi-GPU slabs override _stage)."""
        return (self.range_free and not opts.collect_stats and self.exchange is None
                and type(self)._stage is FusedIntegrator._stage)

    def _integrate_native(self, order, t0, t1, y, opts, mask_prev, mask, use_min, check) -> DeviceIntegration:
        import ctypes

        alphas = self._alphas(t0, y)
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

    def _raise_pending(self, times: dict[int, float], warn: bool = False) -> None:
        """Turn the device flags into the exception the reference raises first."""
        s = self.stats.read()
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


def integrate_fused(g, cfg: TermConfig, order: int, tspan, y0_host: np.ndarray, opts) -> DeviceIntegration:
    fi = FusedIntegrator(g, cfg)
    return fi.integrate(order, tspan, dev.to_dev(y0_host), opts)
