"""Secondary measurements for the BASELINE.json configs other than the
headline (bench.py measures configs[1]).  One JSON line per config:

  C1  Air3D 51x51x36, ENO2 + LF + odeCFL2, t in [0, 2.8], 8 intervals: the
      full horizon through the public solve_tube API (snapshots to host per
      interval), plus the same solve through the CPU oracle;
  C4  4-D double-integrator pair 121^4 WENO5 + RK3 on one GPU: K RK3 steps;
  C5  batch of 8 Air3D 101^3 WENO5 + RK3 problems (one GPU's share of 64):
      K RK3 steps of the stacked batch.
  C2s Air3D 301^3 WENO5 + RK3 full solve_tube over a truncated horizon
      (every interval's snapshot copied to the host), to show the public-API
      cost next to the kernel-only bench.

    python scripts/bench_configs.py [c1] [c4] [c5] [c2s]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import _lib  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402
from paper_2411_03501_b200.engine import FusedIntegrator  # noqa: E402


def sync_time(fn, reps=1):
    """median wall time of ``reps`` calls (synchronised), and the last result"""
    secs = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        secs.append(time.perf_counter() - t0)
    return float(np.median(secs)), out


def c1():
    g = hj.air3d_grid((51, 51, 36))
    cfg = hj.air3d_term_config(scheme="eno2")
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    hj.solve_tube(g, target, cfg, 0.35, 1, order=2)   # warm
    secs, res = sync_time(lambda: hj.solve_tube(g, target, cfg, 2.8, 8, order=2), reps=5)
    fi = FusedIntegrator(g, cfg)
    steps = 0
    t = 0.0
    for k in range(1, 9):   # count RK2 steps exactly as the solve took them
        r = fi.integrate(2, (t, 2.8 * k / 8), dev.to_dev(target.values), hj.IntegratorOptions(), check=False)
        steps += r.steps_taken
        t = 2.8 * k / 8
    cells = int(np.prod(g.counts))
    from oracle import hjoracle as orc
    from hams import oracle_ham

    orc.set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    snaps, _, _ = orc.solve_brt(g, oracle_ham("air3d", g), "eno2", target.values, 2.8, 8, order=2)
    cpu_secs = time.perf_counter() - t0
    same = all(np.array_equal(a.values, b) for a, b in zip(res.snapshots, snaps))
    return {"config": "C1 Air3D 51x51x36 ENO2+LF+odeCFL2 t=[0,2.8] 8 intervals (full solve, public API, median of 5)",
            "gpu_seconds": secs, "rk_steps": steps, "stages": 2 * steps,
            "cell_updates_per_s": cells * 2 * steps / secs,
            "cpu_oracle_seconds": cpu_secs, "cpu_threads": os.cpu_count(),
            "cpu_cell_updates_per_s": cells * 2 * steps / cpu_secs, "bitwise_equal_all_snapshots": same}


def steps_rate(g, cfg, y, k=5, w=2, dg=None):
    fi = FusedIntegrator(g, cfg, dg=dg)
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(alphas / g.spacings))
    for _ in range(w):
        y = fi.step3(y, 0.0, dt)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(k):
        y = fi.step3(y, 0.0, dt)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / k


def c3(scheme="weno5"):
    """C3 Air3D 801^3: one-GPU RK3 steps, and the slab split for 2/4/8 ranks
    emulated on this one GPU (every slab's overlapped core/rim stages run in
    turn, halos copied between stages -- compute only, no NVLink traffic):
    per-rank step time = total / P."""
    from paper_2411_03501_b200.distributed import LocalTransport, SlabIntegrator, lockstep_step3, partition

    n = int(os.environ.get("C3_N", "801"))
    g = hj.air3d_grid(n)
    cfg = hj.air3d_term_config(scheme=scheme)
    dg = dev.device_grid(g)
    y = dev.init_shape_dev(dg, _lib.SHAPE_CYLINDER, [0.0, 0.0, 0.0, 5.0, 4.0])
    sec1 = steps_rate(g, cfg, y, k=3, w=1)
    out = {"config": f"C3 Air3D {n}^3 WENO5+LF+RK3", "scheme": scheme, "ms_per_rk3_step_1gpu": sec1 * 1e3,
           "cell_updates_per_s_1gpu": n ** 3 * 3 / sec1}
    y_host = dev.to_host(y)
    del y
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(alphas / g.spacings))
    emu = {}
    for world in (2, 4, 8):
        slabs = partition(n, world, 3, False)
        hub = LocalTransport(slabs)
        runs = [SlabIntegrator(g, cfg, r, world, transport=hub.for_rank(r)) for r in range(world)]
        ys = [run.scatter(y_host) for run in runs]
        ys = lockstep_step3(runs, hub, ys, 0.0, dt)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(2):
            ys = lockstep_step3(runs, hub, ys, 0.0, dt)
        e.record()
        torch.cuda.synchronize()
        per_rank = s.elapsed_time(e) / 2 / world
        emu[str(world)] = {"ms_per_rk3_step_per_rank": per_rank,
                           "compute_only_strong_scaling_eff": sec1 * 1e3 / (world * per_rank)}
        del runs, ys, hub
        torch.cuda.empty_cache()
    out["slab_emulation_1gpu"] = emu
    return out


def c4(scheme="weno5"):
    n = int(os.environ.get("C4_N", "121"))
    g = hj.di4_grid(n)
    cfg = hj.di4_term_config(scheme=scheme)
    dg = dev.device_grid(g)
    y = dev.init_shape_dev(dg, _lib.SHAPE_CYLINDER, [0.0, 0.0, 0.0, 0.0, 2.0, 12.0])
    sec = steps_rate(g, cfg, y, k=3, w=1)
    cells = n ** 4
    return {"config": f"C4 double-integrator pair {n}^4 WENO5+LF+RK3, 1 GPU", "scheme": scheme,
            "ms_per_rk3_step": sec * 1e3,
            "cell_updates_per_s": cells * 3 / sec}


def c5(scheme="weno5"):
    g = hj.air3d_grid(101)
    cfg = hj.air3d_term_config(scheme=scheme)
    B = 8
    rng = np.random.default_rng(0)
    targets = []
    for _ in range(B):
        cx, cy = rng.uniform(-3.0, 3.0, 2)
        targets.append(hj.cylinder(g, 2, (cx, cy, 0.0), rng.uniform(3.0, 7.0)).values)
    dg = dev.DeviceGrid(g, batch=B)
    y = dev.to_dev(np.stack(targets))
    sec = steps_rate(g, cfg, y, k=5, w=2, dg=dg)
    cells = B * 101 ** 3
    return {"config": "C5 batch of 8 Air3D 101^3 WENO5+LF+RK3 problems (one GPU's share of 64)", "scheme": scheme,
            "ms_per_rk3_step": sec * 1e3, "cell_updates_per_s": cells * 3 / sec}


def c2s(scheme="weno5"):
    g = hj.air3d_grid(301)
    cfg = hj.air3d_term_config(scheme=scheme)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    horizon = 0.02
    hj.solve_tube(g, target, cfg, 0.002, 1)
    secs, res = sync_time(lambda: hj.solve_tube(g, target, cfg, horizon, 4), reps=3)
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(alphas / g.spacings))
    steps = sum(int(np.ceil((horizon / 4) / dt - 1e-12)) for _ in range(4))
    return {"config": "C2 Air3D 301^3 WENO5 solve_tube, horizon 0.02 in 4 intervals (public API, snapshots to host, median of 3)",
            "scheme": scheme,
            "seconds": secs, "approx_rk3_steps": steps,
            "cell_updates_per_s": 301 ** 3 * 3 * steps / secs}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c5", "c4", "c2s"]
    for spec in which:   # name or name:scheme (e.g. c4:weno5_fma)
        name, _, scheme = spec.partition(":")
        out = globals()[name](scheme) if scheme else globals()[name]()
        print(json.dumps({spec: out}), flush=True)
