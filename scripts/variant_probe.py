"""A/B timing of fused-stage kernel variants on the BASELINE grids (device
time of K RK3 steps, CUDA events, inputs larger than L2).

    python scripts/variant_probe.py [c2|c4|c5] variant [variant ...]

variants: auto, brick1, brick_u2, brick_noload (timing bound: bricks after a
CTA's first skip their loads -- wrong results), generic.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402
from paper_2411_03501_b200.engine import FusedIntegrator  # noqa: E402


def setup(cfgname):
    if cfgname == "c4":
        g = hj.di4_grid(int(os.environ.get("C4_N", "121")))
        cfg = hj.di4_term_config(scheme=os.environ.get("SCHEME", "weno5"))
        return g, cfg, dev.to_dev(hj.di4_target(g).values), None
    if cfgname == "c5":
        g = hj.air3d_grid(101)
        cfg = hj.air3d_term_config(scheme=os.environ.get("SCHEME", "weno5"))
        y = dev.to_dev(np.stack([hj.cylinder(g, 2, (0.3 * b, 0.0, 0.0), 5.0).values for b in range(8)]))
        return g, cfg, y, dev.DeviceGrid(g, batch=8)
    n = int(os.environ.get("C2_N", "301"))
    g = hj.air3d_grid(n)
    cfg = hj.air3d_term_config(scheme=os.environ.get("SCHEME", "weno5"))
    return g, cfg, dev.to_dev(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values), None


def main():
    cfgname = sys.argv[1]
    variants = sys.argv[2:] or ["auto"]
    g, cfg, y0, dg = setup(cfgname)
    dt = 0.5 / float(np.sum(cfg.partials.alphas(0.0, g) / g.spacings))
    cells = y0.numel()
    out = {}
    ref = None
    for v in variants:
        old = dev.set_stage_kernel(v)
        fi = FusedIntegrator(g, cfg, dg=dg)
        y = y0.clone()
        for _ in range(3):
            y = fi.step3(y, 0.0, dt)
        ev = []
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        K = 20
        for _ in range(K):
            y = fi.step3(y, 0.0, dt, events=ev)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / K
        stage = [a.elapsed_time(b) for a, b in ev]
        out[v] = {"ms_per_rk3_step": ms, "cell_updates_per_s": cells * 3 / (ms / 1e3),
                  "stage_ms": [float(np.mean(stage[k::3])) for k in range(3)]}
        # bitwise against the first variant after the same 23 steps (timing-only variants differ)
        if ref is None:
            ref = y.clone()
        else:
            out[v]["bitwise_vs_" + variants[0]] = bool(torch.equal(y, ref))
        dev.set_stage_kernel(old)
        del fi, y
    print(json.dumps({"config": cfgname, "grid": list(g.counts), "results": out}), flush=True)


if __name__ == "__main__":
    main()
