"""Small fused-stage workload for compute-sanitizer (memcheck / racecheck /
synccheck): one TVD-RK3 step of every brick-kernel family on grids just big
enough to have interior AND boundary bricks, plus a slab with exchanged halos
(CORE + RIM parts) and a 4-D step.  Prints one line per case.

    compute-sanitizer --tool racecheck python scripts/sanitize_probe.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import _lib  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402
from paper_2411_03501_b200.engine import FusedIntegrator  # noqa: E402


def step3(g, cfg, y):
    run = FusedIntegrator(g, cfg)
    a = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(a / g.spacings))
    out = run.step3(y, 0.0, dt)
    torch.cuda.synchronize()
    return out


def main():
    torch.cuda.set_device(0)
    dev.set_stage_kernel("brick_always")
    quick = "--quick" in sys.argv
    for scheme in (("weno5",) if quick else ("weno5", "weno5_fma", "eno2", "eno3", "first")):
        g = hj.air3d_grid((20, 35, 33))
        cfg = hj.air3d_term_config(scheme=scheme)
        y = dev.init_shape_dev(dev.device_grid(g), _lib.SHAPE_CYLINDER, [0.0, 0.0, 0.0, 5.0, 4.0])
        out = step3(g, cfg, y)
        print(f"3-D {scheme} 20x35x33 ok, sum {float(out.sum()):.6e}", flush=True)
    g4 = hj.di4_grid((9, 10, 17, 18))
    cfg4 = hj.di4_term_config(scheme="weno5")
    y4 = dev.to_dev(hj.di4_target(g4).values)
    out = step3(g4, cfg4, y4)
    print(f"4-D weno5 9x10x17x18 ok, sum {float(out.sum()):.6e}", flush=True)
    # slab with exchanged halos on both sides: CORE + RIM launches (LocalTransport)
    from paper_2411_03501_b200.distributed import LocalTransport, SlabIntegrator, lockstep_step3, partition

    g = hj.air3d_grid((48, 20, 18))
    cfg = hj.air3d_term_config(scheme="weno5")
    slabs = partition(48, 3, 3, False)
    hub = LocalTransport(slabs)
    runs = [SlabIntegrator(g, cfg, r, 3, transport=hub.for_rank(r)) for r in range(3)]
    full = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values
    ys = [r.scatter(full) for r in runs]
    a = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(a / g.spacings))
    outs = lockstep_step3(runs, hub, ys, 0.0, dt)
    torch.cuda.synchronize()
    print(f"slab 3-way 48x20x18 ok, sum {sum(float(r.owned(o).sum()) for r, o in zip(runs, outs)):.6e}",
          flush=True)


if __name__ == "__main__":
    main()
