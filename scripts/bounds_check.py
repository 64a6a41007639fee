"""Bounds-checked runs of every stage-kernel family (the replacement for
compute-sanitizer memcheck, which is closed on this pool).

    HJ_LIB=check python scripts/bounds_check.py

loads libhjb200_check.so (build.py --check: every global access of the
stage kernels is tested against the extent of its field) and runs each case,
then reads hj_bounds_violations().  Prints one line per case and exits 1 if
any access fell outside its field.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HJ_LIB", "check")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import _lib  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402
from paper_2411_03501_b200.engine import FusedIntegrator  # noqa: E402


def step3(g, cfg, y, dg=None):
    run = FusedIntegrator(g, cfg, dg=dg)
    dt = 0.5 / float(np.sum(cfg.partials.alphas(0.0, g) / g.spacings))
    return run.step3(y, 0.0, dt)


def cases():
    for kernel in ("auto", "brick_always", "generic", "tile_stages", "axes"):
        dev.set_stage_kernel(kernel)
        for scheme in ("weno5", "weno5_fma", "eno3", "eno2", "first"):
            for counts in ((20, 35, 33), (41, 17, 18), (9, 40, 23)):
                g = hj.air3d_grid(counts)
                cfg = hj.air3d_term_config(scheme=scheme)
                y = dev.to_dev(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values)
                yield f"{kernel} 3-D {scheme} {counts}", lambda g=g, cfg=cfg, y=y: step3(g, cfg, y)
        g4 = hj.di4_grid((9, 10, 17, 18))
        yield f"{kernel} 4-D weno5", lambda g4=g4: step3(g4, hj.di4_term_config(scheme="weno5"),
                                                           dev.to_dev(hj.di4_target(g4).values))
        g = hj.air3d_grid((33, 21, 19))
        tgts = [hj.cylinder(g, 2, (0.5 * b, 0.0, 0.0), 5.0).values for b in range(3)]
        yield f"{kernel} batch of 3", lambda g=g, t=tgts: step3(g, hj.air3d_term_config(), dev.to_dev(np.stack(t)),
                                                                 dev.DeviceGrid(g, batch=3))
        gp = hj.create_grid((0.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0), (26, 20, 34), periodic_axes={0, 1, 2})
        yp = np.sin(gp.axis_nodes[0])[:, None, None] + 0 * np.zeros(gp.counts)
        yield f"{kernel} all-periodic advection", lambda gp=gp, yp=yp: step3(
            gp, hj.advection_term_config([1.0, -0.5, 0.25], scheme="weno5"), dev.to_dev(yp))
        gd = hj.with_boundary(hj.air3d_grid((22, 19, 17)), 1, hj.dirichlet(3.0))
        yield f"{kernel} dirichlet", lambda gd=gd: step3(gd, hj.air3d_term_config(),
                                                          dev.to_dev(hj.cylinder(gd, 2, (0, 0, 0), 5.0).values))
    dev.set_stage_kernel("auto")
    # tube with the mask fused into the interval's last stage
    g = hj.air3d_grid((40, 36, 30))
    yield "tube with mask", lambda g=g: hj.solve_tube(g, hj.cylinder(g, 2, (0, 0, 0), 5.0),
                                                     hj.air3d_term_config(), 0.1, 2)
    # pipelined host->host step (hj_stage_planes) on a field above the pipeline threshold
    gb = hj.air3d_grid((161, 161, 161))
    yb = hj.ScalarField(hj.cylinder(gb, 2, (0, 0, 0), 5.0).values)

    def pipelined():
        hj.ode_cfl_3(hj.lax_friedrichs_rhs(gb), (0.0, 1.0), yb, hj.IntegratorOptions(single_step=True),
                     hj.air3d_term_config())
    yield "pipelined host step 161^3", pipelined
    # slabs: exchanged halos, CORE + RIM (LocalTransport) and the NCCL self ring
    from paper_2411_03501_b200.distributed import LocalTransport, SlabIntegrator, lockstep_step3, partition

    gs = hj.air3d_grid((60, 22, 20))
    cfg = hj.air3d_term_config()
    full = hj.cylinder(gs, 2, (0, 0, 0), 5.0).values

    def slabs():
        hub = LocalTransport(partition(60, 4, 3, False))
        runs = [SlabIntegrator(gs, cfg, r, 4, transport=hub.for_rank(r)) for r in range(4)]
        ys = [r.scatter(full) for r in runs]
        dt = 0.5 / float(np.sum(cfg.partials.alphas(0.0, gs) / gs.spacings))
        lockstep_step3(runs, hub, ys, 0.0, dt)
    yield "4 slabs core+rim", slabs
    gr = hj.create_grid((0.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0), (32, 18, 20), periodic_axes={0})
    vr = np.sin(gr.axis_nodes[0])[:, None, None] + 0 * np.zeros(gr.counts)

    def ring():
        acfg = hj.advection_term_config([1.0, 0.5, -0.25], scheme="weno5")
        run = SlabIntegrator(gr, acfg, 0, 1, transport="nccl", self_ring=True)
        run.integrate(3, (0.0, 0.1), run.scatter(vr), hj.IntegratorOptions())
        run.transport.close()
    yield "NCCL self ring interval", ring


def main():
    lib = _lib.load()
    assert _lib.library_path().endswith("_check.so"), "run with HJ_LIB=check"
    assert lib.hj_bounds_violations() == 0
    bad = 0
    n = 0
    for name, fn in cases():
        fn()
        torch.cuda.synchronize()
        v = int(lib.hj_bounds_violations())
        bad += v
        n += 1
        print(f"{'ok ' if v == 0 else 'OOB'} {v:6d}  {name}", flush=True)
    print(f"{n} cases, {bad} out-of-extent accesses")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
