"""Slab decomposition on one GPU: every slab of a 2/3/4-way split runs its own
fused stage kernels on its own buffers, halos copied between stages (the
LocalTransport emulation -- no kernel waits on another).  The assembled
result must equal the single-domain run bit for bit."""
import numpy as np
import pytest
import torch

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import _lib
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.distributed import LocalTransport, SlabIntegrator, lockstep_step3, partition
from paper_2411_03501_b200.engine import FusedIntegrator

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("stage_kernel")]


def _run(g, cfg, y0_host, world, steps=3):
    single = FusedIntegrator(g, cfg)
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(alphas / g.spacings))
    y = dev.to_dev(y0_host)
    t = 0.0
    for _ in range(steps):
        y = single.step3(y, t, dt)
        t += dt
    ref = dev.to_host(y)

    slabs = partition(g.counts[0], world, 3, g.is_periodic(0))
    hub = LocalTransport(slabs)
    runs = [SlabIntegrator(g, cfg, r, world, transport=hub.for_rank(r)) for r in range(world)]
    ys = [run.scatter(y0_host) for run in runs]
    t = 0.0
    for _ in range(steps):
        ys = lockstep_step3(runs, hub, ys, t, dt)
        t += dt
    got = np.concatenate([dev.to_host(run.owned(y)) for run, y in zip(runs, ys)], axis=0)
    return ref, got


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("scheme", ["weno5", "eno2"])
def test_air3d_slabs_equal_single_domain(world, scheme):
    g = hj.air3d_grid((61, 40, 36))
    cfg = hj.air3d_term_config(scheme=scheme)
    y0 = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values
    ref, got = _run(g, cfg, y0, world)
    assert np.array_equal(ref, got)


@pytest.mark.parametrize("world", [2, 3])
def test_periodic_axis0_ring(world):
    g = hj.create_grid((0.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0), (48, 20, 24), periodic_axes={0})
    cfg = hj.advection_term_config([1.0, -0.5, 0.25], scheme="weno5")
    x = g.axis_nodes[0][:, None, None]
    y0 = np.sin(x) + 0.1 * np.cos(3 * g.axis_nodes[1][None, :, None]) + 0 * g.axis_nodes[2][None, None, :]
    ref, got = _run(g, cfg, y0, world)
    assert np.array_equal(ref, got)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("scheme", ["weno5", "eno3", "weno5_fma"])
def test_4d_slabs_equal_single_domain(world, scheme):
    """4-D slabs: the axis-0 pre-pass segments and brick slices split into the
    core / rim parts of the overlapped stage."""
    g = hj.di4_grid((41, 14, 17, 18))
    cfg = hj.di4_term_config(scheme=scheme)
    ref, got = _run(g, cfg, hj.di4_target(g).values, world, steps=2)
    assert np.array_equal(ref, got)


@pytest.mark.parametrize("world", [2, 5])
def test_core_rim_split_equals_unsplit(world):
    """Overlapped stages (CORE while the exchange is in flight, then RIM) give
    the same bits as exchange-then-whole-stage, including slabs too thin to
    have a core (world 5: 12-13 planes per slab)."""
    g = hj.air3d_grid((61, 40, 36))
    cfg = hj.air3d_term_config(scheme="weno5_fma")
    y0 = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(alphas / g.spacings))
    outs = []
    for overlap in (True, False):
        slabs = partition(g.counts[0], world, 3, False)
        hub = LocalTransport(slabs)
        runs = [SlabIntegrator(g, cfg, r, world, transport=hub.for_rank(r), overlap=overlap) for r in range(world)]
        ys = [run.scatter(y0) for run in runs]
        for k in range(2):
            ys = lockstep_step3(runs, hub, ys, k * dt, dt)
        outs.append(np.concatenate([dev.to_host(run.owned(y)) for run, y in zip(runs, ys)], axis=0))
    assert np.array_equal(outs[0], outs[1])
