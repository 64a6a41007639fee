"""CUDA path vs the CPU oracle on seeded inputs beyond the golden sizes, and
size-independent properties at the benchmark sizes (BASELINE.json configs).

Bar: bit-exact (np.array_equal) -- both sides restate the reference's
operation order; the north-star tolerance (L-inf rel <= 1e-9, identical
sign(V)) is therefore met with zero error."""
import math
import os

import numpy as np
import pytest
import torch

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.engine import FusedIntegrator
from golden_io import spec_grid
from hams import oracle_ham
from oracle import hjoracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("stage_kernel")]
orc.set_threads(os.cpu_count() or 1)

SPECS = [
    dict(mins=[-1.0], maxs=[2.0], counts=[257], periodic=[], dirichlet={}),
    dict(mins=[-1.0, 0.0], maxs=[1.0, 3.0], counts=[65, 70], periodic=[1], dirichlet={"0": 0.25}),
    dict(mins=[-1.0, -2.0, 0.0], maxs=[1.0, 2.0, 6.0], counts=[33, 34, 35], periodic=[2], dirichlet={}),
    dict(mins=[-1.0, -1.0, -1.0], maxs=[1.0, 1.0, 1.0], counts=[20, 21, 22], periodic=[0],
         dirichlet={"1": -0.5}),
    dict(mins=[-1.0] * 4, maxs=[1.0] * 4, counts=[12, 13, 11, 14], periodic=[3], dirichlet={}),
]


def _grid(spec):
    g = hj.create_grid(spec["mins"], spec["maxs"], spec["counts"], periodic_axes=set(spec["periodic"]))
    for k, v in spec["dirichlet"].items():
        g = hj.with_boundary(g, int(k), hj.dirichlet(v))
    return g


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("scheme", ["first", "eno2", "eno3", "weno5"])
def test_derivatives_random(spec, scheme):
    g = _grid(spec)
    rng = np.random.default_rng([len(scheme), *spec["counts"]])
    v = rng.standard_normal(g.counts) * rng.uniform(0.1, 10.0)
    v[tuple(slice(0, 3) for _ in range(g.dim))] = 0.0   # exact zeros / ties in the ENO picks
    for axis in range(g.dim):
        pair = hj.derivative_pair(g, hj.ScalarField(v), axis, scheme)
        L, R = orc.derivs(g, v, axis, scheme)
        assert np.array_equal(pair.left.values, L) and np.array_equal(pair.right.values, R)


def _air3d(n):
    g = hj.air3d_grid(n)
    cfg = hj.air3d_term_config(scheme="weno5")
    ham = oracle_ham("air3d", g)
    return g, cfg, ham


@pytest.mark.parametrize("scheme,order", [("weno5", 3), ("eno2", 2), ("eno3", 3), ("first", 1)])
def test_air3d_steps_vs_oracle(scheme, order):
    g = hj.air3d_grid((41, 43, 36))
    cfg = hj.air3d_term_config(scheme=scheme)
    ham = oracle_ham("air3d", g)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    opts = hj.IntegratorOptions(cfl_factor=0.5)
    res = hj.ode_cfl_3(hj.lax_friedrichs_rhs(g), (0.0, 0.08), target, opts, cfg) if order == 3 else \
        {1: hj.ode_cfl_1, 2: hj.ode_cfl_2}[order](hj.lax_friedrichs_rhs(g), (0.0, 0.08), target, opts, cfg)
    t, y, steps, mn, mx = orc.integrate(g, ham, scheme, order, (0.0, 0.08), target.values, cfl=0.5)
    assert np.array_equal(res.y_final.values, y)
    assert (res.t_final, res.steps_taken, res.min_dt, res.max_dt) == (t, steps, mn, mx)


def test_c1_full_horizon_vs_oracle():
    """BASELINE configs[0]: Air3D 51x51x36, ENO2 + LF + odeCFL2, t in [0, 2.8],
    8 intervals -- every saved time bit-identical to the oracle."""
    g = hj.air3d_grid((51, 51, 36))
    cfg = hj.air3d_term_config(scheme="eno2")
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    res = hj.solve_tube(g, target, cfg, 2.8, 8, order=2)
    snaps, times, _ = orc.solve_brt(g, oracle_ham("air3d", g), "eno2", target.values, 2.8, 8, order=2)
    assert list(res.times) == times
    for k, s in enumerate(res.snapshots):
        assert np.array_equal(s.values, snaps[k]), k
    # the tube grows and stays nested (reference invariants)
    vol = [int(np.count_nonzero(s.values < 0)) for s in res.snapshots]
    assert all(b >= a for a, b in zip(vol, vol[1:])) and vol[-1] > vol[0]


def test_di4_steps_vs_oracle():
    g = hj.di4_grid((17, 15, 16, 14))
    cfg = hj.di4_term_config(scheme="weno5")
    target = hj.di4_target(g)
    res = hj.ode_cfl_3(hj.lax_friedrichs_rhs(g), (0.0, 0.05), target, hj.IntegratorOptions(), cfg)
    t, y, steps, _, _ = orc.integrate(g, oracle_ham("di4", g), "weno5", 3, (0.0, 0.05), target.values)
    assert np.array_equal(res.y_final.values, y) and res.steps_taken == steps


def test_rockets_extremal_eno3_vs_oracle():
    g = hj.create_grid((-64, -64, -math.pi), (64, 64, math.pi), (31, 29, 30), periodic_axes={2})
    p = hj.RocketParams(capture_radius=15.0)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 15.0)
    for route in ("published", "extremal"):
        cfg = hj.rockets_term_config(p, scheme="eno3", hamiltonian=route)
        res = hj.solve_brt(hj.ReachProblem(grid=g, target=target, params=p, term_config=cfg, horizon=0.3,
                                           global_steps=2))
        ham = oracle_ham("rockets" if route == "published" else "rockets_extremal", g)
        snaps, _, _ = orc.solve_brt(g, ham, "eno3", target.values, 0.3, 2, order=3)
        for k, s in enumerate(res.snapshots):
            assert np.array_equal(s.values, snaps[k])


def test_c2_full_size_one_rk3_step_vs_oracle():
    """BASELINE configs[1] size: Air3D 301^3 WENO5 + RK3 -- one full step,
    every node bit-identical to the (threaded) oracle."""
    g = hj.air3d_grid(301)
    cfg = hj.air3d_term_config(scheme="weno5")
    dg = dev.device_grid(g)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    fi = FusedIntegrator(g, cfg)
    res = fi.integrate(3, (0.0, 1.0), dev.to_dev(target.values), hj.IntegratorOptions(single_step=True))
    y_gpu = dev.to_host(res.y)
    t, y, steps, _, _ = orc.integrate(g, oracle_ham("air3d", g), "weno5", 3, (0.0, 1.0), target.values,
                                      single_step=True)
    assert steps == 1 and res.steps_taken == 1
    assert np.array_equal(y_gpu, y)
    assert np.array_equal(np.sign(y_gpu), np.sign(y))
    del dg


def test_full_size_determinism_and_symmetry():
    """Run-to-run bitwise determinism at 301^3 and the mirror property of the
    upwind pair (test_spatial.py:206-216) on a full-size line bundle."""
    g = hj.air3d_grid(301)
    cfg = hj.air3d_term_config(scheme="weno5")
    target = dev.to_dev(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values)
    opts = hj.IntegratorOptions(single_step=True)
    a = FusedIntegrator(g, cfg).integrate(3, (0.0, 1.0), target, opts).y
    b = FusedIntegrator(g, cfg).integrate(3, (0.0, 1.0), target, opts).y
    assert torch.equal(a, b)
    g1 = hj.create_grid((-1.0,), (2.0,), (301,))
    x = g1.axis_nodes[0]
    vals = np.sin(2 * x) + 0.3 * np.cos(5 * x) + 0.1 * np.abs(x - 0.5)
    for scheme in ("first", "eno2", "eno3", "weno5"):
        p = hj.derivative_pair(g1, hj.ScalarField(vals), 0, scheme)
        pr = hj.derivative_pair(g1, hj.ScalarField(vals[::-1]), 0, scheme)
        assert np.array_equal(p.right.values, -pr.left.values[::-1])
        assert np.array_equal(p.left.values, -pr.right.values[::-1])


def test_nonfinite_detection_matches_reference_message():
    """A dirichlet ghost of 1.7e308 overflows the first difference; the
    reference raises 'term evaluation failed at step 0 (t=0): field contains
    non-finite values' (checked against the reference when the case was
    written).  The fused path must raise the same."""
    g = hj.with_boundary(hj.create_grid((0.0,), (1.0,), (64,)), 0, hj.dirichlet(1.7e308))
    cfg = hj.advection_term_config([1.0], scheme="first")
    y0 = hj.ScalarField(np.sin(2 * np.pi * g.axis_nodes[0]))
    with pytest.raises(RuntimeError) as ei:
        hj.ode_cfl_1(hj.lax_friedrichs_rhs(g), (0.0, 1.0), y0, hj.IntegratorOptions(), cfg)
    assert str(ei.value) == "term evaluation failed at step 0 (t=0): field contains non-finite values"
    g3 = hj.with_boundary(hj.air3d_grid((20, 18, 16)), 0, hj.dirichlet(1.7e308))
    cfg3 = hj.air3d_term_config(scheme="weno5")
    with pytest.raises(RuntimeError, match="tube interval 1 failed: term evaluation failed at step 0"):
        hj.solve_tube(g3, hj.cylinder(g3, 2, (0.0, 0.0, 0.0), 5.0), cfg3, 0.1, 2)


@pytest.mark.parametrize("scheme", ["first", "eno2", "eno3", "weno5"])
def test_4d_brick_path_vs_oracle(scheme):
    """4-D grids run the axis-0 pre-pass + brick kernel over axes 1-3; every
    scheme, partial bricks on every axis, periodic and extrapolated axes."""
    g = hj.create_grid((-1.0, -2.0, -1.0, 0.0), (1.0, 2.0, 1.5, 6.0), (13, 19, 18, 21), periodic_axes={3})
    cfg = hj.advection_term_config([1.0, -0.7, 0.4, 0.3], scheme=scheme)
    X = np.meshgrid(*g.axis_nodes, indexing="ij")
    y0 = np.sin(X[0] * 2.0) + np.cos(X[1]) * X[2] + 0.2 * np.sin(X[3]) + np.abs(X[2] - 0.3)
    res = hj.ode_cfl_3(hj.lax_friedrichs_rhs(g), (0.0, 0.2), hj.ScalarField(y0), hj.IntegratorOptions(), cfg)
    ham = orc.Ham("advection", [1.0, -0.7, 0.4, 0.3], alphas=[1.0, 0.7, 0.4, 0.3])
    t, y, steps, _, _ = orc.integrate(g, ham, scheme, 3, (0.0, 0.2), y0)
    assert steps == res.steps_taken and np.array_equal(res.y_final.values, y)
    gd = hj.di4_grid((11, 12, 17, 18))
    cfgd = hj.di4_term_config(scheme=scheme)
    tgt = hj.di4_target(gd)
    r2 = hj.ode_cfl_2(hj.lax_friedrichs_rhs(gd), (0.0, 0.1), tgt, hj.IntegratorOptions(), cfgd)
    _, y2, _, _, _ = orc.integrate(gd, oracle_ham("di4", gd), scheme, 2, (0.0, 0.1), tgt.values)
    assert np.array_equal(r2.y_final.values, y2)
