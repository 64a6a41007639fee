"""Parity at the BASELINE.json sizes: the CUDA path against the CPU oracle
(oracle/hjoracle.c, threaded, the restatement pinned to the reference's own
goldens by tests/test_oracle_golden.py) on the benchmark configurations
themselves, not only on small grids.

  C1  Air3D 51x51x36 ENO2 + odeCFL2, full horizon [0, 2.8], 8 intervals
  C2  the exact WENO5 + RK3 full-horizon tube [0, 2.8], 8 saved times, at
      51^3 and 101^3 (a 301^3 full horizon is 3936 steps: ~2 h on the CPU
      oracle; one 301^3 step is pinned in test_gpu_oracle.py)
  C3  one RK3 step at 801^3 (or the largest cube the host RAM holds for the
      oracle; the test prints which)
  C4  one RK3 step of the 4-D pair at 121^4
  C5  members of the 8 x 101^3 batch (solve_tube_batch) against single
      oracle tubes

Bar: bit-exact (np.array_equal) at every saved time -- the north-star gate
(L-inf rel <= 1e-9, identical sign(V)) is met with zero error.  Each test
runs the default kernel dispatch (the brick kernels at these sizes)."""
import os

import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.engine import FusedIntegrator
from hams import oracle_ham
from oracle import hjoracle as orc

pytestmark = pytest.mark.gpu
orc.set_threads(os.cpu_count() or 1)


def _avail_bytes() -> int:
    try:
        import psutil

        return int(psutil.virtual_memory().available)
    except Exception:
        return int(os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE"))


def _assert_tube(res, snaps, times):
    assert list(res.times) == list(times)
    assert len(res.snapshots) == len(snaps)
    for k, s in enumerate(res.snapshots):
        assert np.array_equal(s.values, snaps[k]), f"snapshot {k} (t={times[k]}) differs"
        assert np.array_equal(np.sign(s.values), np.sign(snaps[k]))


def test_c1_full_horizon_eno2_rk2():
    g = hj.air3d_grid((51, 51, 36))
    cfg = hj.air3d_term_config(scheme="eno2")
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    res = hj.solve_tube(g, target, cfg, 2.8, 8, order=2)
    snaps, times, steps = orc.solve_brt(g, oracle_ham("air3d", g), "eno2", target.values, 2.8, 8, order=2)
    assert sum(steps) == 632
    _assert_tube(res, snaps, times)


@pytest.mark.parametrize("n", [51, 101])
def test_air3d_weno5_full_horizon_tube(n):
    """The exact-WENO5 Air3D tube over the whole horizon [0, 2.8] with its 8
    saved times -- the configs[1] path (brick kernel, mask fused into each
    interval's last stage) over thousands of stages."""
    g = hj.air3d_grid(n)
    cfg = hj.air3d_term_config(scheme="weno5")
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    res = hj.solve_tube(g, target, cfg, 2.8, 8, order=3)
    snaps, times, steps = orc.solve_brt(g, oracle_ham("air3d", g), "weno5", target.values, 2.8, 8, order=3)
    print(f"air3d {n}^3 weno5 full horizon: {sum(steps)} RK3 steps, 9 snapshots bit-identical")
    _assert_tube(res, snaps, times)


def _one_step(g, cfg, ham, y0):
    fi = FusedIntegrator(g, cfg)
    res = fi.integrate(3, (0.0, 1.0), dev.to_dev(y0), hj.IntegratorOptions(single_step=True))
    y_gpu = dev.to_host(res.y)
    del fi, res
    _, y, steps, _, _ = orc.integrate(g, ham, "weno5", 3, (0.0, 1.0), y0, single_step=True)
    assert steps == 1
    return y_gpu, y


def test_c3_size_one_rk3_step():
    n = 801
    # the oracle holds ~16 fields of the grid at once (ghost-extended tables, stage buffers)
    while n > 301 and 16 * 8 * n ** 3 > _avail_bytes():
        n -= 50
    print(f"C3 parity step at {n}^3 (host RAM available: {_avail_bytes() / 2**30:.0f} GiB)")
    g = hj.air3d_grid(n)
    cfg = hj.air3d_term_config(scheme="weno5")
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values
    y_gpu, y = _one_step(g, cfg, oracle_ham("air3d", g), target)
    assert np.array_equal(y_gpu, y)


def test_c4_full_size_one_rk3_step():
    g = hj.di4_grid(121)
    cfg = hj.di4_term_config(scheme="weno5")
    target = hj.di4_target(g).values
    if 16 * target.nbytes > _avail_bytes():
        pytest.skip(f"host RAM {_avail_bytes() / 2**30:.0f} GiB too small for the 121^4 oracle step")
    y_gpu, y = _one_step(g, cfg, oracle_ham("di4", g), target)
    assert np.array_equal(y_gpu, y)


def test_c5_batch_members_vs_oracle():
    """Two members of the 8 x 101^3 flock (targets from default_rng(0), as the
    runner draws them) against single-problem oracle tubes."""
    g = hj.air3d_grid(101)
    cfg = hj.air3d_term_config(scheme="weno5")
    rng = np.random.default_rng(0)
    targets = []
    for _ in range(8):
        cx, cy = rng.uniform(-3.0, 3.0, 2)
        targets.append(hj.cylinder(g, 2, (cx, cy, 0.0), rng.uniform(3.0, 7.0)).values)
    snaps, times = hj.solve_tube_batch(g, targets, cfg, 0.35, 2, order=3)
    assert snaps.shape == (3, 8, 101, 101, 101)
    for m in (0, 5):
        ref, rtimes, _ = orc.solve_brt(g, oracle_ham("air3d", g), "weno5", targets[m], 0.35, 2, order=3)
        assert list(times) == list(rtimes)
        for k in range(3):
            assert np.array_equal(snaps[k, m], ref[k]), f"member {m} snapshot {k}"


@pytest.mark.parametrize("sign", ["over", "under"])
def test_device_tube_diagnostics_match_host_checks(sign):
    """solve_tube(diagnostics=[...]) evaluates the reference's tube acceptance
    checks (test_reachability.py:218-285: nesting, target containment,
    sublevel volume) on the GPU; they must equal the same counts taken on the
    host snapshots."""
    g = hj.air3d_grid((48, 44, 40))
    base = hj.air3d_term_config(scheme="weno5")
    cfg = hj.TermConfig(hamiltonian=base.hamiltonian, partials=base.partials, derivative_scheme="weno5",
                        approximation_sign=sign)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    diag = []
    res = hj.solve_tube(g, target, cfg, 0.6, 4, diagnostics=diag)
    assert [d["interval"] for d in diag] == [1, 2, 3, 4]
    snaps = [s.values for s in res.snapshots]
    for k, d in enumerate(diag, start=1):
        a, b = snaps[k - 1], snaps[k]
        worse = (b > a) if sign == "over" else (b < a)
        outside = (b > target.values) if sign == "over" else (b < target.values)
        assert d["nesting_violations"] == int(worse.sum()) == 0
        assert d["containment_violations"] == int(outside.sum())
        assert d["sublevel_nodes"] == int((b < 0).sum())
        assert d["captured"] == int(((a >= 0) & (b < 0)).sum())
        assert d["volume"] == pytest.approx(hj.sublevel_volume(g, res.snapshots[k]))
    if sign == "over":
        assert all(d["containment_violations"] == 0 for d in diag)
        assert diag[-1]["sublevel_nodes"] > int((target.values < 0).sum())
    # the same checks without any per-interval snapshot copy
    diag2 = []
    lean = hj.solve_tube(g, target, cfg, 0.6, 4, diagnostics=diag2, keep_snapshots=False)
    assert diag2 == diag and np.array_equal(lean.snapshots[-1].values, snaps[-1])
