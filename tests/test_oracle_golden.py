"""Pin the CPU oracle (oracle/hjoracle.c) to the reference's own outputs.

Every golden vector in tests/golden was produced by running the reference
(tests/golden/make_golden.py).  The oracle must reproduce each of them
bit-for-bit (np.array_equal) before it is trusted as the GPU checker."""
import numpy as np
import pytest

from golden_io import case_list, spec_grid
from hams import oracle_ham
from oracle import hjoracle as orc

SHAPE_SPHERE, SHAPE_CYLINDER, SHAPE_ELLIPSOID, SHAPE_BOX = range(4)


def test_grid_nodes_match_reference():
    for meta, a in case_list("ghost.npz"):
        g = spec_grid(meta["grid"])
        assert np.array_equal(g.spacings, a["spacings"])
        for ax in range(g.dim):
            assert np.array_equal(g.axis_nodes[ax], a[f"nodes{ax}"])


@pytest.mark.parametrize("meta,a", case_list("ghost.npz"))
def test_ghost_extension(meta, a):
    g = spec_grid(meta["grid"])
    assert np.array_equal(orc.extend_ghost(g, a["v"], meta["width"]), a["ext"])


@pytest.mark.parametrize("meta,a", case_list("derivs.npz"))
def test_derivatives(meta, a):
    g = spec_grid(meta["grid"])
    L, R = orc.derivs(g, a["v"], meta["axis"], meta["scheme"], meta["eps_mode"])
    assert np.array_equal(L, a["left"])
    assert np.array_equal(R, a["right"])


@pytest.mark.parametrize("meta,a", case_list("spatial_extra.npz"))
def test_workspace_and_tables(meta, a):
    g = spec_grid(meta["grid"])
    if meta["kind"] == "workspace":
        ws = orc.weno5_workspace(g, a["v"], meta["axis"], meta["side"], meta["eps_mode"])
        for k, v in ws.items():
            assert np.array_equal(v, a[k]), k
    else:
        d0, d1, d2, d3 = orc.divided_differences(g, a["v"], meta["axis"], meta["order"], meta["width"])
        assert np.array_equal(d0, a["d0"]) and np.array_equal(d1, a["d1"])
        if "d2" in a:
            assert np.array_equal(d2, a["d2"])
        if "d3" in a:
            assert np.array_equal(d3, a["d3"])


@pytest.mark.parametrize("meta,a", case_list("term.npz"))
def test_term(meta, a):
    g = spec_grid(meta["grid"])
    ham = oracle_ham(meta["ham"], g, meta, a)
    assert np.array_equal(ham.alphas, a["alphas"])
    delta, bound, ranges, _ = orc.term(g, ham, meta["scheme"], a["v"])
    assert np.array_equal(delta, a["delta"])
    assert bound == float(a["step_bound"])
    assert np.array_equal(np.array(ranges), a["ranges"])


def test_hamiltonians():
    cs = case_list("hamiltonian.npz")
    for meta, a in cs:
        g = spec_grid(meta["grid"])
        if meta["ham"] == "rockets_partials":
            from hams import rockets_alphas
            assert np.array_equal(rockets_alphas(g), a["alphas"])
            continue
        ham = oracle_ham(meta["ham"], g, meta, a)
        H = orc.hamiltonian(g, ham, [a["p0"], a["p1"], a["p2"]])
        assert np.array_equal(H, a["H"])


@pytest.mark.parametrize("meta,a", case_list("integrate.npz"))
def test_integrate(meta, a):
    g = spec_grid(meta["grid"])
    ham = oracle_ham(meta["ham"], g, meta, a)
    t, y, steps, mn, mx = orc.integrate(g, ham, meta["scheme"], meta["order"], (meta["t0"], meta["t1"]), a["y0"],
                                        cfl=meta["cfl"], max_step=meta["max_step"])
    assert np.array_equal(y, a["y"])
    assert [t, steps, mn, mx] == list(a["info"])


@pytest.mark.parametrize("meta,a", case_list("brt.npz"))
def test_brt(meta, a):
    g = spec_grid(meta["grid"])
    ham = oracle_ham(meta["ham"], g, meta, a)
    snaps, times, _ = orc.solve_brt(g, ham, meta["scheme"], a["target"], meta["horizon"], meta["steps"],
                                    order=meta["order"])
    assert times == list(a["times"])
    for k, s in enumerate(snaps):
        assert np.array_equal(s, a["snaps"][k]), f"snapshot {k}"


def test_shapes():
    (meta, a), (meta4, a4) = case_list("shapes.npz")
    g = spec_grid(meta["grid"])
    assert np.array_equal(orc.shape(g, SHAPE_SPHERE, [0.1, 0.5, 0.2, 1.2]), a["sphere"])
    assert np.array_equal(orc.shape(g, SHAPE_CYLINDER, [0.0, 1.0, 0.0, 1.5, 4]), a["cylinder"])
    assert np.array_equal(orc.shape(g, SHAPE_CYLINDER, [0.0, 1.0, 0.3, 0.9, 1]), a["cylinder0"])
    assert np.array_equal(orc.shape(g, SHAPE_ELLIPSOID, [1.0, 4.0, 9.0, 2.0]), a["ellipsoid"])
    assert np.array_equal(orc.shape(g, SHAPE_BOX, [-1.0, 0.0, -1.0, 0.5, 2.0, 1.5]), a["box"])
    g4 = spec_grid(meta4["grid"])
    assert np.array_equal(orc.shape(g4, SHAPE_CYLINDER, [0.0, 0.0, 0.0, 0.0, 2.0, 12]), a4["target"])


def test_threaded_oracle_is_deterministic():
    meta, a = [c for c in case_list("term.npz") if c[0]["ham"] == "air3d" and c[0]["scheme"] == "weno5"][0]
    g = spec_grid(meta["grid"])
    ham = oracle_ham("air3d", g, meta, a)
    orc.set_threads(4)
    try:
        d4 = orc.term(g, ham, "weno5", a["v"])[0]
    finally:
        orc.set_threads(1)
    assert np.array_equal(d4, a["delta"])
