"""CUDA path vs the reference's golden vectors, bit for bit (np.array_equal).

Each case calls the package's public API (the same call a reference user
makes); the arithmetic runs in libhjb200.so on the GPU."""
import math

import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from golden_io import case_list, package_grid
from pkg_configs import package_config

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("stage_kernel")]


@pytest.mark.parametrize("meta,a", case_list("ghost.npz"))
def test_ghost(meta, a):
    g = package_grid(meta["grid"])
    ext = hj.extend_with_ghost_cells(g, hj.ScalarField(a["v"]), meta["width"])
    assert np.array_equal(ext.values, a["ext"])


@pytest.mark.parametrize("meta,a", case_list("derivs.npz"))
def test_derivatives(meta, a):
    g = package_grid(meta["grid"])
    f = hj.ScalarField(a["v"])
    if meta["eps_mode"] == "raw":
        pair = hj.upwind_first_weno5(g, f, meta["axis"], eps_mode="raw")
    else:
        pair = hj.derivative_pair(g, f, meta["axis"], meta["scheme"])
    assert np.array_equal(pair.left.values, a["left"])
    assert np.array_equal(pair.right.values, a["right"])


@pytest.mark.parametrize("meta,a", case_list("spatial_extra.npz"))
def test_workspace_and_tables(meta, a):
    g = package_grid(meta["grid"])
    f = hj.ScalarField(a["v"])
    if meta["kind"] == "workspace":
        ws = hj.weno5_workspace(g, f, meta["axis"], side=meta["side"], eps_mode=meta["eps_mode"])
        for k in ("sigma1", "sigma2", "sigma3", "alpha1", "alpha2", "alpha3", "eps", "w1", "w2", "w3"):
            assert np.array_equal(getattr(ws, k), a[k]), k
    else:
        t = hj.divided_differences(g, f, meta["axis"], order=meta["order"], width=meta["width"])
        assert np.array_equal(t.d0, a["d0"]) and np.array_equal(t.d1, a["d1"])
        assert (t.d2 is None) == ("d2" not in a) and (t.d3 is None) == ("d3" not in a)
        if t.d2 is not None:
            assert np.array_equal(t.d2, a["d2"])
        if t.d3 is not None:
            assert np.array_equal(t.d3, a["d3"])


@pytest.mark.parametrize("meta,a", case_list("term.npz"))
def test_term_fused(meta, a):
    g = package_grid(meta["grid"])
    cfg = package_config(meta["ham"], meta["scheme"], meta, a)
    out = hj.term_lax_friedrichs(0.0, hj.ScalarField(a["v"]), cfg, g)
    assert np.array_equal(out.delta.values, a["delta"])
    assert out.step_bound == float(a["step_bound"])


@pytest.mark.parametrize("meta,a", [c for c in case_list("term.npz") if c[0]["ham"] == "advection"])
def test_term_host_hamiltonian_bridge(meta, a):
    """A plain Python Hamiltonian (not registered) goes through the bridge:
    derivatives / ranges / dissipation on the GPU, H on the host."""
    g = package_grid(meta["grid"])
    c = np.asarray(meta["speeds"])

    def ham(t, gg, v, p):
        out = np.zeros(v.grid_shape)
        for i in range(gg.dim):
            out += c[i] * p[i].values
        return hj.ScalarField(out)

    seen = {}

    def partials(t, gg, v, ranges, axis):
        seen["ranges"] = ranges
        return abs(float(c[axis]))

    cfg = hj.TermConfig(hamiltonian=ham, partials=partials, derivative_scheme=meta["scheme"])
    out = hj.term_lax_friedrichs(0.0, hj.ScalarField(a["v"]), cfg, g)
    assert np.array_equal(out.delta.values, a["delta"])
    assert np.array_equal(np.array(seen["ranges"]), a["ranges"])


def test_hamiltonian_api():
    cs = case_list("hamiltonian.npz")
    for meta, a in cs[:2]:
        g = package_grid(meta["grid"])
        if not (np.array_equal(np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel(), a["cos"])
                and np.array_equal(np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel(), a["sin"])):
            pytest.skip("this host's np.cos/np.sin differ from the golden host's; covered via fixed tables")
        p = [hj.ScalarField(a[f"p{i}"]) for i in range(3)]
        fn = hj.rockets_hamiltonian if meta["ham"] == "rockets" else hj.rockets_hamiltonian_extremal
        assert np.array_equal(fn(0.0, g, None, p, hj.RocketParams()).values, a["H"])


@pytest.mark.parametrize("meta,a", case_list("integrate.npz"))
def test_integrate_fused(meta, a):
    g = package_grid(meta["grid"])
    cfg = package_config(meta["ham"], meta["scheme"], meta, a)
    integ = {1: hj.ode_cfl_1, 2: hj.ode_cfl_2, 3: hj.ode_cfl_3}[meta["order"]]
    opts = hj.IntegratorOptions(cfl_factor=meta["cfl"], max_step=meta["max_step"])
    res = integ(hj.lax_friedrichs_rhs(g), (meta["t0"], meta["t1"]), hj.ScalarField(a["y0"]), opts, cfg)
    assert np.array_equal(res.y_final.values, a["y"])
    assert [res.t_final, res.steps_taken, res.min_dt, res.max_dt] == list(a["info"])


@pytest.mark.parametrize("meta,a", [c for c in case_list("integrate.npz") if c[0]["ham"] == "advection"])
def test_integrate_reference_style_closure(meta, a):
    """The reference tests' own idiom -- a lambda calling term_lax_friedrichs --
    runs the generic integrator route (term per stage, combos on the GPU)."""
    g = package_grid(meta["grid"])
    cfg = package_config(meta["ham"], meta["scheme"], meta, a)
    integ = {1: hj.ode_cfl_1, 2: hj.ode_cfl_2, 3: hj.ode_cfl_3}[meta["order"]]
    opts = hj.IntegratorOptions(cfl_factor=meta["cfl"], max_step=meta["max_step"])
    res = integ(lambda t, y, c: hj.term_lax_friedrichs(t, y, c, g), (meta["t0"], meta["t1"]),
                hj.ScalarField(a["y0"]), opts, cfg)
    assert np.array_equal(res.y_final.values, a["y"])
    assert [res.t_final, res.steps_taken, res.min_dt, res.max_dt] == list(a["info"])


@pytest.mark.parametrize("meta,a", case_list("brt.npz"))
def test_brt(meta, a):
    g = package_grid(meta["grid"])
    rp = hj.RocketParams(capture_radius=meta["params"]["capture_radius"]) if "params" in meta else None
    cfg = package_config(meta["ham"], meta["scheme"], meta, a, rocket_params=rp)
    target = hj.ScalarField(a["target"])
    if meta["ham"].startswith("rockets"):
        prob = hj.ReachProblem(grid=g, target=target, params=rp, term_config=cfg, horizon=meta["horizon"],
                               global_steps=meta["steps"])
        res = hj.solve_brt(prob)
    else:
        res = hj.solve_tube(g, target, cfg, meta["horizon"], meta["steps"], order=meta["order"])
    assert list(res.times) == list(a["times"])
    for k, s in enumerate(res.snapshots):
        assert np.array_equal(s.values, a["snaps"][k]), f"snapshot {k}"


def test_shapes():
    (meta, a), (meta4, a4) = case_list("shapes.npz")
    g = package_grid(meta["grid"])
    sph = hj.sphere(g, (0.1, 0.5, 0.2), 1.2)
    box = hj.hyper_rectangle(g, (-1.0, 0.0, -1.0), (0.5, 2.0, 1.5))
    cyl = hj.cylinder(g, 2, (0.0, 1.0, 0.0), 1.5)
    assert np.array_equal(sph.values, a["sphere"])
    assert np.array_equal(cyl.values, a["cylinder"])
    assert np.array_equal(hj.cylinder(g, 0, (0.0, 1.0, 0.3), 0.9).values, a["cylinder0"])
    assert np.array_equal(hj.ellipsoid(g, (1.0, 4.0, 9.0), 2.0).values, a["ellipsoid"])
    assert np.array_equal(box.values, a["box"])
    assert np.array_equal(hj.csg_union(sph, box).values, a["union"])
    assert np.array_equal(hj.csg_intersect(sph, box).values, a["intersect"])
    assert np.array_equal(hj.csg_complement(cyl).values, a["complement"])
    assert np.array_equal(hj.csg_difference(box, sph).values, a["difference"])
    assert np.array_equal(hj.mesh_coordinates(g, 0).values, a["mesh0"])
    assert [hj.sublevel_volume(g, sph), hj.sublevel_volume(g, box, level=0.3)] == list(a["vol"])
    g4 = package_grid(meta4["grid"])
    assert np.array_equal(hj.di4_target(g4).values, a4["target"])
