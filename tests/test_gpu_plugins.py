"""The reference's plug-in contract (TermConfig.hamiltonian / partials
callables, term.py:29-30) through the integrator, against goldens made by
running the REFERENCE (tests/golden/make_golden.py gen_plugins ->
plugins.npz):

* range-dependent partials on a registered device Hamiltonian (rockets): the
  fused path's two-pass GLF (a ranges-only pass, the host partials, the term
  pass -- each RK stage with its own costate ranges, term.py:71-83) and the
  per-stage host-term route must both reproduce the reference's ode_cfl_3
  bit for bit;
* Python-lambda Hamiltonians (the host-Hamiltonian bridge) through ode_cfl_3;
* the error contract of _rhs (integrator.py:59-66): the same exception type
  and message as the reference for an invalid bound and a non-finite H, on
  a lambda Hamiltonian and on a registered one;
* dissipation_glf as a public call (term.py:63-87): the ranges handed to
  partials and the dissipation field, against the same formula in NumPy.
"""
import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from golden_io import case_list, package_grid

pytestmark = pytest.mark.gpu

CASES = case_list("plugins.npz")


def range_partials(params):
    # restates make_golden.range_partials
    def partials(t, g, v, ranges, i):
        base = hj.rockets_partials(t, g, v, ranges, i, params)
        return base + 0.01 * (abs(ranges[i][0]) + abs(ranges[i][1]))
    return partials


def lambda_ham(t, g, v, p):
    # restates make_golden.lambda_ham
    x = np.asarray(g.axis_nodes[0]).reshape((-1,) + (1,) * (g.dim - 1))
    h = 0.5 * p[0].values * p[0].values - 0.25 * p[1].values + 0.1 * x * p[g.dim - 1].values
    return type(p[0])(h)


def lambda_partials(t, g, v, ranges, i):
    return max(abs(ranges[i][0]), abs(ranges[i][1])) + 0.5


def _routes(g):
    """The two ways a reference caller reaches the term: the closure the
    package can fuse, and the reference's own lambda idiom."""
    return {"fused": hj.lax_friedrichs_rhs(g),
            "lambda": lambda t, y, c: hj.term_lax_friedrichs(t, y, c, g)}


@pytest.mark.parametrize("i", [i for i, (m, _) in enumerate(CASES) if m["kind"] == "rockets_range_partials"])
@pytest.mark.parametrize("route", ["fused", "lambda"])
def test_range_dependent_partials_on_registered_hamiltonian(i, route):
    meta, arr = CASES[i]
    g = package_grid(meta["grid"])
    params = hj.RocketParams()
    base = hj.rockets_term_config(params, scheme=meta["scheme"])
    cfg = hj.TermConfig(hamiltonian=base.hamiltonian, partials=range_partials(params),
                        derivative_scheme=meta["scheme"])
    assert cfg.on_device   # the registered H keeps the fused route; the partials force the two-pass GLF
    res = hj.ode_cfl_3(_routes(g)[route], (0.0, meta["t1"]), hj.ScalarField(arr["y0"]), hj.IntegratorOptions(),
                       cfg)
    assert np.array_equal(res.y_final.values, arr["y"])
    assert [res.t_final, res.steps_taken, res.min_dt, res.max_dt] == arr["info"].tolist()


@pytest.mark.parametrize("i", [i for i, (m, _) in enumerate(CASES) if m["kind"] == "lambda_ham"])
@pytest.mark.parametrize("route", ["fused", "lambda"])
def test_lambda_hamiltonian_through_the_integrator(i, route):
    meta, arr = CASES[i]
    g = package_grid(meta["grid"])
    cfg = hj.TermConfig(hamiltonian=lambda_ham, partials=lambda_partials, derivative_scheme=meta["scheme"])
    assert not cfg.on_device
    res = hj.ode_cfl_3(_routes(g)[route], (0.0, meta["t1"]), hj.ScalarField(arr["y0"]),
                       hj.IntegratorOptions(cfl_factor=meta["cfl"]), cfg)
    assert np.array_equal(res.y_final.values, arr["y"])
    assert [res.t_final, res.steps_taken, res.min_dt, res.max_dt] == arr["info"].tolist()


def _error_cfg(name, g):
    if name == "invalid_bound":
        return hj.TermConfig(hamiltonian=lambda_ham, partials=lambda *a: -1.0, derivative_scheme="eno2")
    if name == "nan_hamiltonian":
        return hj.TermConfig(hamiltonian=lambda t, gg, v, p: np.full(p[0].values.shape, np.nan),
                             partials=lambda *a: 1.0, derivative_scheme="eno2")
    base = hj.rockets_term_config(hj.RocketParams(), scheme="eno2")
    return hj.TermConfig(hamiltonian=base.hamiltonian, partials=lambda t, gg, v, r, i: -2.0 if i == 1 else 1.0,
                         derivative_scheme="eno2")


@pytest.mark.parametrize("i", [i for i, (m, _) in enumerate(CASES) if m["kind"] == "error"])
@pytest.mark.parametrize("route", ["fused", "lambda"])
def test_error_contract_matches_reference(i, route):
    meta, arr = CASES[i]
    g = package_grid(meta["grid"])
    cfg = _error_cfg(meta["name"], g)
    t1 = 0.05 if meta["name"].startswith("rockets") else 0.08
    opts = hj.IntegratorOptions() if meta["name"].startswith("rockets") else hj.IntegratorOptions(cfl_factor=0.4)
    with pytest.raises((RuntimeError, ValueError)) as info:
        hj.ode_cfl_3(_routes(g)[route], (0.0, t1), hj.ScalarField(arr["y0"]), opts, cfg)
    assert type(info.value).__name__ == meta["error"]
    assert str(info.value) == meta["message"]


def test_dissipation_glf_public_call():
    """term.py:63-87: partials sees the global costate range of each axis,
    and diss = sum_i (alpha_i * 0.5) * (R_i - L_i) accumulated from zeros in
    axis order -- as the reference's test_term.py:136-150 probes it."""
    g = hj.create_grid((-1.0, -2.0, 0.0), (1.0, 2.0, 2 * np.pi), (12, 13, 14), periodic_axes={2})
    rng = np.random.default_rng(17)
    v = hj.ScalarField(rng.standard_normal(g.counts))
    derivs = [hj.derivative_pair(g, v, a, "weno5") for a in range(3)]
    seen = {}

    def partials(t, gg, vv, ranges, i):
        seen[i] = ranges[i]
        return 0.5 + i

    diss, alphas = hj.dissipation_glf(derivs, partials, 0.0, v, g)
    for a, d in enumerate(derivs):
        want = (float(min(d.left.values.min(), d.right.values.min())),
                float(max(d.left.values.max(), d.right.values.max())))
        assert seen[a] == want
    assert alphas.tolist() == [0.5, 1.5, 2.5]
    ref = np.zeros(g.counts)
    for a, d in enumerate(derivs):
        ref += alphas[a] * 0.5 * (d.right.values - d.left.values)
    assert np.array_equal(diss.values, ref)
    with pytest.raises(ValueError, match="invalid bound"):
        hj.dissipation_glf(derivs, lambda *a: float("nan"), 0.0, v, g)
