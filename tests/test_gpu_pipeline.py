"""The host->host single-step pipeline (engine.FusedIntegrator.integrate_host):
H2D chunks, stages over the planes whose stencils are complete
(hj_stage_planes), D2H of finished planes -- must give the same bits as the
unpipelined device integration, for every order, scheme and kernel family."""
import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import _lib
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.engine import FusedIntegrator

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("stage_kernel")]


@pytest.fixture(params=[(16, True), (8, False)], ids=["chunk16-prio", "chunk8-noprio"])
def small_pipeline(monkeypatch, request):
    chunk, prio = request.param
    monkeypatch.setattr(FusedIntegrator, "pipeline_min_cells", 0)
    monkeypatch.setattr(FusedIntegrator, "pipeline_chunk", chunk)
    monkeypatch.setattr(FusedIntegrator, "pipeline_priority", prio)


def _both(g, cfg, y0, order, opts):
    fi = FusedIntegrator(g, cfg)
    t, y, steps, mn, mx = fi.integrate_host(order, (0.0, 1.0), y0, opts)
    ref = FusedIntegrator(g, cfg).integrate(order, (0.0, 1.0), dev.to_dev(y0), opts)
    assert fi.launches > order   # really pipelined (several plane ranges per stage)
    return (t, y, steps, mn, mx), (ref.t_final, dev.to_host(ref.y), ref.steps_taken, ref.min_dt, ref.max_dt)


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("scheme", ["weno5", "eno2", "weno5_fma"])
def test_air3d_single_step(small_pipeline, order, scheme):
    g = hj.air3d_grid((61, 40, 36))
    y0 = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values
    a, b = _both(g, hj.air3d_term_config(scheme=scheme), y0, order, hj.IntegratorOptions(single_step=True))
    assert a[0] == b[0] and a[2:] == b[2:]
    assert np.array_equal(a[1], b[1])


@pytest.mark.parametrize("periodic0", [False, True])
def test_short_span_is_one_step(small_pipeline, periodic0):
    """A span shorter than one CFL step is a single step too; a periodic first
    axis (stencils of the first planes wrap onto the last) takes the plain path."""
    g = hj.create_grid((0.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0), (50, 20, 24),
                       periodic_axes={0} if periodic0 else set())
    g = hj.with_boundary(g, 1, hj.dirichlet(0.25))
    cfg = hj.advection_term_config([1.0, -0.5, 0.25], scheme="weno5")
    x = g.axis_nodes[0][:, None, None]
    y0 = np.sin(x) + 0.1 * np.cos(3 * g.axis_nodes[1][None, :, None]) + 0 * g.axis_nodes[2][None, None, :]
    fi = FusedIntegrator(g, cfg)
    t, y, steps, mn, mx = fi.integrate_host(3, (0.0, 1e-3), y0, hj.IntegratorOptions())
    ref = FusedIntegrator(g, cfg).integrate(3, (0.0, 1e-3), dev.to_dev(y0), hj.IntegratorOptions())
    assert steps == 1 == ref.steps_taken and t == ref.t_final
    assert np.array_equal(y, dev.to_host(ref.y))
    assert (fi.launches == 3) == periodic0


def test_4d_single_step(small_pipeline):
    g = hj.di4_grid((41, 14, 17, 18))
    y0 = hj.di4_target(g).values
    a, b = _both(g, hj.di4_term_config(scheme="weno5"), y0, 3, hj.IntegratorOptions(single_step=True))
    assert np.array_equal(a[1], b[1])


def test_public_api_uses_pipeline(small_pipeline):
    """ode_cfl_3 on a host ScalarField (single step) through the pipeline
    equals the oracle-pinned device path."""
    g = hj.air3d_grid((41, 43, 36))
    cfg = hj.air3d_term_config(scheme="weno5")
    y0 = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    opts = hj.IntegratorOptions(single_step=True)
    res = hj.ode_cfl_3(hj.lax_friedrichs_rhs(g), (0.0, 1.0), y0, opts, cfg)
    ref = FusedIntegrator(g, cfg).integrate(3, (0.0, 1.0), dev.to_dev(y0.values), opts)
    assert np.array_equal(res.y_final.values, dev.to_host(ref.y))


def test_plane_range_validation():
    g = hj.air3d_grid((40, 20, 18))
    cfg = hj.air3d_term_config(scheme="weno5")
    fi = FusedIntegrator(g, cfg)
    y = dev.to_dev(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values)
    out = y.clone()
    a = _lib.doubles(fi._alphas(0.0, None), _lib.HJ_MAX_DIM)
    with pytest.raises(ValueError, match="multiples of 8"):
        dev.stage_dev(fi.dg, "weno5", fi.dh, a, 1e-3, _lib.STAGE_EULER, y, None, out, planes=(4, 16))
