"""Host-side logic of the package (no GPU needed): validation messages,
metadata, node tables, options -- mirrors the reference's own unit tests
(pkg/tests/test_grid.py, test_term.py, test_integrator.py,
test_reachability.py, test_cli_io.py) for everything that is not arithmetic
on the grid."""
import math
import os

import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from golden_io import case_list, package_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestGrid:
    def test_three_dim_periodic_spacings(self):
        g = hj.create_grid((-5, -5, -math.pi), (5, 5, math.pi), (41, 41, 41), periodic_axes={2})
        assert np.allclose(g.spacings, [0.25, 0.25, 2 * math.pi / 41])
        assert g.dim == 3 and g.num_nodes == 41 ** 3
        assert g.axis_nodes[2][0] == pytest.approx(-math.pi) and g.axis_nodes[2][-1] < math.pi

    def test_two_node_line(self):
        g = hj.create_grid((0,), (1,), (2,))
        assert np.array_equal(g.axis_nodes[0], [0.0, 1.0]) and g.spacings[0] == 1.0

    def test_periodic_exclusive_endpoint(self):
        g = hj.create_grid((0,), (1,), (4,), periodic_axes={0})
        assert np.allclose(g.axis_nodes[0], [0.0, 0.25, 0.5, 0.75]) and g.spacings[0] == 0.25

    @pytest.mark.parametrize("args,match", [
        (((0, 0), (1,), (5,)), "lengths differ"),
        (((0, 2), (1, 2), (5, 5)), "axis 1"),
        (((0, 0), (1, 1), (1, 5)), "axis 0"),
    ])
    def test_validation(self, args, match):
        with pytest.raises(ValueError, match=match):
            hj.create_grid(*args)

    def test_periodic_axis_out_of_range(self):
        with pytest.raises(ValueError, match="periodic axis"):
            hj.create_grid((0,), (1,), (5,), periodic_axes={3})

    def test_nodes_and_spacings_equal_reference(self):
        # node tables are host data consumed by the kernels: must be the reference's bits
        for meta, a in case_list("ghost.npz"):
            g = package_grid(meta["grid"])
            assert np.array_equal(g.spacings, a["spacings"])
            for ax in range(g.dim):
                assert np.array_equal(g.axis_nodes[ax], a[f"nodes{ax}"])

    def test_with_boundary(self):
        g = hj.create_grid((0,), (1,), (2,))
        g2 = hj.with_boundary(g, 0, hj.dirichlet(7.0))
        assert g2.boundary[0] == hj.BoundaryCondition("dirichlet", 7.0)
        with pytest.raises(ValueError, match="periodicity"):
            hj.with_boundary(g, 0, hj.periodic())
        with pytest.raises(ValueError, match="axis 3"):
            hj.with_boundary(g, 3, hj.extrapolate())
        with pytest.raises(ValueError, match="unknown boundary kind"):
            hj.BoundaryCondition("reflect")

    def test_mesh_coordinates(self):
        g = hj.create_grid((0, 0), (1, 1), (2, 2))
        assert np.array_equal(hj.mesh_coordinates(g, 1).flat, [0.0, 1.0, 0.0, 1.0])
        with pytest.raises(ValueError, match="axis 2"):
            hj.mesh_coordinates(g, 2)


class TestScalarField:
    def test_rejects_nonfinite(self):
        for bad in (np.array([1.0, np.nan]), np.array([np.inf, 0.0])):
            with pytest.raises(ValueError, match="non-finite"):
                hj.ScalarField(bad)

    def test_flat_shape(self):
        f = hj.ScalarField(np.arange(6.0), grid_shape=(2, 3))
        assert f.values.shape == (2, 3) and f.values[1, 0] == 3.0
        assert np.array_equal(f.flat, np.arange(6.0))
        with pytest.raises(ValueError, match="needs"):
            hj.ScalarField(np.arange(5.0), grid_shape=(2, 3))


class TestConfigs:
    def test_term_config_validation(self):
        with pytest.raises(ValueError, match="scheme"):
            hj.TermConfig(hamiltonian=lambda *a: None, partials=lambda *a: 0.0, derivative_scheme="spectral")
        with pytest.raises(ValueError, match="dissipation"):
            hj.TermConfig(hamiltonian=lambda *a: None, partials=lambda *a: 0.0, dissipation="local")
        with pytest.raises(ValueError, match="approximation_sign"):
            hj.TermConfig(hamiltonian=lambda *a: None, partials=lambda *a: 0.0, approximation_sign="sideways")

    def test_integrator_options(self):
        for kw, m in (({"cfl_factor": 0.0}, "cfl_factor"), ({"cfl_factor": 1.5}, "cfl_factor"),
                      ({"max_step": -1.0}, "max_step")):
            with pytest.raises(ValueError, match=m):
                hj.IntegratorOptions(**kw)

    def test_registered_configs_are_device_terms(self):
        assert hj.advection_term_config([1.0]).on_device
        assert hj.rockets_term_config(hj.RocketParams()).on_device
        assert hj.air3d_term_config().on_device and hj.di4_term_config().on_device
        assert not hj.TermConfig(hamiltonian=lambda *a: None, partials=lambda *a: 0.0).on_device

    def test_rocket_params_and_partials(self):
        with pytest.raises(ValueError, match="positive"):
            hj.RocketParams(a=0.0)
        with pytest.raises(ValueError, match="u_min < u_max"):
            hj.RocketParams(u_min=1.0, u_max=-1.0)
        g = hj.create_grid((-64, -64, -math.pi), (64, 64, math.pi), (9, 9, 9), periodic_axes={2})
        p = hj.RocketParams()
        assert [hj.rockets_partials(0.0, g, None, None, a, p) for a in range(3)] == [65.0, 96.0, 2.0]
        with pytest.raises(ValueError, match="axis 3"):
            hj.rockets_partials(0.0, g, None, None, 3, p)

    def test_rockets_oracle_scalar(self):
        p = hj.RocketParams()
        assert hj.rockets_hamiltonian_oracle(0.0, (1.0, 2.0, 0.3), (0, 0, 0), p) == 0.0
        assert hj.rockets_hamiltonian_oracle(0.0, (5.0, -3.0, 0.7), (0, 0, 1), p) == pytest.approx(0.0, abs=1e-15)

    def test_air3d_alphas_match_survey(self):
        g = hj.air3d_grid((51, 51, 36))
        a = hj.air3d_term_config().partials.alphas(0.0, g)
        assert np.allclose(a, [20.0, 25.0, 2.0])

    def test_reach_problem_validation(self):
        cfg = hj.rockets_term_config(hj.RocketParams())
        g2 = hj.create_grid((0, 0), (1, 1), (5, 5))
        with pytest.raises(ValueError, match="3-D"):
            hj.ReachProblem(grid=g2, target=hj.ScalarField(np.zeros(g2.counts)), params=hj.RocketParams(),
                            term_config=cfg, horizon=1.0, global_steps=2)
        g3 = hj.create_grid((-1, -1, -math.pi), (1, 1, math.pi), (5, 5, 5))
        with pytest.raises(ValueError, match="periodic"):
            hj.ReachProblem(grid=g3, target=hj.ScalarField(np.zeros(g3.counts)), params=hj.RocketParams(),
                            term_config=cfg, horizon=1.0, global_steps=2)


class TestSnapshot:
    def test_round_trip_and_layout(self, tmp_path):
        g = hj.create_grid((0, 0, 0), (1, 1, 1), (41, 41, 41))
        f = hj.ScalarField(np.random.default_rng(0).standard_normal(g.counts))
        p = tmp_path / "v.hjls"
        hj.export_field(f, g, p)
        assert os.path.getsize(p) == 16 + 24 + 41 ** 3 * 8
        back, shape = hj.import_field(p)
        assert shape == (41, 41, 41) and np.array_equal(back.values, f.values)
        raw = p.read_bytes()
        assert raw[:4] == b"HJLS"

    @pytest.mark.parametrize("mutate,match", [
        (lambda b: b[:10], "truncated header"), (lambda b: b"XXXX" + b[4:], "bad magic"),
        (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "version"), (lambda b: b[:-8], "expected")])
    def test_errors(self, tmp_path, mutate, match):
        g = hj.create_grid((0,), (1,), (5,))
        p = tmp_path / "v.hjls"
        hj.export_field(hj.ScalarField(np.arange(5.0)), g, p)
        p.write_bytes(mutate(p.read_bytes()))
        with pytest.raises(ValueError, match=match):
            hj.import_field(p)


def test_reference_names_exported():
    for name in hj.REFERENCE_ALL:
        assert hasattr(hj, name), name
    ref_init = "/root/reference/pkg/src/hjls/__init__.py"
    if os.path.exists(ref_init):
        import ast

        tree = ast.parse(open(ref_init).read())
        for node in tree.body:
            if isinstance(node, ast.Assign) and node.targets[0].id == "__all__":
                ref_all = [e.value for e in node.value.elts]
        assert sorted(ref_all) == sorted(hj.REFERENCE_ALL)


# ---------------------------------------------------------------- pipelined host->host step (engine.pipeline_plan)
@pytest.mark.parametrize("n0", [16, 17, 40, 61, 301, 801])
@pytest.mark.parametrize("stages", [1, 2, 3])
@pytest.mark.parametrize("chunk", [8, 16, 32, 48, 64])
@pytest.mark.parametrize("shape", [(16, 0, 0, 16), (11, 2, 24, 8), (5, 1, 100, 4), (40, 3, 8, 24)])
def test_pipeline_plan_covers_and_respects_dependencies(n0, stages, chunk, shape):
    from paper_2411_03501_b200.engine import pipeline_plan

    first, ramp, tail, drain = shape
    plan = pipeline_plan(n0, stages, chunk, first=first, ramp=ramp, tail=tail, drain=drain)
    arrived = 0
    done = [0] * stages
    copied = 0
    for op, k, lo, hi in plan:
        assert lo < hi
        if op == "h2d":
            assert lo == arrived
            arrived = hi
        elif op == "stage":
            assert lo == done[k] and lo % 8 == 0 and (hi % 8 == 0 or hi == n0)
            src_front = arrived if k == 0 else done[k - 1]
            # the launch reads planes [lo-3, hi+3) of its input: all produced
            # (beyond n0 they are boundary ghosts of a complete input)
            assert src_front == n0 or hi + 3 <= src_front
            done[k] = hi
        else:
            assert op == "d2h" and lo == copied and hi <= done[-1]
            copied = hi
    assert arrived == n0 and done == [n0] * stages and copied == n0


def test_compute_api_fails_loudly_without_cuda():
    """No CPU fallback: without a GPU every compute entry point raises."""
    import torch

    import paper_2411_03501_b200 as hj

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = hj.create_grid((0.0,), (1.0,), (16,))
    with pytest.raises(RuntimeError, match="CUDA"):
        hj.upwind_first_weno5(g, hj.ScalarField(np.linspace(0.0, 1.0, 16)), 0)


def test_bench_refuses_more_gpus_than_present():
    """bench.py --gpus N launches N ranks itself, and fails loudly (exit 2)
    when the host has fewer GPUs -- it never silently measures one."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "needs 2 CUDA devices" in r.stderr


def test_bench_config_table():
    import bench

    assert bench.CONFIGS == ("c1", "c2", "c3", "c4", "c5")
    assert bench.parse([]).config == "c2"
    assert abs(bench.BYTES_RK3 - 64 / 3) < 1e-12 and bench.BYTES_RK2 == 20.0
    assert bench.kernel_symbol("void k_stage_brick<3, 3, 2, 0, 2>(StageArgs, int)") == \
        "_ZN2hj13k_stage_brickILi3ELi3ELi2ELi0ELi2EEEvNS_9StageArgsEi"
    assert bench.kernel_symbol("void hj::k_axis_col<3, 4, 4, 0>(hj::StageArgs, hj::AxesScratch)") == \
        "_ZN2hj10k_axis_colILi3ELi4ELi4ELi0EEEvNS_9StageArgsENS_11AxesScratchE"
    assert bench.kernel_symbol("void k_axis_x<3>(StageArgs, AxesScratch)") == \
        "_ZN2hj8k_axis_xILi3EEEvNS_9StageArgsENS_11AxesScratchE"
