"""Host-side tests of the experiment runner (cli.py) and the snapshot format --
the reference's test_cli_io.py cases that need no solve, plus the benchmark
problems' config handling and the background snapshot writer.  No GPU."""
import json
import struct

import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import cli, snapshot
from paper_2411_03501_b200.cli import ConfigError, load_config, main, run_experiment


class TestSnapshotFormat:
    # test_cli_io.py:12-67
    def test_round_trip_bit_exact(self, tmp_path):
        g = hj.create_grid((0, 0, 0), (1, 1, 1), (4, 5, 6))
        f = hj.ScalarField(np.random.default_rng(12).standard_normal(g.counts))
        hj.export_field(f, g, tmp_path / "field.f64")
        back, shape = hj.import_field(tmp_path / "field.f64")
        assert shape == (4, 5, 6) and np.array_equal(back.values, f.values)

    def test_file_size_arithmetic(self, tmp_path):
        g = hj.create_grid((0, 0, 0), (1, 1, 1), (41, 41, 41))
        hj.export_field(hj.ScalarField(np.zeros(g.counts)), g, tmp_path / "field.f64")
        assert (tmp_path / "field.f64").stat().st_size == 16 + 3 * 8 + 41 ** 3 * 8

    def test_truncated_payload_reports_byte_counts(self, tmp_path):
        g = hj.create_grid((0,), (1,), (8,))
        path = tmp_path / "field.f64"
        hj.export_field(hj.ScalarField(np.arange(8.0)), g, path)
        path.write_bytes(path.read_bytes()[:-8])
        with pytest.raises(ValueError, match=r"expected 88 bytes .* got 80"):
            hj.import_field(path)

    def test_bad_magic_and_version(self, tmp_path):
        path = tmp_path / "field.f64"
        path.write_bytes(b"NOPE" + struct.pack("<III", 1, 1, 0) + struct.pack("<Q", 1) + struct.pack("<d", 0.0))
        with pytest.raises(ValueError, match="magic"):
            hj.import_field(path)
        path.write_bytes(b"HJLS" + struct.pack("<III", 9, 1, 0) + struct.pack("<Q", 1) + struct.pack("<d", 0.0))
        with pytest.raises(ValueError, match="version"):
            hj.import_field(path)

    def test_shape_mismatch_on_export(self, tmp_path):
        g = hj.create_grid((0,), (1,), (8,))
        with pytest.raises(ValueError, match="match"):
            hj.export_field(hj.ScalarField(np.zeros(5)), g, tmp_path / "x.f64")

    def test_header_layout(self, tmp_path):
        g = hj.create_grid((0, 0), (1, 1), (3, 2))
        path = tmp_path / "field.f64"
        hj.export_field(hj.ScalarField(np.arange(6.0).reshape(3, 2)), g, path)
        raw = path.read_bytes()
        assert struct.unpack_from("<4sIII", raw) == (b"HJLS", 1, 2, 0)
        assert struct.unpack_from("<2Q", raw, 16) == (3, 2)
        assert np.frombuffer(raw, dtype="<f8", offset=32).tolist() == list(range(6))

    def test_export_array_matches_export_field(self, tmp_path):
        g = hj.create_grid((0, 0), (1, 1), (5, 3))
        f = hj.ScalarField(np.random.default_rng(1).standard_normal(g.counts))
        hj.export_field(f, g, tmp_path / "a")
        snapshot.export_array(f.values, tmp_path / "b")
        assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()

    def test_batched_array_round_trip(self, tmp_path):
        vals = np.random.default_rng(2).standard_normal((3, 4, 5, 6))
        snapshot.export_array(vals, tmp_path / "batch.f64")
        back, shape = hj.import_field(tmp_path / "batch.f64")
        assert shape == (3, 4, 5, 6) and np.array_equal(back.values, vals)


class TestSnapshotWriter:
    def test_writes_in_order_and_waits(self, tmp_path):
        rng = np.random.default_rng(5)
        arrays = [rng.standard_normal((7, 9)) for _ in range(6)]
        with snapshot.SnapshotWriter() as w:
            for k, a in enumerate(arrays):
                w.submit(a, tmp_path / f"v{k}.f64")
        for k, a in enumerate(arrays):
            back, _ = hj.import_field(tmp_path / f"v{k}.f64")
            assert np.array_equal(back.values, a)

    def test_write_failure_surfaces_on_close(self, tmp_path):
        w = snapshot.SnapshotWriter()
        w.submit(np.zeros(3), tmp_path / "missing_dir" / "x.f64")
        with pytest.raises(OSError):
            w.close()


def write_config(tmp_path, **overrides):
    cfg = {"problem": "rockets", "resolution": 11, "horizon": 0.5, "global_steps": 3, "scheme": "eno2"}
    cfg.update(overrides)
    path = tmp_path / "config.json"
    path.write_text(json.dumps(cfg))
    return path


class TestConfig:
    # test_cli_io.py:82-127
    def test_missing_file_is_exit_2(self, tmp_path, capsys):
        assert run_experiment(tmp_path / "nope.json", tmp_path / "out") == 2
        assert "nope.json" in capsys.readouterr().err

    def test_invalid_json_names_line(self, tmp_path):
        path = tmp_path / "config.json"
        path.write_text('{"problem": "rockets",\n  "resolution": }\n')
        with pytest.raises(ConfigError, match="line 2"):
            load_config(path)

    def test_top_level_must_be_object(self, tmp_path):
        path = tmp_path / "config.json"
        path.write_text("[1, 2]")
        with pytest.raises(ConfigError, match="JSON object"):
            load_config(path)

    def test_unknown_problem(self, tmp_path):
        path = tmp_path / "config.json"
        path.write_text('{"problem": "heat"}')
        with pytest.raises(ConfigError, match="unknown problem"):
            load_config(path)

    def test_unknown_key(self, tmp_path):
        with pytest.raises(ConfigError, match="typo_key"):
            load_config(write_config(tmp_path, typo_key=3))

    def test_weno5_on_8_node_axis_rejected_before_solving(self, tmp_path, capsys):
        path = write_config(tmp_path, resolution=8, scheme="weno5")
        assert run_experiment(path, tmp_path / "out") == 2
        assert "weno5" in capsys.readouterr().err
        assert not (tmp_path / "out" / "value_0000.f64").exists()

    def test_weno5_on_9_nodes_accepted(self, tmp_path):
        assert load_config(write_config(tmp_path, resolution=9, scheme="weno5"))["resolution"] == 9

    def test_overrides_replace_config_values(self, tmp_path):
        cfg = load_config(write_config(tmp_path), overrides={"global_steps": 5, "scheme": "first", "cfl": None})
        assert cfg["global_steps"] == 5 and cfg["scheme"] == "first" and cfg["cfl"] == 0.5

    @pytest.mark.parametrize("key,value,match", [
        ("global_steps", 0, "global_steps"), ("horizon", 0.0, "horizon"), ("cfl", 1.5, "cfl"),
        ("scheme", "weno7", "unknown scheme"),
    ])
    def test_value_checks(self, tmp_path, key, value, match):
        with pytest.raises(ConfigError, match=match):
            load_config(write_config(tmp_path, **{key: value}))

    def test_bad_scheme_flag_is_usage_error(self, tmp_path):
        with pytest.raises(SystemExit) as e:
            main(["solve", "--config", str(write_config(tmp_path)), "--out", str(tmp_path), "--scheme", "x"])
        assert e.value.code == 2


class TestBenchmarkProblems:
    def test_defaults_are_the_baseline_configs(self, tmp_path):
        path = tmp_path / "c.json"
        path.write_text('{"problem": "air3d"}')
        cfg = load_config(path)
        assert cli._counts(cfg) == [51, 51, 36]   # C1
        assert (cfg["scheme"], cfg["order"], cfg["global_steps"], cfg["horizon"]) == ("eno2", 2, 8, 2.8)
        path.write_text('{"problem": "air3d_batch"}')
        cfg = load_config(path)
        assert cli._counts(cfg) == [101, 101, 101] and cfg["batch"] == 8   # C5, one GPU's share

    def test_resolution_sets_every_axis(self, tmp_path):
        path = tmp_path / "c.json"
        path.write_text('{"problem": "di4"}')
        assert cli._counts(load_config(path, {"resolution": 121})) == [121] * 4   # C4
        path.write_text('{"problem": "air3d", "scheme": "weno5", "order": 3}')
        assert cli._counts(load_config(path, {"resolution": 301})) == [301] * 3   # C2

    @pytest.mark.parametrize("cfg,match", [
        ({"problem": "air3d", "counts": [20, 20, 8], "scheme": "weno5"}, "periodic axis"),
        ({"problem": "air3d", "counts": [20, 20]}, "3 axis counts"),
        ({"problem": "di4", "counts": [9, 9, 9, 1]}, "at least 2 nodes"),
        ({"problem": "di4", "order": 4}, "order"),
        ({"problem": "air3d_batch", "batch": 0}, "batch"),
    ])
    def test_validation(self, tmp_path, cfg, match):
        path = tmp_path / "c.json"
        path.write_text(json.dumps(cfg))
        with pytest.raises(ConfigError, match=match):
            load_config(path)
