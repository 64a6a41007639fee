"""Golden outputs of the REFERENCE experiment runner (hjls.cli), run here only.

    python tests/golden/make_cli_golden.py [/root/reference]

Runs the reference's ``run_experiment`` / ``main`` (cli.py:226-296) on small
configurations -- the ones its own tests use (test_cli_io.py:70-79,
test_acceptance.py:249-262) plus WENO5 / advection variants -- and records,
per run, the SHA-256 of every snapshot file it wrote and its meta.json
(timings.json holds wall-clock numbers and is not compared).  The package's
runner (paper_2411_03501_b200.cli) must reproduce the snapshot files byte for
byte and the meta.json exactly; tests/test_gpu_cli.py checks that on the GPU.
Output: tests/golden/cli.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import load_reference  # noqa: E402

# name -> (config file contents, argv overrides for main(["solve", ...]) or None)
RUNS = {
    "rockets_eno2_r11": ({"problem": "rockets", "resolution": 11, "horizon": 0.5, "global_steps": 3,
                          "scheme": "eno2"}, None),
    "rockets_eno2_r15": ({"problem": "rockets", "resolution": 15, "horizon": 0.8, "global_steps": 4,
                          "scheme": "eno2"}, None),
    "rockets_weno5_r13": ({"problem": "rockets", "resolution": 13, "horizon": 0.3, "global_steps": 2,
                           "scheme": "weno5"}, None),
    "rockets_eno3_r12_cfl": ({"problem": "rockets", "resolution": 12, "horizon": 0.4, "global_steps": 2,
                              "scheme": "eno3", "cfl": 0.8}, None),
    "advection_weno5_r40": ({"problem": "advection", "resolution": 40, "speed": 1.0, "horizon": 0.5,
                             "global_steps": 2, "scheme": "weno5"}, None),
    "advection_defaults": ({"problem": "advection"}, None),
    "rockets_weno5_r31": ({"problem": "rockets", "resolution": 31, "horizon": 0.5, "global_steps": 3,
                           "scheme": "weno5"}, None),
    "rockets_defaults": ({"problem": "rockets"}, None),
    "main_overrides": ({"problem": "rockets", "resolution": 11, "horizon": 0.5, "global_steps": 3,
                        "scheme": "eno2"}, ["--steps", "2", "--scheme", "first"]),
}


def sha(path: Path) -> str:
    return hashlib.sha256(path.read_bytes()).hexdigest()


def run_all(ref) -> dict:
    from hjls_ref.cli import main, run_experiment

    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (cfg, argv) in RUNS.items():
            d = Path(tmp) / name
            d.mkdir()
            cfg_path = d / "config.json"
            cfg_path.write_text(json.dumps(cfg))
            dst = d / "out"
            if argv is None:
                status = run_experiment(cfg_path, dst)
            else:
                status = main(["solve", "--config", str(cfg_path), "--out", str(dst), *argv])
            assert status == 0, (name, status)
            meta = json.loads((dst / "meta.json").read_text())
            out[name] = {
                "config": cfg,
                "argv": argv,
                "files": {f: sha(dst / f) for f in meta["snapshots"]},
                "sizes": {f: (dst / f).stat().st_size for f in meta["snapshots"]},
                "meta": meta,
                "listing": sorted(p.name for p in dst.iterdir()),
            }
            print(f"{name}: {len(meta['snapshots'])} snapshots")
    return out


def main_() -> None:
    root = sys.argv[1] if len(sys.argv) > 1 else "/root/reference"
    ref = load_reference(root)
    res = run_all(ref)
    (HERE / "cli.json").write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
    print(f"wrote {HERE / 'cli.json'}")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONHASHSEED", "0")
    main_()
