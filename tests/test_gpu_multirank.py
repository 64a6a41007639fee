"""The multi-process slab path end to end on one GPU: torchrun ranks over the
gloo backend (halos and the snapshot gather staged through the host, so no
kernel ever waits on another rank's kernel), full tube solve with snapshots
gathered to rank 0, compared bit for bit with the single-GPU tube
(scripts/check_multirank.py --tube)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,scheme", [(2, "weno5"), (3, "eno2")])
def test_tube_over_slabs_equals_single_gpu(world, scheme):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(world),
           os.path.join(ROOT, "scripts", "check_multirank.py"), "--backend", "gloo", "--tube", "--planes", "12",
           "--scheme", scheme]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "bitwise_equal=True" in r.stdout


def test_runner_under_torchrun_matches_single_gpu(tmp_path):
    """`torchrun -m paper_2411_03501_b200 solve` splits the tube across ranks;
    rank 0 writes snapshot files byte-identical to a one-process run."""
    import json

    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"problem": "air3d", "counts": [26, 24, 20], "horizon": 0.4, "global_steps": 2,
                               "scheme": "weno5", "order": 3}))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    one = subprocess.run([sys.executable, "-m", "paper_2411_03501_b200", "solve", "--config", str(cfg), "--out",
                          str(tmp_path / "one")], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-4000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                          "-m", "paper_2411_03501_b200", "solve", "--config", str(cfg), "--out",
                          str(tmp_path / "two")], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert two.returncode == 0, two.stdout[-2000:] + two.stderr[-4000:]
    for k in range(3):
        name = f"value_{k:04d}.f64"
        assert (tmp_path / "one" / name).read_bytes() == (tmp_path / "two" / name).read_bytes(), name
    meta = json.loads((tmp_path / "two" / "meta.json").read_text())
    assert meta["config"]["ranks"] == 2
