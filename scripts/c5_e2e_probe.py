"""Where the C5 end-to-end call (solve_tube_batch of 8 Air3D 101^3 host
targets, one RK3 step, keep_snapshots=False) spends its time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import reachability as R  # noqa: E402

sys.path.insert(0, ROOT)
import bench  # noqa: E402

W = bench.Workload("c5", bench.parse([]), 0, 1)
targets = [W.target(b) for b in range(W.batch)]
hj.solve_tube_batch(W.grid, targets, W.cfg, W.dt, 1, keep_snapshots=False)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    hj.solve_tube_batch(W.grid, targets, W.cfg, W.dt, 1, keep_snapshots=False)
    ts.append((time.perf_counter() - t0) * 1e3)
print("solve_tube_batch ms", np.median(ts), ts)
fi, staging, pool = R._batch_runner(W.grid, W.cfg, len(targets))
st = staging.numpy()
for name, fn in [
    ("stage copies", lambda: [f.result() for f in [pool.submit(np.copyto, st[b], a) for b, a in enumerate(targets)]]),
    ("h2d", lambda: torch.empty(staging.shape, dtype=torch.float64, device="cuda").copy_(staging, non_blocking=True)),
]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, "ms", (time.perf_counter() - t0) * 1e3 / 5)
prev = torch.empty(staging.shape, dtype=torch.float64, device="cuda").copy_(staging)
opts = hj.IntegratorOptions()
torch.cuda.synchronize()
t0 = time.perf_counter()
res = fi.integrate(3, (0.0, W.dt), prev, opts, mask_prev=prev, use_min=True)
torch.cuda.synchronize()
print("integrate ms", (time.perf_counter() - t0) * 1e3, "steps", res.steps_taken, "dt W", W.dt)
t0 = time.perf_counter()
out = hj.device.to_host(res.y) if hasattr(hj, "device") else None
torch.cuda.synchronize()
print("to_host ms", (time.perf_counter() - t0) * 1e3)
t0 = time.perf_counter()
ok = bool(torch.isfinite(prev).all())
print("isfinite ms", (time.perf_counter() - t0) * 1e3)
