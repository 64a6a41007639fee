"""A/B of the per-interval snapshot path: SnapshotPipe (worker-thread copy
overlapped with the next interval) vs a synchronous copy, on C1 (0.75 MB
fields, 8 intervals) and a C2 slice (218 MB fields)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import device as dev, reachability  # noqa: E402
from paper_2411_03501_b200.grid import ScalarField  # noqa: E402


class SyncPipe:
    """the synchronous alternative: dev.to_host (pinned for >= 1 MB) per interval"""

    def __init__(self, deliver):
        self.deliver = deliver

    def push(self, k, t, state):
        self.deliver(k, t, dev.to_host(state))

    def drain(self):
        pass

    def close(self):
        pass


def timed(g, cfg, target, horizon, steps, order, reps):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hj.solve_tube(g, target, cfg, horizon, steps, order=order)
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return float(np.median(out))


res = {}
cases = {
    "c1": (hj.air3d_grid((51, 51, 36)), "eno2", 2.8, 8, 2, 5),
    "c2_slice": (hj.air3d_grid(301), "weno5", 0.02, 4, 3, 2),
}
Pipe = reachability.SnapshotPipe
for name, (g, scheme, horizon, steps, order, reps) in cases.items():
    cfg = hj.air3d_term_config(scheme=scheme)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    hj.solve_tube(g, target, cfg, horizon / steps, 1, order=order)
    for label, cls in (("pipe", Pipe), ("sync", SyncPipe), ("pipe2", Pipe)):
        reachability.SnapshotPipe = cls
        res[f"{name}_{label}_s"] = timed(g, cfg, target, horizon, steps, order, reps)
reachability.SnapshotPipe = Pipe
print(json.dumps(res))
