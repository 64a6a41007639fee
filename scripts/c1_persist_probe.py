"""C1 (Air3D 51x51x36 ENO2 + odeCFL2, full horizon [0, 2.8], 8 intervals):
device time of one tube under the persistent integration (default dispatch)
and under per-stage launches of the generic kernel, bitwise compared."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402

g = hj.air3d_grid((51, 51, 36))
cfg = hj.air3d_term_config(scheme="eno2")
target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
res = {}
for v in sys.argv[1:] or ["auto", "generic"]:
    old = dev.set_stage_kernel(v)
    r = hj.solve_tube(g, target, cfg, 2.8, 8, order=2)
    times = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = hj.solve_tube(g, target, cfg, 2.8, 8, order=2)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    res[v] = [s.values for s in r.snapshots]
    dev.set_stage_kernel(old)
    print(f"{v:10s} tube {np.median(times):.3f} ms (wall, median of 5)", flush=True)
ks = list(res)
for k in ks[1:]:
    print(k, "bitwise vs", ks[0], all(np.array_equal(a, b) for a, b in zip(res[ks[0]], res[k])))
