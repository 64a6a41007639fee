"""C1: host issue time of one interval's native stage loop vs its device time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import time
import numpy as np
import torch
import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.engine import FusedIntegrator

g = hj.air3d_grid((51, 51, 36))
cfg = hj.air3d_term_config(scheme="eno2")
y = dev.to_dev(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values)
fi = FusedIntegrator(g, cfg)
opts = hj.IntegratorOptions()
for _ in range(3):
    fi.integrate(2, (0.0, 0.35), y, opts, check=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.record()
    r = fi.integrate(2, (0.0, 0.35), y, opts, check=False)
    t1 = time.perf_counter()
    e.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res.append((t1 - t0, t2 - t0, s.elapsed_time(e) / 1e3, r.steps_taken))
for h, w, d, n in res:
    print(f"host issue {h*1e3:.3f} ms, wall {w*1e3:.3f} ms, device {d*1e3:.3f} ms, {2*n} stages -> "
          f"{h/(2*n)*1e6:.2f} us/stage issue, {d/(2*n)*1e6:.2f} us/stage device")
