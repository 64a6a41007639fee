"""Where does the C1 time go?  Per-stage device time vs the whole solve."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.engine import FusedIntegrator

g = hj.air3d_grid((51, 51, 36))
cfg = hj.air3d_term_config(scheme="eno2")
target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
fi = FusedIntegrator(g, cfg)
y = dev.to_dev(target.values)
alphas = cfg.partials.alphas(0.0, g)
dt = 0.5 / float(np.sum(alphas / g.spacings))
ev = []
for _ in range(20):
    y = fi.step3(y, 0.0, dt, events=ev)
torch.cuda.synchronize()
stage_us = [a.elapsed_time(b) * 1e3 for a, b in ev[15:]]
opts = hj.IntegratorOptions()
torch.cuda.synchronize(); t0 = time.perf_counter()
r = fi.integrate(2, (0.0, 0.35), dev.to_dev(target.values), opts)
torch.cuda.synchronize(); one_interval = time.perf_counter() - t0
t0 = time.perf_counter()
res = hj.solve_tube(g, target, cfg, 2.8, 8, order=2)
torch.cuda.synchronize(); full = time.perf_counter() - t0
print(json.dumps({"kernel": os.environ.get("HJ_STAGE_KERNEL", "brick"), "stage_us_median": float(np.median(stage_us)),
                  "interval_s": one_interval, "interval_steps": r.steps_taken, "full_solve_s": full}))
