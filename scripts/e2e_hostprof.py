import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_03501_b200 as hj
from paper_2411_03501_b200.engine import FusedIntegrator
g = hj.air3d_grid(301)
cfg = hj.air3d_term_config(scheme="weno5")
host = torch.empty(g.counts, dtype=torch.float64, pin_memory=True)
host.copy_(torch.from_numpy(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values))
fi = FusedIntegrator(g, cfg)
opts = hj.IntegratorOptions(single_step=True)
for _ in range(3): fi.integrate_host(3, (0.0, 1.0), host.numpy(), opts)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): fi.integrate_host(3, (0.0, 1.0), host.numpy(), opts)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
