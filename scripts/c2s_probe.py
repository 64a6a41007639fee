"""Where does the public-API time of a C2 tube slice go?  cProfile of
solve_tube on Air3D 301^3 (horizon 0.02, 4 intervals) after a warm-up."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03501_b200 as hj  # noqa: E402

g = hj.air3d_grid(301)
cfg = hj.air3d_term_config(scheme="weno5")
target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
hj.solve_tube(g, target, cfg, 0.005, 1)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = hj.solve_tube(g, target, cfg, 0.02, 4)
torch.cuda.synchronize()
pr.disable()
print("total", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
