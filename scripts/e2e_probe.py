"""Where the end-to-end (host field in, host field out) single RK3 step spends
its time at 301^3: per-call setup, and the pipelined step per chunk size and
stream-priority setting."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import time
import numpy as np
import torch

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200.engine import FusedIntegrator

g = hj.air3d_grid(301)
cfg = hj.air3d_term_config(scheme="weno5")
host = torch.empty(g.counts, dtype=torch.float64, pin_memory=True)
host.copy_(torch.from_numpy(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values))
y = host.numpy()
opts = hj.IntegratorOptions(single_step=True)


def t(fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return float(np.median(out)) * 1e3


print("construct FusedIntegrator ms", t(lambda: FusedIntegrator(g, cfg)))
fi = FusedIntegrator(g, cfg)
fi.integrate_host(3, (0.0, 1.0), y, opts)
ref = fi.integrate_host(3, (0.0, 1.0), y, opts)[1].copy()
fi.pipeline_chunk = 16
for first in (8, 16):
    for drain in (8, 16, 32):
        fi.pipeline_first, fi.pipeline_drain = first, drain
        same = np.array_equal(fi.integrate_host(3, (0.0, 1.0), y, opts)[1], ref)
        print("chunk 16 first", first, "drain", drain, "ms",
              t(lambda: fi.integrate_host(3, (0.0, 1.0), y, opts), reps=9), "bit-identical", same, flush=True)
fi.pipeline_first, fi.pipeline_drain = 16, 16
for prio in (False, True):
    fi.pipeline_priority = prio
    for c in (8, 16, 24, 32):
        fi.pipeline_chunk = c
        same = np.array_equal(fi.integrate_host(3, (0.0, 1.0), y, opts)[1], ref)
        print("priority", prio, "chunk", c, "ms", t(lambda: fi.integrate_host(3, (0.0, 1.0), y, opts), reps=9),
              "bit-identical", same, flush=True)
fi.pipeline_min_cells = 1 << 40
print("unpipelined ms", t(lambda: fi.integrate_host(3, (0.0, 1.0), y, opts)))
rhs = hj.lax_friedrichs_rhs(g)
yf = hj.ScalarField(y)
print("public ode_cfl_3 ms", t(lambda: hj.ode_cfl_3(rhs, (0.0, 1.0), yf, opts, cfg)))
