"""Compute-only cost of the pipelined host->host step's launch schedule at
301^3: the same plane-range stage launches, streams, priorities and event
dependencies as engine.FusedIntegrator._pipelined_step, without the copies
(the input is already on the device).  Compared with the one-launch-per-stage
device step, it separates schedule overhead from the PCIe floor."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import time
import numpy as np
import torch

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import _lib
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.engine import FusedIntegrator, pipeline_plan, _STAGES

g = hj.air3d_grid(301)
cfg = hj.air3d_term_config(scheme="weno5")
y = dev.to_dev(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values)
opts = hj.IntegratorOptions(single_step=True)
fi = FusedIntegrator(g, cfg)
kinds = _STAGES[3]
bufs = [y] + [torch.empty_like(y) for _ in kinds]
alphas_c = _lib.doubles(fi._alphas(0.0, None), _lib.HJ_MAX_DIM)
dt = 1e-3


def sched(chunk, prio, ranged=True):
    sts = [torch.cuda.Stream(priority=-k if prio else 0) for k in range(len(kinds))]
    comp = torch.cuda.current_stream()
    for st in sts:
        st.wait_stream(comp)
    last = [None] * (len(kinds) + 1)
    plan = pipeline_plan(301, len(kinds), chunk) if ranged else [("stage", k, 0, 301) for k in range(3)]
    for op, k, lo, hi in plan:
        if op != "stage":
            continue
        st = sts[k]
        if last[k] is not None:
            st.wait_event(last[k])
        kind = kinds[k]
        dev.stage_dev(fi.dg, fi.scheme, fi.dh, alphas_c, dt, kind, bufs[k], y if kind != _lib.STAGE_EULER else None,
                      bufs[k + 1], None, _lib.MASK_NONE, fi.stats, k, lib=fi.lib, strm=st.cuda_stream,
                      planes=(lo, hi))
        last[k + 1] = torch.cuda.Event()
        last[k + 1].record(st)
    for st in sts:
        comp.wait_stream(st)


def t(fn, reps=9):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return float(np.median(out))


sched(16, True)
print("one launch per stage (planes 0..301) ms", t(lambda: sched(16, True, ranged=False)), flush=True)
for c in (8, 16, 32, 64):
    for prio in (False, True):
        n = sum(1 for p in pipeline_plan(301, 3, c) if p[0] == "stage")
        print("chunk", c, "priority", prio, "launches", n, "ms", t(lambda: sched(c, prio)), flush=True)
