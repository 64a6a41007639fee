"""Device timeline of the pipelined host->host RK3 step at 301^3 (the e2e
leg of bench.py): the same schedule as FusedIntegrator._pipelined_step, with
a timing event after every H2D chunk, stage launch and D2H chunk, printed as
(op, stage, planes, start ms, end ms) relative to the first H2D.  Shows the
fill, the drain and where the copy engines or the SMs idle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import time  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import _lib  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402
from paper_2411_03501_b200.engine import _STAGES, FusedIntegrator, pipeline_plan  # noqa: E402

n = int(os.environ.get("N", "301"))
g = hj.air3d_grid(n)
cfg = hj.air3d_term_config(scheme="weno5")
host = torch.empty(g.counts, dtype=torch.float64, pin_memory=True)
host.copy_(torch.from_numpy(hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values))
fi = FusedIntegrator(g, cfg)
opts = hj.IntegratorOptions(single_step=True)
fi.integrate_host(3, (0.0, 1.0), host.numpy(), opts)   # warm (allocates the pipeline buffers)


def run(chunk, first, drain, ramp=0, tail=0, prio=True):
    kinds = _STAGES[3]
    shape = tuple(g.counts)
    bufs = [torch.empty(shape, dtype=dev.F64, device=dev.device()) for _ in range(4)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    s_st = [torch.cuda.Stream(priority=-k if prio else 0) for k in range(3)]
    out_host = torch.empty(shape, dtype=dev.F64, pin_memory=True)
    y_dev = bufs[0]
    alphas_c = _lib.doubles(fi._alphas(0.0, None), _lib.HJ_MAX_DIM)
    dt = 0.5 * float(1.0 / np.sum(cfg.partials.alphas(0.0, g) / g.spacings))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(s_in)
    for st in (s_out, *s_st):
        st.wait_stream(s_in)
    rec = []
    last_ev = [None] * 4
    h0 = time.perf_counter()
    for op, k, lo, hi in pipeline_plan(shape[0], 3, chunk, first=first, drain=drain, ramp=ramp, tail=tail):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if op == "h2d":
            a.record(s_in)
            with torch.cuda.stream(s_in):
                y_dev[lo:hi].copy_(host[lo:hi], non_blocking=True)
            b.record(s_in)
            last_ev[0] = b
        elif op == "stage":
            st = s_st[k]
            st.wait_event(last_ev[k])
            a.record(st)
            dev.stage_dev(fi.dg, fi.scheme, fi.dh, alphas_c, dt, kinds[k], bufs[k],
                          y_dev if kinds[k] != _lib.STAGE_EULER else None, bufs[k + 1], None, _lib.MASK_NONE,
                          fi.stats, k, lib=fi.lib, strm=st.cuda_stream, planes=(lo, hi))
            b.record(st)
            last_ev[k + 1] = b
        else:
            s_out.wait_event(last_ev[-1])
            a.record(s_out)
            with torch.cuda.stream(s_out):
                out_host[lo:hi].copy_(bufs[-1][lo:hi], non_blocking=True)
            b.record(s_out)
        rec.append((op, k, lo, hi, a, b))
    host_ms = (time.perf_counter() - h0) * 1e3
    torch.cuda.synchronize()
    rows = [(op, k, lo, hi, t0.elapsed_time(a), t0.elapsed_time(b)) for op, k, lo, hi, a, b in rec]
    run.host_ms = host_ms
    return rows


ref = fi.integrate_host(3, (0.0, 1.0), host.numpy(), opts)[1].copy()
shapes = [(16, 16, 16, 0, 0), (16, 11, 8, 2, 24), (24, 11, 8, 2, 24), (32, 11, 8, 2, 24), (32, 11, 8, 2, 40),
          (24, 19, 8, 1, 16), (32, 19, 8, 1, 32), (24, 11, 16, 2, 16), (48, 11, 8, 2, 24)]
best = None
for chunk, first, drain, ramp, tail in shapes:
    run(chunk, first, drain, ramp, tail)
    tot = []
    for _ in range(3):
        rows = run(chunk, first, drain, ramp, tail)
        tot.append(max(r[5] for r in rows))
    # the same plan through the public path (host wall clock, median of 9)
    fi.pipeline_chunk, fi.pipeline_first, fi.pipeline_drain = chunk, first, drain
    fi.pipeline_ramp, fi.pipeline_tail = ramp, tail
    same = np.array_equal(fi.integrate_host(3, (0.0, 1.0), host.numpy(), opts)[1], ref)
    wall = []
    for _ in range(9):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fi.integrate_host(3, (0.0, 1.0), host.numpy(), opts)
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
    busy = {}
    for op, k, lo, hi, s0, e in rows:
        key = op if op != "stage" else f"stage{k}"
        busy[key] = busy.get(key, 0.0) + (e - s0)
    first_d2h = min(r[4] for r in rows if r[0] == "d2h")
    last_h2d = max(r[5] for r in rows if r[0] == "h2d")
    print(f"# chunk {chunk} first {first} drain {drain} ramp {ramp} tail {tail}: device {min(tot):.3f} ms, "
          f"integrate_host {np.median(wall):.3f} ms, bit-identical {same}; first d2h {first_d2h:.3f}, "
          f"last h2d end {last_h2d:.3f}; host issue {run.host_ms:.3f} ms ({len(rows)} ops); busy " + ", ".join(f"{k} {v:.2f}" for k, v in busy.items()), flush=True)
    if best is None or min(tot) < best[0]:
        best = (min(tot), rows)
for op, k, lo, hi, s0, e in best[1]:
    print(f"{op:5s} {k:2d} [{lo:3d},{hi:3d})  {s0:7.3f} -> {e:7.3f}")
