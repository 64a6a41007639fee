"""Benchmark of the HJ grid-update hot path (BASELINE.json metric):

    fp64 grid cell-updates/s per RK stage, WENO5 + Lax-Friedrichs + TVD-RK3,
    Air3D 301^3 (configs[1]) on one B200; weak-scaled slabs on N GPUs.

A "step" is one TVD-RK3 time step = three fused stage kernels over the whole
grid.  value = cells * 3 * K / (device time of K steps, max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  The reference arm (--impl reference) times
the CPU restatement of the reference (oracle/, C, all host threads) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 grid cell-updates/sec per RK stage (WENO5+LF+RK3), % of HBM roofline, 1/2/4/8 GPU"
UNIT = "cell-updates/s"
N_AIR3D = 301
# algorithmic bytes per node for one RK3 step: stage 1 reads y, writes y1 (16 B);
# stages 2 and 3 read the stage input and y0 and write (24 B each) -- SURVEY 8(d)
BYTES_PER_NODE_STEP = 16 + 24 + 24


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_AIR3D, help="nodes per axis (default 301 = configs[1])")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tolerance-mode", action="store_true", help="skip the weno5_fma side measurement")
    ap.add_argument("--scheme", default="weno5", choices=["weno5", "weno5_fma"],
                    help="weno5: bit-exact with the reference; weno5_fma: tolerance mode (<= 1e-9, hjb200.h)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak(dev, lib):
    """Measured FP64-pipe throughput (DFMA lane-ops/s) from hj_fp64_probe:
    148*8 CTAs x 256 threads x 8 independent DFMA chains."""
    import torch

    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = 148 * 8, 4096
    lib.hj_fp64_probe(iters, blocks, sink.data_ptr(), dev.stream())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.hj_fp64_probe(iters, blocks, sink.data_ptr(), dev.stream())
    e.record()
    torch.cuda.synchronize()
    return blocks * 256 * iters * 8 / (s.elapsed_time(e) / 1e3)


def fp64_ops_per_node(key: str):
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_ops.json")) as fh:
            d = json.load(fh)
        return d.get(key), d.get("source")
    except Exception:
        return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------- CPU oracle timing (baseline / reference arm)
def oracle_rk3_step(n: int, threads: int):
    """One TVD-RK3 step of Air3D WENO5 on an n^3 grid through the oracle.
    Returns (seconds, cell-stages)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import spec_grid
    from hams import oracle_ham
    from oracle import hjoracle as orc

    orc.set_threads(threads)
    spec = dict(mins=[-6.0, -10.0, 0.0], maxs=[20.0, 10.0, 2 * math.pi], counts=[n, n, n], periodic=[2],
                dirichlet={})
    g = spec_grid(spec)
    ham = oracle_ham("air3d", g)
    target = orc.shape(g, 1, [0.0, 0.0, 0.0, 5.0, 4])
    t0 = time.perf_counter()
    orc.integrate(g, ham, "weno5", 3, (0.0, 1.0), target, single_step=True)
    return time.perf_counter() - t0, 3 * n ** 3


def cpu_baseline(threads: int, budget_s: float = 10.0):
    n = 161
    secs, work, steps = 0.0, 0, 0
    while secs < budget_s and steps < 128:
        s, w = oracle_rk3_step(n, threads)
        secs += s
        work += w
        steps += 1
    return {"value": work / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{steps} TVD-RK3 step(s) ({secs:.1f} s) of Air3D WENO5+LF on {n}^3 through oracle/hjoracle.c "
                      f"(C restatement of the reference, {threads} threads); per-node work is size-independent"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = 201
    for _ in range(args.warmup):
        oracle_rk3_step(n, threads)
    secs, work = 0.0, 0
    for _ in range(args.steps):
        s, w = oracle_rk3_step(n, threads)
        secs += s
        work += w
    value = work / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"Air3D {N_AIR3D}^3 WENO5+LF+TVD-RK3 (sampled at {n}^3 on CPU)",
                   "grid": [n, n, n], "scheme": "weno5", "integrator": "ode_cfl_3", "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"each step = one TVD-RK3 step of Air3D WENO5 on {n}^3 via oracle/hjoracle.c"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2411_03501_b200 as hj
    from paper_2411_03501_b200 import _lib
    from paper_2411_03501_b200 import device as dev
    from paper_2411_03501_b200.engine import FusedIntegrator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()   # (ranks may share a GPU in the gloo path check)
    torch.cuda.set_device(local)
    backend = os.environ.get("HJ_DIST_BACKEND", "nccl")   # gloo only for 1-GPU path checks
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    n = args.n
    cfg = hj.air3d_term_config(scheme=args.scheme)
    if world > 1:
        from paper_2411_03501_b200.distributed import SlabIntegrator

        g = hj.air3d_grid((n * world, n, n))
        runner = SlabIntegrator(g, cfg, rank, world)
        y = runner.init_cylinder(5.0)
        cells_local = runner.owned_cells
    else:
        g = hj.air3d_grid(n)
        runner = FusedIntegrator(g, cfg)
        dg = runner.dg
        y = dev.init_shape_dev(dg, _lib.SHAPE_CYLINDER, [0.0, 0.0, 0.0, 5.0, 4.0])
        cells_local = dg.cells
    opts = hj.IntegratorOptions(cfl_factor=0.5)
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 * (1.0 / float(np.sum(alphas / g.spacings)))

    stream = torch.cuda.current_stream()
    ev_stage = []

    def step(y, t, timed=False):
        return runner.step3(y, t, dt, events=ev_stage if timed else None)

    t = 0.0
    for _ in range(args.warmup):
        y = step(y, t)
        t += dt
    torch.cuda.synchronize()

    # timed region: K steps, barrier + sync on both sides, device events, max over ranks
    launches0 = _lib.launch_count()
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES") else local
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(gpu_index) as clk:
        start.record(stream)
        for _ in range(args.steps):
            y = step(y, t, timed=True)
            t += dt
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    ms = start.elapsed_time(end)
    stage_ms = [a.elapsed_time(b) for a, b in ev_stage]
    if world > 1:
        tt = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    total_cells = cells_local * world
    value = total_cells * 3 * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (the fused stage): algorithmic bytes per launch / mean launch time
    peak, peak_src = measured_peaks()
    bytes_per_launch = BYTES_PER_NODE_STEP / 3.0 * cells_local
    mean_stage_s = float(np.mean(stage_ms)) / 1e3 if stage_ms else (ms / 1e3) / (3 * args.steps)
    achieved = bytes_per_launch / mean_stage_s / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get(f"air3d_{args.scheme}_{n}")
        except Exception:
            traffic = None

    # end to end through the public API: host ScalarField in (pinned), host ScalarField out, every step
    e2e = None
    if world == 1 and args.e2e_steps > 0:
        host = torch.empty(g.counts, dtype=torch.float64, pin_memory=True)
        host.copy_(y.cpu())
        y_host = hj.ScalarField(host.numpy())
        rhs = hj.lax_friedrichs_rhs(g)
        one = hj.IntegratorOptions(cfl_factor=0.5, single_step=True)
        hj.ode_cfl_3(rhs, (t, t + 1.0), y_host, one, cfg)   # warm the path
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            # the same pinned host input each step: H2D in, 3 fused stages, D2H out
            res = hj.ode_cfl_3(rhs, (t, t + 1.0), y_host, one, cfg)
            del res
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        e2e = {"value": total_cells * 3 * args.e2e_steps / secs, "unit": UNIT,
               "h2d_bytes_per_step": 8 * total_cells, "d2h_bytes_per_step": 8 * total_cells,
               "api": "ode_cfl_3(lax_friedrichs_rhs(g), ..., ScalarField(host), single_step) per step"}
    elif world > 1 and args.e2e_steps > 0:
        # every rank: its owned planes H2D from pinned host memory, one RK3 step of
        # its slab (distributed.SlabIntegrator, halo exchange overlapped), its owned
        # planes D2H; barrier on both sides, max over ranks
        host_in = torch.empty(runner.owned(y).shape, dtype=torch.float64, pin_memory=True)
        host_in.copy_(runner.owned(y).cpu())
        host_out = torch.empty_like(host_in, pin_memory=True)
        buf = runner.empty()

        def e2e_step():
            runner.owned(buf).copy_(host_in, non_blocking=True)
            yo = runner.step3(buf, t, dt)
            host_out.copy_(runner.owned(yo), non_blocking=True)
            torch.cuda.current_stream().synchronize()

        e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        secs = time.perf_counter() - t0
        st = torch.tensor([secs], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        secs = float(st.item())
        e2e = {"value": total_cells * 3 * args.e2e_steps / secs, "unit": UNIT,
               "h2d_bytes_per_step": 8 * total_cells, "d2h_bytes_per_step": 8 * total_cells,
               "api": "per rank: owned planes H2D (pinned), distributed.SlabIntegrator.step3, owned planes D2H; "
                      "max over ranks"}

    # the binding roofline: FP64 pipe -- ops/node from the committed ncu count
    fp64 = None
    ops, src = fp64_ops_per_node(f"air3d_{args.scheme}_{os.environ.get('HJ_STAGE_KERNEL', 'brick')}")
    if world == 1:
        peak64 = fp64_peak(dev, _lib.load())
        fp64 = {"peak_ops_per_s": peak64, "peak_source": "measured: hj_fp64_probe DFMA chains, this run",
                "ops_per_unit": ops, "ops_source": src}
        if ops:
            fp64["achieved_ops_per_s"] = value * ops
            fp64["frac"] = value * ops / peak64
    # the same workload in tolerance mode (HJ_WENO5_FMA): reported beside the
    # bit-exact headline, not instead of it -- the full-horizon C2 tube is too
    # ill-conditioned for any non-bit-exact evaluation to hold 1e-9
    # (profiles/r01_fma_conditioning.txt)
    tol = None
    if world == 1 and args.scheme == "weno5" and not args.no_tolerance_mode:
        cfg_f = hj.air3d_term_config(scheme="weno5_fma")
        run_f = FusedIntegrator(g, cfg_f)
        yf = y.clone()
        tf = 0.0
        for _ in range(args.warmup):
            yf = run_f.step3(yf, tf, dt)
            tf += dt
        ev_f = []
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            yf = run_f.step3(yf, tf, dt, events=ev_f)
            tf += dt
        s1.record(stream)
        torch.cuda.synchronize()
        ms_f = s0.elapsed_time(s1)
        v_f = total_cells * 3 * args.steps / (ms_f / 1e3)
        st_f = float(np.mean([a.elapsed_time(b) for a, b in ev_f])) / 1e3
        ops_f, _ = fp64_ops_per_node("air3d_weno5_fma_brick")
        tol = {"scheme": "weno5_fma", "value": v_f, "unit": UNIT, "ms_per_step": ms_f / args.steps,
               "roofline_frac": bytes_per_launch / st_f / 1e9 / peak,
               "fp64_ops_per_unit": ops_f,
               "fp64_frac": (v_f * ops_f / fp64["peak_ops_per_s"]) if (ops_f and fp64) else None,
               "parity": "within 1e-9 where the solve is conditioned for it (51^3/101^3 full horizon: "
                         "<= 8e-12); at 301^3 full horizon within the exact path's own 1-ulp input "
                         "sensitivity (tests/test_gpu_weno_fma.py)"}
        del yf, run_f
    if rank != 0:
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(os.cpu_count() or 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"Air3D {n}^3 per GPU, WENO5 + Lax-Friedrichs (GLF) + TVD-RK3 (configs[1])",
                   "grid": [n * world, n, n], "scheme": args.scheme, "integrator": "ode_cfl_3", "cfl": 0.5,
                   "parallelism": f"slab{world}" if world > 1 else "single",
                   "l2": f"inputs larger than L2 ({8 * cells_local / 2**20:.0f} MiB per field vs 126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "kernel": "hj_stage fused WENO5+LF+RK stage",
                     "bytes_per_launch": bytes_per_launch,
                     "note": "fp64 WENO5 is FP64-pipe bound (SURVEY 0.4); see fp64 block"},
        "fp64": fp64,
        "tolerance_mode": tol,
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
