"""Benchmark of the HJ grid-update hot path (BASELINE.json metric):

    fp64 grid cell-updates/s per RK stage, % of HBM roofline, 1/2/4/8 GPU

one line per BASELINE config (``--config``, default c2 = configs[1], the
headline):

  c1  Air3D 51x51x36, ENO2 + LF + odeCFL2, t in [0, 2.8], 8 intervals
      (configs[0]); a step = one full-horizon tube solve (632 RK2 steps);
  c2  Air3D 301^3 WENO5 + LF + TVD-RK3 (configs[1]); a step = one RK3 step
      (three fused stage launches); N GPUs: weak scaling, 301 planes per rank;
  c3  Air3D 801^3, the same path slab-decomposed over N GPUs (strong scaling;
      NCCL halo exchange of 3 planes per stage overlapped with the interior);
  c4  4-D double-integrator pair 121^4 WENO5 + RK3, slabs over N GPUs (strong);
  c5  8 Air3D 101^3 problems per GPU (the flock: 64 on 8 GPUs, replicas).

value = cells x stages x K / (device time of K steps, CUDA events, max over
ranks).  Launch: ``python bench.py [--config cK] [--gpus N] [--steps K]
[--warmup W] [--impl ours|reference]``; with ``--gpus N > 1`` and no
torchrun environment the script re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU) and refuses to run on
fewer GPUs.  Rank 0 prints ONE JSON line.  The reference arm
(``--impl reference``) times the CPU restatement of the reference
(oracle/, C, all host threads) on the same config (a bounded sample where the
config is too large for a CPU run; the line says which).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 grid cell-updates/sec per RK stage (WENO5+LF+RK3), % of HBM roofline, 1/2/4/8 GPU"
UNIT = "cell-updates/s"
CONFIGS = ("c1", "c2", "c3", "c4", "c5")
# algorithmic bytes per node and stage: stage 1 reads y and writes (16 B), the
# combination stages also read y0 (24 B) -- SURVEY 8(d)
BYTES_RK3 = (16 + 24 + 24) / 3.0
BYTES_RK2 = (16 + 24) / 2.0
L2_BYTES = 126 * 2**20


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=CONFIGS)
    ap.add_argument("--size", dest="n", type=int, default=None, help="override the nodes per axis of the config (tests)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tolerance-mode", action="store_true", help="skip the weno5_fma side measurement")
    ap.add_argument("--no-overlap", action="store_true", help="slabs: exchange, then the whole stage (A/B)")
    ap.add_argument("--scheme", default=None, choices=["weno5", "weno5_fma", "eno2"],
                    help="override the config's scheme (weno5_fma: tolerance mode, hjb200.h)")
    return ap.parse_args(argv)


# ----------------------------------------------------------------- multi-rank launch
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: one process per GPU through
    torch.distributed.run, or a loud failure when the box has fewer GPUs."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, this host has {have}", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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
            # nvidia-smi takes ~0.1-0.3 s to start: the timed region begins once it samples
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.005)
            self.n_before = len(self.lines)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            # a timed region shorter than the 20 ms period still gets the sample that follows it
            t0 = time.perf_counter()
            while len(self.lines) <= self.n_before and time.perf_counter() - t0 < 2.0:
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines[max(0, getattr(self, "n_before", 1) - 1):]:
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


# ----------------------------------------------------------------- peaks / FP64 accounting
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak(lib, stream):
    """Measured FP64-pipe throughput (DFMA lane-ops/s) from hj_fp64_probe:
    148*8 CTAs x 256 threads x 8 independent DFMA chains."""
    import torch

    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = 148 * 8, 4096
    lib.hj_fp64_probe(iters, blocks, sink.data_ptr(), stream)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.hj_fp64_probe(iters, blocks, sink.data_ptr(), stream)
    e.record()
    torch.cuda.synchronize()
    return blocks * 256 * iters * 8 / (s.elapsed_time(e) / 1e3)


def sass_hash(symbol: str) -> str | None:
    """sha256 of the SASS of one kernel (full mangled ``symbol``) in the
    loaded library (cuobjdump -fun): the FP64 op count below was measured by
    ncu on exactly this code, or it is reported stale."""
    from paper_2411_03501_b200 import _lib

    try:
        out = subprocess.run(["cuobjdump", "-sass", "-fun", symbol, _lib.library_path()], capture_output=True,
                             text=True, timeout=120).stdout
    except Exception:
        return None
    import re

    h = hashlib.sha256()
    n = 0
    for line in out.splitlines():
        # "/*0a30*/   DFMA R4, R2, R6, R8 ;   /* 0x... */": keep the instruction text only
        body = re.sub(r"/\*[^*]*\*/", "", line).strip()
        if re.match(r"^[@A-Z]", body) and not body.startswith(("Fatbin", "Function")):
            h.update(body.encode())
            n += 1
    return h.hexdigest() if n > 100 else None


_PARAMS = {"(StageArgs, int)": "NS_9StageArgsEi", "(StageArgs)": "NS_9StageArgsE",
           "(StageArgs, AxesScratch)": "NS_9StageArgsENS_11AxesScratchE",
           "(StageArgs, PersistArgs)": "NS_9StageArgsENS_11PersistArgsE"}


def kernel_symbol(kernel: str) -> str:
    """'void k_axis_col<3, 4, 4, 0>(StageArgs, AxesScratch)' (ncu's name) ->
    '_ZN2hj10k_axis_colILi3ELi4ELi4ELi0EEEvNS_9StageArgsENS_11AxesScratchE'"""
    import re

    m = re.search(r"(\w+)<([^>]*)>(\(.*\))", kernel)
    if m:
        base, targs, params = m.group(1), [a.strip() for a in m.group(2).split(",")], m.group(3)
        frag = base + "I" + "".join(f"Li{a}E" for a in targs) + "E"
    else:
        m = re.search(r"(\w+)(\(.*\))", kernel)
        base, params, frag = m.group(1), m.group(2), m.group(1)
    params = params.replace("hj::", "")
    return f"_ZN2hj{len(base)}{frag}Ev{_PARAMS.get(params, 'NS_9StageArgsE')}"


def fp64_ops(key: str):
    """ncu-measured FP64 ops per node-stage of the kernel (profiles/fp64_ops.json,
    written by scripts/fp64_stamp.py) -- trusted only if the stamped SASS hash
    still matches the loaded library."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_ops.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None, "no profiles/fp64_ops.json"
    ent = d.get(key)
    if not isinstance(ent, dict) and key.startswith("c3_"):
        ent = d.get("c2_" + key[3:])   # C3 runs the C2 kernel (same instantiation; the SASS hash is checked)
    if not isinstance(ent, dict):
        return None, f"no entry {key}"
    # one kernel per stage (brick) or the stage's kernel sequence (per-axis walk pipeline)
    for k in ent.get("kernels", [ent]):
        now = sass_hash(k.get("symbol", ""))
        if now is None or now != k.get("sass_sha256"):
            return None, f"stale: SASS of {k.get('kernel')} changed since the ncu count ({ent.get('source')})"
    return float(ent["ops_per_node"]), ent.get("source")


# ----------------------------------------------------------------- configs
class Workload:
    """One BASELINE config on this rank: grid, term config, initial state and
    the per-step device work."""

    def __init__(self, name: str, args, rank: int, world: int):
        import paper_2411_03501_b200 as hj

        self.name, self.rank, self.world = name, rank, world
        self.hj = hj
        self.scheme = args.scheme or ("eno2" if name == "c1" else "weno5")
        self.order = 2 if name == "c1" else 3
        self.batch = 1
        self.scaling = "weak"
        self.slabbed = False
        if name == "c1":
            n = args.n or 51
            self.grid = hj.air3d_grid((n, n, 36) if args.n is None else n)
            self.cfg = hj.air3d_term_config(scheme=self.scheme)
            self.workload = f"Air3D {'x'.join(map(str, self.grid.counts))} ENO2+LF+odeCFL2, t in [0,2.8], 8 intervals " \
                            "(configs[0]); a step = one full-horizon tube solve"
            self.scaling = "weak"
        elif name in ("c2", "c3"):
            n = args.n or (301 if name == "c2" else 801)
            if name == "c2":
                self.grid = hj.air3d_grid((n * world, n, n))
                self.workload = f"Air3D {n}^3 per GPU WENO5+LF+TVD-RK3 (configs[1]); a step = one RK3 step"
                self.scaling = "weak"
            else:
                self.grid = hj.air3d_grid(n)
                self.workload = f"Air3D {n}^3 WENO5+LF+TVD-RK3 slab-decomposed over {world} GPU(s) (configs[2]); " \
                                "a step = one RK3 step"
                self.scaling = "strong"
            self.cfg = hj.air3d_term_config(scheme=self.scheme)
            self.slabbed = world > 1
        elif name == "c4":
            n = args.n or 121
            self.grid = hj.di4_grid(n)
            self.cfg = hj.di4_term_config(scheme=self.scheme)
            self.workload = f"4-D double-integrator pair {n}^4 WENO5+LF+TVD-RK3 slab-decomposed over {world} " \
                            "GPU(s) (configs[3]); a step = one RK3 step"
            self.scaling = "strong"
            self.slabbed = world > 1
        else:   # c5
            n = args.n or 101
            self.grid = hj.air3d_grid(n)
            self.cfg = hj.air3d_term_config(scheme=self.scheme)
            self.batch = 8
            self.workload = f"batch of 8 Air3D {n}^3 WENO5+LF+TVD-RK3 problems per GPU (configs[4]: 64 on 8 GPUs, " \
                            "replicas, no exchange); a step = one RK3 step of the batch"
            self.scaling = "weak"
        alphas = self.cfg.partials.alphas(0.0, self.grid)
        self.dt = 0.5 * (1.0 / float(np.sum(alphas / self.grid.spacings)))
        self.bytes_per_node_stage = BYTES_RK2 if self.order == 2 else BYTES_RK3

    # -- targets (the same initial fields the tests use)
    def target(self, b: int = 0) -> np.ndarray:
        hj = self.hj
        if self.name == "c4":
            return hj.di4_target(self.grid).values
        if self.name == "c5":
            rng = np.random.default_rng(0)
            for k in range(b + 1):
                cx, cy = rng.uniform(-3.0, 3.0, 2)
                r = rng.uniform(3.0, 7.0)
            return hj.cylinder(self.grid, 2, (cx, cy, 0.0), r).values
        return hj.cylinder(self.grid, 2, (0.0, 0.0, 0.0), 5.0).values


def rank_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------- CPU oracle (baseline / reference arm)
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import spec_grid
    from hams import oracle_ham
    from oracle import hjoracle as orc

    return orc, spec_grid, oracle_ham


def oracle_unit(name: str, threads: int, n: int | None = None):
    """One unit of CPU work on config ``name`` through the oracle (C
    restatement of the reference, ``threads`` host threads): returns
    (seconds, cell-stages, sample description)."""
    orc, spec_grid, oracle_ham = _oracle()
    orc.set_threads(threads)
    if name == "c1":
        n = n or 51
        spec = dict(mins=[-6.0, -10.0, 0.0], maxs=[20.0, 10.0, 2 * math.pi], counts=[n, n, 36], periodic=[2],
                    dirichlet={})
        g = spec_grid(spec)
        tgt = orc.shape(g, 1, [0.0, 0.0, 0.0, 5.0, 4])
        t0 = time.perf_counter()
        _, _, steps = orc.solve_brt(g, oracle_ham("air3d", g), "eno2", tgt, 2.8, 8, order=2)
        secs = time.perf_counter() - t0
        return secs, 2 * sum(steps) * int(np.prod(g.counts)), f"full-horizon C1 tube ({sum(steps)} RK2 steps)"
    if name == "c4":
        n = n or 61
        spec = dict(mins=[-8.0, -8.0, -4.0, -4.0], maxs=[8.0, 8.0, 4.0, 4.0], counts=[n] * 4, periodic=[],
                    dirichlet={})
        g = spec_grid(spec)
        tgt = orc.shape(g, 1, [0.0, 0.0, 0.0, 0.0, 2.0, 12])
        t0 = time.perf_counter()
        orc.integrate(g, oracle_ham("di4", g), "weno5", 3, (0.0, 1.0), tgt, single_step=True)
        return time.perf_counter() - t0, 3 * n ** 4, f"one RK3 step of the 4-D pair on {n}^4"
    n = n or {"c2": 301, "c3": 401, "c5": 101}[name]
    spec = dict(mins=[-6.0, -10.0, 0.0], maxs=[20.0, 10.0, 2 * math.pi], counts=[n, n, n], periodic=[2],
                dirichlet={})
    g = spec_grid(spec)
    tgt = orc.shape(g, 1, [0.0, 0.0, 0.0, 5.0, 4])
    t0 = time.perf_counter()
    orc.integrate(g, oracle_ham("air3d", g), "weno5", 3, (0.0, 1.0), tgt, single_step=True)
    return time.perf_counter() - t0, 3 * n ** 3, f"one RK3 step of Air3D WENO5 on {n}^3"


# sizes the CPU runs at: the config's own size where a CPU step fits in a few
# seconds, else a smaller grid of the same per-node work (stated in the line)
CPU_SIZE = {"c1": None, "c2": None, "c3": 401, "c4": 61, "c5": None}


def cpu_baseline(name: str, threads: int, budget_s: float = 10.0):
    secs, work, steps, what = 0.0, 0, 0, ""
    while secs < budget_s and steps < 64:
        s, w, what = oracle_unit(name, threads, CPU_SIZE[name])
        secs += s
        work += w
        steps += 1
    return {"value": work / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{steps} x [{what}] ({secs:.1f} s) through oracle/hjoracle.c (C restatement of the "
                      f"reference, {threads} threads); per-node work is size-independent"}


def run_reference(args):
    world, rank, _ = rank_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    name = args.config
    size = CPU_SIZE[name] if args.n is None else args.n
    for _ in range(args.warmup):
        oracle_unit(name, threads, size)
    secs, work, what = 0.0, 0, ""
    for _ in range(args.steps):
        s, w, what = oracle_unit(name, threads, size)
        secs += s
        work += w
    value = work / secs
    same = size is None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{name}: {what}" + ("" if same else " (the config's per-node work on a CPU-sized grid)"),
                   "config": name, "same_size_as_ours": same, "parallelism": f"cpu threads ({threads})"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"each step = {what} via oracle/hjoracle.c ({threads} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2411_03501_b200 import _lib
    from paper_2411_03501_b200 import device as dev
    from paper_2411_03501_b200.engine import FusedIntegrator

    world, rank, local = rank_env()
    ndev = torch.cuda.device_count()
    shared = os.environ.get("HJ_SLAB_COMM") == "torch"   # 1-GPU path check: ranks share a GPU, gloo-staged halos
    if world > ndev and not shared:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, this host has {ndev}")
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        # torch.distributed is plumbing only (barriers, the NCCL unique id, the
        # max over ranks); the halo data plane is libhjb200's own NCCL
        # communicator (hj_dd_*), whose init lines NCCL_DEBUG=INFO prints
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo")
    lib = _lib.load()
    W = Workload(args.config, args, rank, world)
    g, cfg = W.grid, W.cfg
    stream = torch.cuda.current_stream()
    ev_stage = []
    overlap = not args.no_overlap

    # ---- the runner of this rank
    if W.slabbed:
        from paper_2411_03501_b200.distributed import SlabIntegrator

        runner = SlabIntegrator(g, cfg, rank, world, transport=None if shared else "nccl", overlap=overlap)
        y = runner.scatter(W.target())
        cells_local = runner.owned_cells
    elif W.name == "c2" and world > 1:
        # weak scaling: this rank owns 301 planes of a (301 N) x 301 x 301 grid
        from paper_2411_03501_b200.distributed import SlabIntegrator

        runner = SlabIntegrator(g, cfg, rank, world, transport=None if shared else "nccl", overlap=overlap)
        y = runner.init_cylinder(5.0)
        cells_local = runner.owned_cells
        W.slabbed = True
    elif W.batch > 1:
        dgb = dev.DeviceGrid(g, batch=W.batch)
        runner = FusedIntegrator(g, cfg, dg=dgb)
        y = dev.to_dev(np.stack([W.target(b) for b in range(W.batch)]))
        cells_local = W.batch * int(np.prod(g.counts))
    else:
        runner = FusedIntegrator(g, cfg)
        y = dev.to_dev(W.target())
        cells_local = int(np.prod(g.counts))
    total_cells = cells_local * world

    # ---- one step of device work
    if W.name == "c1":
        opts = W.hj.IntegratorOptions()
        target_dev = y
        stages_per_step = 0

        def step(y, t, timed=False):
            # the full-horizon tube from the resident target: 8 intervals, the
            # native loop per interval, the mask in each interval's last stage
            prev, t0 = target_dev, 0.0
            nst = 0
            for k in range(1, 9):
                t1 = 2.8 * k / 8
                r = runner.integrate(2, (t0, t1), prev, opts, mask_prev=prev, use_min=True, check=False)
                prev, t0 = r.y, t1
                nst += 2 * r.steps_taken
            W.c1_stages = nst
            return prev
    else:
        def step(y, t, timed=False):
            return runner.step3(y, t, W.dt, events=ev_stage if timed else None)

    flush = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device="cuda") if W.name in ("c1", "c5") else None
    t = 0.0
    for _ in range(args.warmup):
        y = step(y, t)
        t += W.dt
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides, device events, max over ranks
    launches0 = _lib.launch_count()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    gpu_index = int(vis.split(",")[local]) if vis else local
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    with ClockSampler(gpu_index) as clk:
        if flush is None:
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for _ in range(args.steps):
                y = step(y, t, timed=True)
                t += W.dt
            end.record(stream)
            torch.cuda.synchronize()
            ms = start.elapsed_time(end)
        else:
            # small working sets: L2 flushed between timed steps (outside the events)
            pairs = []
            for _ in range(args.steps):
                flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                y = step(y, t, timed=True)
                b.record(stream)
                pairs.append((a, b))
                t += W.dt
            torch.cuda.synchronize()
            step_ms = [a.elapsed_time(b) for a, b in pairs]
            ms = float(sum(step_ms))
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    stages_per_step = W.c1_stages if W.name == "c1" else 3
    value = total_cells * stages_per_step * args.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (the fused stage)
    peak, peak_src = measured_peaks()
    bytes_per_launch = W.bytes_per_node_stage * cells_local
    stage_ms = [a.elapsed_time(b) for a, b in ev_stage]
    if stage_ms:
        mean_stage_s = float(np.mean(stage_ms)) / 1e3
        stage_src = "mean of per-stage CUDA events on the launching stream"
    else:
        mean_stage_s = (ms / 1e3) / (stages_per_step * args.steps)
        stage_src = "device time of the timed steps / stages (launch-bound small grid)"
    achieved = bytes_per_launch / mean_stage_s / 1e9
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(
            f"{args.config}_{W.scheme}_{world}")
    except Exception:
        traffic = None

    # ---- FP64-pipe accounting (the binding roofline for WENO5)
    fp64 = None
    if rank == 0 and world == 1:
        peak64 = fp64_peak(lib, stream.cuda_stream)
        ops, src = fp64_ops(f"{args.config}_{W.scheme}")
        fp64 = {"peak_ops_per_s": peak64, "peak_source": "measured: hj_fp64_probe DFMA chains, this run",
                "ops_per_unit": ops, "ops_source": src}
        if ops:
            fp64["achieved_ops_per_s"] = value * ops
            fp64["frac"] = value * ops / peak64

    # ---- end to end through the public API (host buffers, copies inside the timed region)
    e2e = e2e_pageable = None
    if args.e2e_steps > 0:
        e2e, e2e_pageable = measure_e2e(W, runner, y, t, args, world, total_cells)

    # ---- tolerance mode beside the exact headline (c2 only)
    tol = None
    if (world == 1 and args.config == "c2" and W.scheme == "weno5" and not args.no_tolerance_mode):
        tol = tolerance_mode(W, y, args, cells_local, bytes_per_launch, peak, fp64)

    comm = None
    if W.slabbed and hasattr(runner.transport, "traffic"):
        ex, by = runner.transport.traffic()
        comm = {"transport": "hj_dd (libhjb200 NCCL communicator)", "nccl_version": int(lib.hj_dd_nccl_version()),
                "exchanges": ex, "halo_bytes_sent": by, "overlap": overlap}
    elif W.slabbed:
        comm = {"transport": type(runner.transport).__name__, "overlap": overlap}
    del runner
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, os.cpu_count() or 1)
    l2 = (f"inputs larger than L2 ({8 * cells_local / 2**20:.0f} MiB per field vs 126 MB L2)"
          if flush is None else "L2 flushed between timed steps (252 MB write outside the events)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": W.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W.workload, "config": args.config,
                   "grid": list(g.counts), "batch_per_gpu": W.batch, "scheme": W.scheme,
                   "integrator": f"ode_cfl_{W.order}", "cfl": 0.5,
                   "parallelism": (f"slab{world} (NCCL halo exchange, hj_dd)" if W.slabbed else
                                   (f"replicas{world}" if world > 1 else "single")),
                   "stages_per_step": stages_per_step, "l2": l2},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": "hj_stage fused LF+RK stage",
                     "bytes_per_launch": bytes_per_launch, "bytes_per_node": W.bytes_per_node_stage,
                     "launch_time": stage_src,
                     "note": "fp64 WENO5 is FP64-pipe bound (SURVEY 0.4); see the fp64 block"},
        "fp64": fp64,
        "tolerance_mode": tol,
        "clocks": clk.summary(),
        "e2e": e2e,
        "e2e_pageable": e2e_pageable,
        "gpu_launches": launches,
        "cpu_baseline": cpu,
        "comm": comm,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_e2e(W, runner, y, t, args, world, total_cells):
    """The same metric through the public API with host buffers: every step
    copies its input from host memory to the device and its result back,
    inside the timed region.  Returns (pinned-input e2e, pageable-input e2e)."""
    import torch
    import torch.distributed as dist

    hj = W.hj
    from paper_2411_03501_b200 import device as dev

    K = args.e2e_steps
    cells_one = int(np.prod(W.grid.counts))
    if W.name == "c1":
        target = hj.ScalarField(W.target())
        hj.solve_tube(W.grid, target, W.cfg, 2.8, 8, order=2)    # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            hj.solve_tube(W.grid, target, W.cfg, 2.8, 8, order=2)
        secs = time.perf_counter() - t0
        stages = W.c1_stages
        return ({"value": cells_one * stages * K / secs, "unit": UNIT, "h2d_bytes_per_step": 8 * cells_one,
                 "d2h_bytes_per_step": 8 * cells_one * 8,
                 "api": "solve_tube(grid, ScalarField(host target), cfg, 2.8, 8, order=2): host target in, the 8 "
                        "interval snapshots out"}, None)
    if W.name == "c5":
        targets = [W.target(b) for b in range(W.batch)]
        hj.solve_tube_batch(W.grid, targets, W.cfg, W.dt, 1, keep_snapshots=False)   # warm
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            hj.solve_tube_batch(W.grid, targets, W.cfg, W.dt, 1, keep_snapshots=False)
        secs = _max_over_ranks(time.perf_counter() - t0, world)
        return ({"value": total_cells * 3 * K / secs, "unit": UNIT,
                 "h2d_bytes_per_step": 8 * W.batch * cells_one, "d2h_bytes_per_step": 8 * W.batch * cells_one,
                 "api": "per rank: solve_tube_batch(grid, 8 host targets, cfg, dt, 1) = one RK3 step of the batch, "
                        "host targets in, host result out; max over ranks"}, None)
    if not W.slabbed:
        rhs = hj.lax_friedrichs_rhs(W.grid)
        one = hj.IntegratorOptions(cfl_factor=0.5, single_step=True)
        pinned = torch.empty(W.grid.counts, dtype=torch.float64, pin_memory=True)
        pinned.copy_(y.cpu())
        out = []
        for label, arr in (("pinned", pinned.numpy()), ("pageable", np.array(pinned.numpy()))):
            field = hj.ScalarField(arr)
            hj.ode_cfl_3(rhs, (t, t + 1.0), field, one, W.cfg)    # warm the path
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(K):
                res = hj.ode_cfl_3(rhs, (t, t + 1.0), field, one, W.cfg)
                del res
            torch.cuda.synchronize()
            secs = time.perf_counter() - t0
            out.append({"value": total_cells * 3 * K / secs, "unit": UNIT,
                        "h2d_bytes_per_step": 8 * total_cells, "d2h_bytes_per_step": 8 * total_cells,
                        "api": f"ode_cfl_3(lax_friedrichs_rhs(g), ..., ScalarField({label} host array), "
                               "single_step) per step"})
        return out[0], out[1]
    # slabs: each rank's owned planes H2D (pinned), one RK3 step of its slab
    # (hj_dd halo exchange overlapped), owned planes D2H; max over ranks
    host_in = torch.empty(runner.owned(y).shape, dtype=torch.float64, pin_memory=True)
    host_in.copy_(runner.owned(y).cpu())
    host_out = torch.empty_like(host_in, pin_memory=True)
    buf = runner.empty()

    def e2e_step():
        runner.owned(buf).copy_(host_in, non_blocking=True)
        yo = runner.step3(buf, t, W.dt)
        host_out.copy_(runner.owned(yo), non_blocking=True)
        torch.cuda.current_stream().synchronize()

    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        e2e_step()
    secs = _max_over_ranks(time.perf_counter() - t0, world)
    return ({"value": total_cells * 3 * K / secs, "unit": UNIT,
             "h2d_bytes_per_step": 8 * total_cells, "d2h_bytes_per_step": 8 * total_cells,
             "api": "per rank: owned planes H2D (pinned), SlabIntegrator.step3 (hj_dd_stage: NCCL halo exchange "
                    "overlapped with the interior), owned planes D2H; max over ranks"}, None)


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def tolerance_mode(W, y, args, cells_local, bytes_per_launch, peak, fp64):
    """The same workload in tolerance mode (HJ_WENO5_FMA), reported beside the
    bit-exact headline, not instead of it: the full-horizon C2 tube is too
    ill-conditioned for any non-bit-exact evaluation to hold 1e-9
    (profiles/r01_fma_conditioning.txt)."""
    import torch

    from paper_2411_03501_b200.engine import FusedIntegrator

    cfg_f = W.hj.air3d_term_config(scheme="weno5_fma")
    run_f = FusedIntegrator(W.grid, cfg_f)
    yf = y.clone()
    tf = 0.0
    for _ in range(args.warmup):
        yf = run_f.step3(yf, tf, W.dt)
        tf += W.dt
    ev_f = []
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        yf = run_f.step3(yf, tf, W.dt, events=ev_f)
        tf += W.dt
    s1.record()
    torch.cuda.synchronize()
    ms_f = s0.elapsed_time(s1)
    v_f = cells_local * 3 * args.steps / (ms_f / 1e3)
    st_f = float(np.mean([a.elapsed_time(b) for a, b in ev_f])) / 1e3
    ops_f, _ = fp64_ops("c2_weno5_fma")
    return {"scheme": "weno5_fma", "value": v_f, "unit": UNIT, "ms_per_step": ms_f / args.steps,
            "roofline_frac": bytes_per_launch / st_f / 1e9 / peak, "fp64_ops_per_unit": ops_f,
            "fp64_frac": (v_f * ops_f / fp64["peak_ops_per_s"]) if (ops_f and fp64) else None,
            "parity": "within 1e-9 where the solve is conditioned for it (51^3/101^3 full horizon: <= 8e-12); at "
                      "301^3 full horizon within the exact path's own 1-ulp input sensitivity "
                      "(tests/test_gpu_weno_fma.py)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
