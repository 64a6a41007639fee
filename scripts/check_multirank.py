"""End-to-end check of the multi-rank slab path (what `bench.py --gpus N`
runs), with N ranks sharing the available GPU(s):

    torchrun --standalone --nproc-per-node 2 scripts/check_multirank.py [--backend gloo|nccl]

Each rank advances its slab of a decomposed Air3D grid through
SlabIntegrator (halo exchange every stage through torch.distributed), rank 0
gathers the owned planes and compares them bit for bit with a single-domain
run.  With one GPU use gloo (halos staged through the host; no kernel ever
waits on another); on a multi-GPU box use nccl.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_03501_b200 as hj  # noqa: E402
from paper_2411_03501_b200 import device as dev  # noqa: E402
from paper_2411_03501_b200.distributed import SlabIntegrator  # noqa: E402
from paper_2411_03501_b200.engine import FusedIntegrator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--planes", type=int, default=61)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tube", action="store_true",
                    help="full tube solve (solve_tube_slabs, snapshots gathered to rank 0) vs solve_tube")
    ap.add_argument("--scheme", default="weno5")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group(args.backend)
    if args.tube:
        return tube(args, rank, world)
    g = hj.air3d_grid((args.planes * world, 40, 36))
    cfg = hj.air3d_term_config(scheme="weno5")
    y0 = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0).values
    alphas = cfg.partials.alphas(0.0, g)
    dt = 0.5 / float(np.sum(alphas / g.spacings))
    run = SlabIntegrator(g, cfg, rank, world)
    y = run.scatter(y0)
    t = 0.0
    for _ in range(args.steps):
        y = run.step3(y, t, dt)
        t += dt
    mine = torch.from_numpy(dev.to_host(run.owned(y)).copy())
    parts = [torch.empty((s.n,) + tuple(g.counts[1:]), dtype=torch.float64)
             for s in __import__("paper_2411_03501_b200.distributed", fromlist=["partition"]).partition(
                 g.counts[0], world, 3, g.is_periodic(0))]
    dist.all_gather(parts, mine) if args.backend == "gloo" else None
    if args.backend != "gloo":
        gathered = [torch.empty_like(p, device="cuda") for p in parts]
        dist.all_gather(gathered, mine.cuda())
        parts = [p.cpu() for p in gathered]
    if rank == 0:
        single = FusedIntegrator(g, cfg)
        ys = dev.to_dev(y0)
        t = 0.0
        for _ in range(args.steps):
            ys = single.step3(ys, t, dt)
            t += dt
        ref = dev.to_host(ys)
        got = np.concatenate([p.numpy() for p in parts], axis=0)
        ok = np.array_equal(ref, got)
        print(f"multirank world={world} backend={args.backend}: bitwise_equal={ok}", flush=True)
        if not ok:
            sys.exit(1)
    dist.destroy_process_group()


def tube(args, rank, world):
    from paper_2411_03501_b200.distributed import solve_tube_slabs

    g = hj.air3d_grid((args.planes * world, 34, 30))
    cfg = hj.air3d_term_config(scheme=args.scheme)
    target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
    seen = []
    res = solve_tube_slabs(g, target, cfg, 0.5, 3, order=3, progress=lambda k, t, v: seen.append(k))
    if rank == 0:
        ref = hj.solve_tube(g, target, cfg, 0.5, 3, order=3)
        ok = tuple(res.times) == tuple(ref.times) and seen == [1, 2, 3] and len(res.snapshots) == 4
        ok = ok and all(np.array_equal(a.values, b.values) for a, b in zip(res.snapshots, ref.snapshots))
        print(f"multirank tube world={world} backend={args.backend} scheme={args.scheme}: bitwise_equal={ok}",
              flush=True)
        if not ok:
            sys.exit(1)
    else:
        assert res.snapshots == () and len(res.times) == 4
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
