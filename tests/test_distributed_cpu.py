"""Multi-rank plumbing of the slab decomposition on CPU (gloo, world 2-4):
partitioning, halo message plan and the exchange itself.  The kernels that
consume the halos are covered on the GPU by tests/test_gpu_distributed.py
(all slabs emulated on one device, bitwise against the single-domain run)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_03501_b200.distributed import TorchDistTransport, halo_plan, partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_balanced_and_validated():
    sl = partition(301, 4, 3, periodic=False)
    assert [s.n for s in sl] == [76, 75, 75, 75] and [s.lo for s in sl] == [0, 76, 151, 226]
    assert not sl[0].has_lo and sl[0].has_hi and sl[-1].has_lo and not sl[-1].has_hi
    sp = partition(10, 2, 3, periodic=True)
    assert all(s.has_lo and s.has_hi for s in sp)
    with pytest.raises(ValueError, match="too few"):
        partition(5, 4, 3, periodic=False)
    single = partition(7, 1, 3, periodic=True)[0]
    assert not single.has_lo and not single.has_hi


def test_halo_plan_pairs_messages_for_two_periodic_slabs():
    a, b = partition(10, 2, 3, periodic=True)
    sa, ra = halo_plan(a)
    sb, rb = halo_plan(b)
    # k-th send from a to b must land in b's k-th receive from a
    for (pa, (s0, s1)), (pb, (r0, r1)) in zip(sa, rb):
        assert pa == 1 and pb == 0
    # a's first owned planes -> b's upper halo; a's last owned planes -> b's lower halo
    assert sa[0][1] == (3, 6) and rb[0][1] == (b.n + 3, b.n + 6)
    assert sa[1][1] == (a.n, a.n + 3) and rb[1][1] == (0, 3)


def _worker(rank, world, port, n0, periodic, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        full = rng.standard_normal((n0, 4, 5))
        s = partition(n0, world, 3, periodic)[rank]
        buf = torch.full((s.n + 6, 4, 5), float("nan"), dtype=torch.float64)
        buf[3:3 + s.n] = torch.from_numpy(full[s.lo:s.lo + s.n])
        TorchDistTransport(s).exchange(buf)
        ok = True
        if s.has_lo:
            idx = [(s.lo - 3 + k) % n0 for k in range(3)]
            ok &= bool(np.array_equal(buf[0:3].numpy(), full[idx]))
        if s.has_hi:
            idx = [(s.lo + s.n + k) % n0 for k in range(3)]
            ok &= bool(np.array_equal(buf[s.n + 3:s.n + 6].numpy(), full[idx]))
        flags = TorchDistTransport(s).max_flags(rank + 1)
        ok &= flags == world
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n0,periodic", [(2, 13, False), (2, 12, True), (3, 20, True), (4, 17, False)])
def test_gloo_halo_exchange(world, n0, periodic):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n0, periodic, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert list(out) == [1] * world


def _gather_worker(rank, world, port, n0, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_03501_b200.distributed import gather_owned

        full = np.random.default_rng(3).standard_normal((n0, 3, 4))
        slabs = partition(n0, world, 3, False)
        s = slabs[rank]
        got = gather_owned(slabs, torch.from_numpy(full[s.lo:s.lo + s.n].copy()))
        out[rank] = int(np.array_equal(got, full)) if rank == 0 else int(got is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n0", [(2, 13), (3, 20), (4, 17)])
def test_gloo_gather_owned_uneven_slabs(world, n0):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n0, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert list(out) == [1] * world


def test_partition_self_ring():
    (s,) = partition(12, 1, 3, periodic=True, self_ring=True)
    assert s.has_lo and s.has_hi and s.lo_rank == 0 and s.hi_rank == 0
    sends, recvs = halo_plan(s)
    # first owned planes -> own upper halo, last owned planes -> own lower halo
    assert sends == [(0, (3, 6)), (0, (12, 15))] and recvs == [(0, (15, 18)), (0, (0, 3))]
    with pytest.raises(ValueError, match="self ring"):
        partition(12, 1, 3, periodic=False, self_ring=True)
    with pytest.raises(ValueError, match="self ring"):
        partition(12, 2, 3, periodic=True, self_ring=True)


def test_slab_halo_must_cover_the_kernels_planes():
    """the brick kernels stage HJ_HALO_MIN = 3 planes whatever the
    scheme's ghost width; thinner slab halos are refused before any device work."""
    import paper_2411_03501_b200 as hj
    from paper_2411_03501_b200 import _lib
    from paper_2411_03501_b200.distributed import SlabIntegrator

    assert _lib.HALO_MIN == 3
    g = hj.air3d_grid((24, 10, 12))
    with pytest.raises(ValueError, match="halo 2 thinner"):
        SlabIntegrator(g, hj.air3d_term_config(scheme="eno2"), 0, 2, halo=2)


class _FakeStats:
    """Stands in for device.Stats on CPU: read() returns a fixed hj_stats."""

    def __init__(self, nonfinite, tag, lo, hi):
        from paper_2411_03501_b200 import _lib

        self.s = _lib.HjStats()
        self.s.nonfinite = nonfinite
        self.s.first_bad_tag = tag
        for a in range(_lib.HJ_MAX_DIM):
            self.s.lo_key[a] = lo + a
            self.s.hi_key[a] = hi - a

    def read(self):
        return self.s


def _merge_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = partition(30, world, 3, False)[rank]
        # rank r: flag bit r, first failing key 100 - 10 r (rank world-1 failed first), ranges shifted by r
        st = _FakeStats(1 << rank, 100 - 10 * rank if rank else 0x7FFFFFFF, -5 - rank, 7 + rank)
        m = TorchDistTransport(s).merge_stats(st)
        ok = m.nonfinite == (1 << world) - 1
        ok &= m.first_bad_tag == 100 - 10 * (world - 1)
        ok &= m.lo_key[0] == -5 - (world - 1) and m.hi_key[0] == 7 + (world - 1) and m.hi_key[2] == 5 + world - 1
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_merge_stats_like_one_gpu(world):
    """flags are OR-ed (not max-ed) and first_bad_tag is min-reduced
    across ranks, so every rank raises the error the single-GPU run raises."""
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_merge_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert list(out) == [1] * world
