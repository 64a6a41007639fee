"""Slab domain decomposition of the grid-update path across GPUs.

Axis 0 is split into contiguous slabs, one per rank (one process per GPU,
torch.distributed / NCCL over NVLink for the plumbing).  Each rank's state
buffer holds ``halo`` exchanged planes in front of and behind its owned
planes; the fused stage kernels read those planes where a single-GPU run
would read its neighbours' nodes, and synthesise the boundary ghosts only on
the global edges.  Per stage: one grouped send/recv of ``halo`` planes with
each neighbour, then the stage kernel.  Because the halos are exact copies
and every node update is local to its star stencil, the decomposed result is
bit-identical to the single-GPU one.  Dissipation bounds are global and
range-free, so dt needs no collective; non-finite flags are max-reduced once
per interval.

Transports:
* ``NcclTransport`` -- the data plane on GPUs: libhjb200's own NCCL
  communicator behind the C ABI (hj_dd_*, csrc/hj_dd.cu).  Each stage is ONE
  ABI call (grouped send/recv of the halo planes on the communicator's
  stream, CORE launch meanwhile, stream wait, RIM launch); per interval the
  device stats are all-reduced (first failing stage / error class, ranges)
  and snapshots are gathered with hj_dd_gather.  torch.distributed only
  broadcasts the communicator's unique id (any backend);
* ``TorchDistTransport`` -- a torch.distributed process group (gloo: the
  CPU-side multi-process tests, halos staged through the host);
* ``LocalTransport`` -- all slabs of one process on one device with plain
  copies (tests / emulation: no kernel ever waits on another).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dev
from .engine import FusedIntegrator
from .term import TermConfig


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    lo: int          # first owned global plane
    n: int           # owned planes
    halo: int
    has_lo: bool     # a neighbour provides planes below lo
    has_hi: bool     # a neighbour provides planes above lo + n
    lo_rank: int
    hi_rank: int


def partition(n0: int, world: int, halo: int, periodic: bool, self_ring: bool = False) -> list[Slab]:
    """Balanced contiguous split of axis 0; every slab must hold >= halo planes
    (its boundary planes are a neighbour's halo) and >= 2 (extrapolation).
    ``self_ring``: a single slab of a periodic axis 0 exchanges its halos with
    itself (the NCCL data plane on one GPU; the periodic wrap of
    grid.py:208-211 then arrives as exchanged planes)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if self_ring and not (world == 1 and periodic):
        raise ValueError("a self ring needs one slab of a periodic axis 0")
    base, extra = divmod(n0, world)
    sizes = [base + (1 if r < extra else 0) for r in range(world)]
    if (world > 1 or self_ring) and min(sizes) < max(halo, 2):
        raise ValueError(f"axis 0 has {n0} nodes: too few for {world} slabs with halo {halo}")
    slabs, lo = [], 0
    for r, n in enumerate(sizes):
        has_lo = self_ring or (world > 1 and (r > 0 or periodic))
        has_hi = self_ring or (world > 1 and (r < world - 1 or periodic))
        slabs.append(Slab(r, world, lo, n, halo, has_lo, has_hi, (r - 1) % world, (r + 1) % world))
        lo += n
    return slabs


def halo_plan(s: Slab):
    """Halo messages of one slab in buffer-plane coordinates (buffer plane p =
    owned plane p - halo).  Returns (sends, recvs): sends ordered [to lower,
    to upper], recvs ordered [from upper, from lower].  With that order the
    k-th send from A to B always pairs with B's k-th receive from A, even when
    the lower and upper neighbour are the same rank (two periodic slabs)."""
    h = s.halo
    sends, recvs = [], []
    if s.has_lo:   # my first h owned planes become the lower neighbour's upper halo
        sends.append((s.lo_rank, (h, 2 * h)))
    if s.has_hi:   # my last h owned planes become the upper neighbour's lower halo
        sends.append((s.hi_rank, (s.n, s.n + h)))
    if s.has_hi:
        recvs.append((s.hi_rank, (s.n + h, s.n + 2 * h)))
    if s.has_lo:
        recvs.append((s.lo_rank, (0, h)))
    return sends, recvs


class TorchDistTransport:
    """Halo exchange through a torch.distributed process group (NCCL on GPUs)."""

    def __init__(self, slab: Slab, group=None):
        self.slab = slab
        self.group = group

    def start(self, buf: torch.Tensor):
        """Post the halo exchange of ``buf``; returns what ``finish`` waits on.
        NCCL: the sends/receives run on NCCL's stream, ordered after the work
        already queued on the current stream, so the caller can launch the
        CORE part of the stage (which reads no halo plane) meanwhile."""
        import torch.distributed as dist

        sends, recvs = halo_plan(self.slab)
        if not sends and not recvs:
            return None
        staged = buf.is_cuda and dist.get_backend(self.group) != "nccl"
        if staged:
            # gloo moves host tensors only: stage the halo planes through the host
            torch.cuda.current_stream().synchronize()
            sbufs = [buf[a:b].cpu() for _, (a, b) in sends]
            rbufs = [torch.empty_like(buf[a:b], device="cpu") for _, (a, b) in recvs]
        else:
            sbufs = [buf[a:b] for _, (a, b) in sends]
            rbufs = [buf[a:b] for _, (a, b) in recvs]
        ops = [dist.P2POp(dist.isend, t, peer, self.group) for (peer, _), t in zip(sends, sbufs)]
        ops += [dist.P2POp(dist.irecv, t, peer, self.group) for (peer, _), t in zip(recvs, rbufs)]
        works = dist.batch_isend_irecv(ops)
        if staged:
            for w in works:
                w.wait()
            for (_, (a, b)), t in zip(recvs, rbufs):
                buf[a:b].copy_(t)
            return None
        return works

    def finish(self, pending) -> None:
        """Order the current stream after the exchange (NCCL: no host wait)."""
        for w in pending or ():
            w.wait()

    def exchange(self, buf: torch.Tensor) -> None:
        self.finish(self.start(buf))

    def max_flags(self, flags: int) -> int:
        import torch.distributed as dist

        t = torch.tensor([int(flags)], dtype=torch.int64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def merge_stats(self, stats: dev.Stats) -> "_lib.HjStats":
        """Every rank's hj_stats combined as one GPU would have accumulated
        them (nonfinite OR, first_bad_tag min, ranges min/max) -- host side,
        one MAX all-reduce of [bits, -tag, -lo keys, hi keys]."""
        import torch.distributed as dist

        st = stats.read()
        vals = [(int(st.nonfinite) >> b) & 1 for b in range(8)] + [-int(st.first_bad_tag)]
        vals += [-int(k) for k in st.lo_key] + [int(k) for k in st.hi_key]
        t = torch.tensor(vals, dtype=torch.int64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        v = [int(x) for x in t.tolist()]
        out = _lib.HjStats()
        out.nonfinite = sum(1 << b for b in range(8) if v[b])
        out.first_bad_tag = -v[8]
        for a in range(_lib.HJ_MAX_DIM):
            out.lo_key[a] = -v[9 + a]
            out.hi_key[a] = v[9 + _lib.HJ_MAX_DIM + a]
        return out

    def gather(self, slabs, owned: torch.Tensor, dst: int = 0):
        return gather_owned(slabs, owned, dst, self.group)


class NcclTransport:
    """The GPU data plane: libhjb200's NCCL communicator (hj_dd_*).

    torch.distributed (any backend) only broadcasts the communicator's
    unique id; with one rank (a self ring) no process group is needed."""

    native = True

    def __init__(self, slab: Slab, group=None):
        self.slab = slab
        self.group = group
        self.lib = dev.require()
        uid = ctypes.create_string_buffer(_lib.DD_UID_BYTES)
        if slab.world > 1:
            import torch.distributed as dist

            obj = [None]
            if dist.get_rank(group) == 0:
                _lib.check(self.lib.hj_dd_unique_id(uid), "hj_dd_unique_id")
                obj = [bytes(uid.raw)]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], _lib.DD_UID_BYTES)
        else:
            _lib.check(self.lib.hj_dd_unique_id(uid), "hj_dd_unique_id")
        h = ctypes.c_void_p()
        _lib.check(self.lib.hj_dd_init(uid, slab.world, slab.rank, slab.lo_rank if slab.has_lo else -1,
                                       slab.hi_rank if slab.has_hi else -1, ctypes.byref(h)), "hj_dd_init")
        self.h = h

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.hj_dd_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage(self, dg, scheme, dh, alphas_c, dt, kind, y_in, y0, y_out, mask_prev, mask, stats, tag, strm,
              overlap: bool) -> None:
        p = dev.ptr
        rc = self.lib.hj_dd_stage(self.h, dg.ref, _lib.SCHEME_CODES[scheme], dh.ref, alphas_c, float(dt), int(kind),
                                  p(y_in), p(y0), p(y_out), p(mask_prev), int(mask), stats.p if stats else None,
                                  int(tag), 1 if overlap else 0, strm)
        if rc:
            _lib.check(rc, "hj_dd_stage")

    def exchange_full(self, dg, buf: torch.Tensor) -> None:
        _lib.check(self.lib.hj_dd_exchange(self.h, dg.ref, dev.ptr(buf), dev.stream()), "hj_dd_exchange")

    def merge_stats(self, stats: dev.Stats) -> "_lib.HjStats":
        _lib.check(self.lib.hj_dd_reduce_stats(self.h, stats.p, dev.stream()), "hj_dd_reduce_stats")
        return stats.read()

    def gather(self, slabs, owned: torch.Tensor, dst: int = 0):
        mine = owned.contiguous()
        counts = (ctypes.c_int64 * len(slabs))(*[s.n * (mine.numel() // max(owned.shape[0], 1)) for s in slabs])
        full = None
        if self.slab.rank == dst:
            full = torch.empty((sum(s.n for s in slabs),) + tuple(mine.shape[1:]), dtype=mine.dtype,
                               device=mine.device)
        _lib.check(self.lib.hj_dd_gather(self.h, dev.ptr(mine), mine.numel(), dev.ptr(full) if full is not None
                                         else None, counts, int(dst), dev.stream()), "hj_dd_gather")
        return dev.to_host(full) if full is not None else None

    def traffic(self) -> tuple[int, int]:
        ex, by = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(self.lib.hj_dd_stats(self.h, ctypes.byref(ex), ctypes.byref(by)), "hj_dd_stats")
        return int(ex.value), int(by.value)


def default_transport(slab: Slab, group=None):
    """NCCL data plane (hj_dd) when the ranks drive GPUs through an NCCL
    process group (or HJ_SLAB_COMM=nccl), else the torch.distributed one."""
    import os

    import torch.distributed as dist

    want = os.environ.get("HJ_SLAB_COMM", "auto")
    if want == "nccl" or (want == "auto" and slab.world > 1 and dist.get_backend(group) == "nccl"):
        return NcclTransport(slab, group)
    return TorchDistTransport(slab, group)


class SlabIntegrator(FusedIntegrator):
    """FusedIntegrator on one slab of a decomposed grid.

    State tensors are FULL buffers of shape (halo + n + halo, n1, ...); the
    owned region is ``buf[halo:halo+n]``.  ``step3`` / ``integrate`` take and
    return full buffers.
    """

    def __init__(self, g, cfg: TermConfig, rank: int, world: int, halo: int = 3, transport=None, group=None,
                 overlap: bool = True, self_ring: bool = False):
        if halo < _lib.HALO_MIN:
            raise ValueError(f"slab halo {halo} thinner than the {_lib.HALO_MIN} planes the stage kernels read")
        self.slab = partition(g.counts[0], world, halo, g.is_periodic(0), self_ring=self_ring)[rank]
        # overlap: each stage = CORE launch while the halo exchange is in flight, then RIM
        self.overlap = overlap
        s = self.slab
        dg = dev.DeviceGrid(g, slab=(s.lo, s.n, int(s.has_lo), int(s.has_hi), s.halo))
        if transport == "nccl":
            transport = NcclTransport(s, group)
        self.transport = transport or default_transport(s, group)
        super().__init__(g, cfg, dg=dg, exchange=None)
        self.full_shape = (s.n + 2 * s.halo,) + tuple(g.counts[1:])
        self.owned_cells = dg.cells

    # -- buffers ---------------------------------------------------------
    def empty(self) -> torch.Tensor:
        return torch.zeros(self.full_shape, dtype=dev.F64, device=dev.device())

    def owned(self, buf: torch.Tensor) -> torch.Tensor:
        h = self.slab.halo
        return buf[h:h + self.slab.n]

    def init_shape(self, kind: int, params) -> torch.Tensor:
        buf = self.empty()
        self.owned(buf).copy_(dev.init_shape_dev(self.dg, kind, params))
        return buf

    def init_cylinder(self, radius: float, center=(0.0, 0.0, 0.0), ignore_mask: int = 4) -> torch.Tensor:
        return self.init_shape(_lib.SHAPE_CYLINDER, [*center, float(radius), float(ignore_mask)])

    def scatter(self, full: np.ndarray) -> torch.Tensor:
        buf = self.empty()
        self.owned(buf).copy_(dev.to_dev(full[self.slab.lo:self.slab.lo + self.slab.n]))
        return buf

    # -- stage plumbing ----------------------------------------------------
    def _buffers(self, like: torch.Tensor) -> list[torch.Tensor]:
        if not self._bufs:
            self._bufs = [self.empty() for _ in range(3)]
        return self._bufs

    def _stage(self, alphas_c, dt, kind, y_in, y0, y_out, mask_prev, mask, tag, strm):
        o = self.owned
        if getattr(self.transport, "native", False):
            # one ABI call: exchange on the communicator's stream, CORE, wait, RIM
            self.transport.stage(self.dg, self.scheme, self.dh, alphas_c, dt, kind, o(y_in),
                                 None if y0 is None else o(y0), o(y_out),
                                 None if mask_prev is None else o(mask_prev), mask, self.stats, tag, strm,
                                 self.overlap)
            self.launches += 2 if (self.overlap and (self.slab.has_lo or self.slab.has_hi)) else 1
            return
        args = (self.dg, self.scheme, self.dh, alphas_c, dt, kind, o(y_in), None if y0 is None else o(y0),
                o(y_out), None if mask_prev is None else o(mask_prev), mask, self.stats, tag)
        if self.overlap and (self.slab.has_lo or self.slab.has_hi):
            # halo exchange in flight while the core planes compute; the rim after it
            pending = self.transport.start(y_in)
            dev.stage_dev(*args, lib=self.lib, strm=strm, part=_lib.PART_CORE)
            self.transport.finish(pending)
            dev.stage_dev(*args, lib=self.lib, strm=strm, part=_lib.PART_RIM)
            self.launches += 2
            return
        self.transport.exchange(y_in)
        dev.stage_dev(*args, lib=self.lib, strm=strm)
        self.launches += 1

    def _read_stats(self):
        # every rank raises the error the single-GPU run raises: the stats are
        # combined across ranks first (flags OR, first failing stage min)
        return self.transport.merge_stats(self.stats)


class LocalTransport:
    """All slabs of a decomposition in one process on one device: before each
    stage every slab registers its input buffer, then each slab pulls its
    halos from the neighbours' buffers with plain device copies.  Emulation
    for tests -- kernels never wait on one another."""

    def __init__(self, slabs: list[Slab]):
        self.slabs = slabs
        self.buffers: dict[int, torch.Tensor] = {}
        self.flags: dict[int, int] = {}

    def register(self, rank: int, buf: torch.Tensor) -> None:
        self.buffers[rank] = buf

    def for_rank(self, rank: int) -> "_LocalEndpoint":
        return _LocalEndpoint(self, rank)


class _LocalEndpoint:
    def __init__(self, hub: LocalTransport, rank: int):
        self.hub, self.rank = hub, rank

    def start(self, buf: torch.Tensor):
        self.exchange(buf)

    def finish(self, pending) -> None:
        pass

    def exchange(self, buf: torch.Tensor) -> None:
        s = self.hub.slabs[self.rank]
        h = s.halo
        _, recvs = halo_plan(s)
        for peer, (a, b) in recvs:
            src = self.hub.buffers[peer]
            p = self.hub.slabs[peer]
            if a == 0:   # lower halo <- lower neighbour's last h owned planes
                buf[a:b].copy_(src[p.n:p.n + h])
            else:        # upper halo <- upper neighbour's first h owned planes
                buf[a:b].copy_(src[h:2 * h])

    def max_flags(self, flags: int) -> int:
        self.hub.flags[self.rank] = flags
        return max(self.hub.flags.values())

    def merge_stats(self, stats: dev.Stats):
        # emulation: each slab reports its own stats (the slabs run in one process)
        return stats.read()


def lockstep_step3(runs: list[SlabIntegrator], hub: LocalTransport, ys: list[torch.Tensor], t: float,
                   dt: float) -> list[torch.Tensor]:
    """One TVD-RK3 step of every slab, stage by stage (LocalTransport runs)."""
    from .engine import _STAGES

    bufs = [r._buffers(y) for r, y in zip(runs, ys)]
    outs = [[b for b in bs if b is not y][:2] for bs, y in zip(bufs, ys)]
    alphas = [_lib.doubles(r._alphas(t, y), _lib.HJ_MAX_DIM) for r, y in zip(runs, ys)]
    src = list(ys)
    for k, kind in enumerate(_STAGES[3]):
        dst = [(o[0], o[1], o[0])[k] for o in outs]
        for r in range(len(runs)):
            hub.register(r, src[r])
        for r, run in enumerate(runs):
            run._stage(alphas[r], dt, kind, src[r], ys[r] if k else None, dst[r], None, _lib.MASK_NONE, k,
                       dev.stream())
        src = dst
    return src


# ---------------------------------------------------------------- tube solve over slabs
def gather_owned(slabs: list[Slab], owned: torch.Tensor, dst: int = 0, group=None) -> np.ndarray | None:
    """Assemble the full field on rank ``dst`` from every rank's owned planes
    (point-to-point, so slabs of unequal size need no padding).  NCCL moves
    the device tensors directly; gloo stages them through the host.  Returns
    the field on ``dst`` and None elsewhere."""
    import torch.distributed as dist

    rank = dist.get_rank()
    nccl = dist.get_backend(group) == "nccl"
    mine = owned.contiguous() if (nccl or not owned.is_cuda) else owned.cpu()
    if rank != dst:
        dist.send(mine, dst, group=group)
        return None
    parts = []
    for s in slabs:
        if s.rank == dst:
            parts.append(mine)
            continue
        buf = torch.empty((s.n,) + tuple(mine.shape[1:]), dtype=mine.dtype, device=mine.device)
        dist.recv(buf, s.rank, group=group)
        parts.append(buf)
    full = torch.cat(parts, dim=0)
    return dev.to_host(full) if full.is_cuda else full.numpy()


def solve_tube_slabs(g, target, cfg: TermConfig, horizon: float, global_steps: int, order: int = 3, opts=None,
                     progress=None, group=None, halo: int | None = None, transport=None):
    """solve_tube (reachability.solve_tube) with axis 0 split across the ranks
    of a torch.distributed group: every rank integrates its slab (halo
    exchange per stage, non-finite flags max-reduced per interval), masks
    against its own previous slab, and per interval the owned planes are
    gathered to rank 0, which collects the snapshots and calls ``progress``.
    Rank 0 returns the BRTResult; the other ranks return one with the same
    times and no snapshots.  Bit-identical to the single-GPU tube."""
    import torch.distributed as dist

    from .integrator import IntegratorOptions
    from .reachability import BRTResult
    from .spatial import SCHEME_WIDTH

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    target_vals = np.asarray(target.values if hasattr(target, "values") else target, dtype=np.float64)
    if horizon == 0:
        return BRTResult(snapshots=(target,) if rank == 0 else (), times=(0.0,))
    opts = opts or IntegratorOptions()
    # the stage kernels stage HJ_HALO_MIN (3) exchanged planes whatever the
    # scheme's ghost width (spatial.py:27), so every slab carries 3
    halo = halo if halo is not None else max(SCHEME_WIDTH[cfg.derivative_scheme], _lib.HALO_MIN)
    if halo < _lib.HALO_MIN:
        raise ValueError(f"slab halo {halo} thinner than the {_lib.HALO_MIN} planes the stage kernels read")
    si = SlabIntegrator(g, cfg, rank, world, halo=halo, transport=transport, group=group)
    slabs = partition(g.counts[0], world, halo, g.is_periodic(0))
    use_min = cfg.approximation_sign == "over"
    prev = si.scatter(target_vals)
    snaps = [target] if rank == 0 else []
    times = [0.0]
    for k in range(1, global_steps + 1):
        t0, t1 = times[-1], horizon * k / global_steps
        try:
            res = si.integrate(order, (t0, t1), prev, opts, mask_prev=prev, use_min=use_min)
        except Exception as err:
            raise RuntimeError(f"tube interval {k} failed: {err}") from err
        prev = res.y
        full = si.transport.gather(slabs, si.owned(prev), 0)
        times.append(t1)
        if rank == 0:
            from .grid import ScalarField

            v = ScalarField._from_device(full)
            snaps.append(v)
            if progress is not None:
                progress(k, t1, v)
    return BRTResult(snapshots=tuple(snaps), times=tuple(times))
