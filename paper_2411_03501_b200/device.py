"""Device plumbing: torch owns the HBM buffers and the stream, libhjb200.so
does the arithmetic.  Every function here launches CUDA kernels through the
C ABI; there is no host implementation to fall back to.
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np
import torch

from . import _lib
from ._lib import HJ_MAX_DIM, HjGrid, HjHam, HjStats, check

F64 = torch.float64


def require():
    """Return the loaded library; raise loudly when CUDA or the build is missing."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2411_03501_b200 needs a CUDA device (B200); there is no CPU path")
    return _lib.load()


STAGE_KERNELS = {"env": -1, "generic": 0, "auto": 1, "brick1": 2, "brick_always": 3, "brick_u2": 4,
                 "brick_noload": 5,   # brick_noload: A/B timing bound only, results are wrong
                 "brick_nopf": 6,     # no L2 prefetch of the next brick (A/B)
                 "brick_x": 7,        # A/B slot: the variant under test (hj_brick_weno.cu)
                 "tile_stages": 8,    # small 3-D grids: the tile kernel launched per stage (no persistent launch)
                 "axes": 9,           # the per-axis walk pipeline (hj_axes.cuh) forced on every WENO5 grid size
                 # per-axis pipeline A/B: every walk rolled (the r02g default), the
                 # contiguous-axis walk unrolled too (hj_axes.cuh launch_axes_t)
                 "axes_r1": 10, "axes_u2x": 11,
                 "axes_l32": 12,      # ... the last-axis kernel on 32-node segments
                 "axes_s16": 13}      # ... column kernels on 16-node segments (the default is 32)


def set_stage_kernel(name: str) -> str:
    """Select the fused-stage kernel family (A/B runs, test coverage); returns the previous one."""
    old = require().hj_set_stage_kernel(STAGE_KERNELS[name])
    if old < 0:
        raise ValueError(f"unknown stage kernel {name!r}")
    return {v: k for k, v in STAGE_KERNELS.items()}[old]


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a) -> torch.Tensor:
    """Host array -> contiguous float64 CUDA tensor."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=F64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device())


def host_empty(shape, dtype=torch.float64) -> torch.Tensor:
    """Host buffer for device copies: pinned (direct DMA) when the OS lets the
    process lock that much memory, else pageable (the copy is then staged by
    the driver -- slower, same bytes)."""
    try:
        return torch.empty(shape, dtype=dtype, pin_memory=True)
    except RuntimeError:   # cudaHostAlloc refused (locked-memory limit / host RAM)
        return torch.empty(shape, dtype=dtype)


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy.  Large fields land in pinned host memory (torch's
    caching host allocator) so the copy is a direct DMA, not a staged one."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= (1 << 20):
        out = host_empty(t.shape, t.dtype)
        out.copy_(t)
        return out.numpy()
    return t.cpu().numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous() and t.dtype == F64, "expected a contiguous float64 CUDA tensor"
    return t.data_ptr()


# ---------------------------------------------------------------- grids on the device
class DeviceGrid:
    """hj_grid for a Grid: node tables resident in HBM, ghost rules, spacings.

    ``batch`` stacks independent problems in front; ``slab`` = (lo, n_owned,
    halo_lo, halo_hi, halo) restricts axis 0 to a slab of a decomposed grid.
    """

    def __init__(self, g, batch: int = 1, slab=None):
        require()
        self.grid = g
        self.batch = int(batch)
        lo0 = 0
        counts = list(g.counts)
        s = HjGrid()
        s.dim = g.dim
        s.batch = self.batch
        if slab is not None:
            lo0, n0, hlo, hhi, halo = slab
            counts[0] = n0
            s.halo_lo, s.halo_hi, s.halo = int(hlo), int(hhi), int(halo)
        self.counts = tuple(counts)
        self.nodes = []
        for a in range(g.dim):
            nodes = np.asarray(g.axis_nodes[a], dtype=np.float64)
            if a == 0 and slab is not None:
                nodes = nodes[lo0:lo0 + counts[0]]
            t = to_dev(nodes)
            self.nodes.append(t)
            s.n[a] = counts[a]
            s.h[a] = float(g.spacings[a])
            s.bc[a] = _lib.BC_CODES[g.boundary[a].kind]
            s.bc_value[a] = float(g.boundary[a].value)
            s.nodes[a] = t.data_ptr()
        self.cells = int(np.prod(counts))
        self.plane = int(np.prod(counts[1:])) if g.dim > 1 else 1
        s.batch_stride = 0
        self.s = s

    def set_batch_stride(self, stride: int) -> None:
        self.s.batch_stride = int(stride)

    @property
    def ref(self):
        return ctypes.byref(self.s)

    @property
    def shape(self) -> tuple[int, ...]:
        return (self.batch,) + self.counts if self.batch > 1 else self.counts


_GRIDS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def device_grid(g) -> DeviceGrid:
    """Cached single-problem DeviceGrid of a Grid (node tables uploaded once)."""
    dg = _GRIDS.get(g)
    if dg is None:
        dg = DeviceGrid(g)
        _GRIDS[g] = dg
    return dg


# ---------------------------------------------------------------- statistics
class Stats:
    """Device-resident hj_stats (non-finite flags, costate ranges)."""

    def __init__(self):
        self.buf = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=device())

    @property
    def p(self) -> int:
        return self.buf.data_ptr()

    def reset(self) -> "Stats":
        check(require().hj_stats_reset(self.p, stream()), "hj_stats_reset")
        return self

    def read(self) -> HjStats:
        raw = bytes(self.buf.cpu().numpy().tobytes())
        return HjStats.from_buffer_copy(raw)

    @staticmethod
    def ranges(st: HjStats, dim: int):
        return tuple((_lib.decode_key(st.lo_key[a]), _lib.decode_key(st.hi_key[a])) for a in range(dim))


# ---------------------------------------------------------------- registered Hamiltonians on the device
class DeviceHam:
    """hj_ham with its tables resident in HBM."""

    def __init__(self, kind: int, params, tables=()):
        require()
        self.s = HjHam()
        self.s.kind = int(kind)
        for i, x in enumerate(params):
            self.s.p[i] = float(x)
        self.tabs = [to_dev(np.asarray(t, dtype=np.float64)) for t in tables]
        for i, t in enumerate(self.tabs):
            self.s.tab[i] = t.data_ptr()

    @property
    def ref(self):
        return ctypes.byref(self.s)


# ---------------------------------------------------------------- kernel wrappers (device tensors in/out)
def extend_ghost(g, values: np.ndarray, width: int) -> np.ndarray:
    lib = require()
    dg = device_grid(g)
    v = to_dev(values)
    out = torch.empty(tuple(n + 2 * width for n in g.counts), dtype=F64, device=device())
    check(lib.hj_extend_ghost(dg.ref, int(width), ptr(v), ptr(out), stream()), "hj_extend_ghost")
    return to_host(out)


def derivs_dev(dg: DeviceGrid, v: torch.Tensor, axis: int, scheme: str, eps_mode: str = "squared"):
    lib = require()
    L = torch.empty_like(v)
    R = torch.empty_like(v)
    check(lib.hj_derivs(dg.ref, _lib.SCHEME_CODES[scheme], int(axis), _lib.EPS_CODES[eps_mode], ptr(v), ptr(L),
                        ptr(R), stream()), "hj_derivs")
    return L, R


def weno5_workspace_dev(dg: DeviceGrid, v: torch.Tensor, axis: int, side: str, eps_mode: str) -> torch.Tensor:
    lib = require()
    ws = torch.empty((10,) + tuple(v.shape), dtype=F64, device=v.device)
    check(lib.hj_weno5_workspace(dg.ref, int(axis), 0 if side == "left" else 1, _lib.EPS_CODES[eps_mode], ptr(v),
                                 ptr(ws), stream()), "hj_weno5_workspace")
    return ws


def divided_differences_dev(dg: DeviceGrid, v: torch.Tensor, axis: int, order: int, width: int):
    lib = require()
    counts = list(dg.counts)
    n = counts.pop(axis)
    lead = tuple(counts)
    ne = n + 2 * width
    mk = lambda k: torch.empty(lead + (ne - k,), dtype=F64, device=v.device)  # noqa: E731
    d0, d1 = mk(0), mk(1)
    d2 = mk(2) if order >= 2 else None
    d3 = mk(3) if order >= 3 else None
    check(lib.hj_divided_differences(dg.ref, int(axis), int(width), int(order), ptr(v), ptr(d0), ptr(d1), ptr(d2),
                                     ptr(d3), stream()), "hj_divided_differences")
    return d0, d1, d2, d3


def eval_hamiltonian_dev(dg: DeviceGrid, dh: DeviceHam, p) -> torch.Tensor:
    lib = require()
    out = torch.empty(dg.shape, dtype=F64, device=device())
    arr = _lib.ptr_array([ptr(x) for x in p])
    check(lib.hj_eval_hamiltonian(dg.ref, dh.ref, arr, ptr(out), stream()), "hj_eval_hamiltonian")
    return out


def init_shape_dev(dg: DeviceGrid, kind: int, params) -> torch.Tensor:
    lib = require()
    out = torch.empty(dg.shape, dtype=F64, device=device())
    prm = _lib.doubles(params)
    check(lib.hj_init_shape(dg.ref, int(kind), prm, len(params), ptr(out), stream()), "hj_init_shape")
    return out


def csg_dev(op: int, a: torch.Tensor, b: torch.Tensor | None) -> torch.Tensor:
    lib = require()
    out = torch.empty_like(a)
    check(lib.hj_csg(int(op), a.numel(), ptr(a), ptr(b), ptr(out), stream()), "hj_csg")
    return out


def mask_dev(v: torch.Tensor, prev: torch.Tensor, use_min: bool) -> None:
    lib = require()
    check(lib.hj_mask(v.numel(), ptr(prev), ptr(v), _lib.MASK_MIN if use_min else _lib.MASK_MAX, stream()),
          "hj_mask")


def count_below_dev(v: torch.Tensor, level: float) -> int:
    lib = require()
    c = torch.zeros(1, dtype=torch.int64, device=v.device)
    check(lib.hj_count_below(v.numel(), ptr(v), float(level), c.data_ptr(), stream()), "hj_count_below")
    return int(c.item())


def tube_check_dev(prev: torch.Tensor, v: torch.Tensor, target: torch.Tensor, use_min: bool, level: float,
                   out: torch.Tensor) -> None:
    """hj_tube_check: add this interval's nesting / containment violations,
    sublevel count and newly captured nodes to the int64[4] device tensor ``out``."""
    lib = require()
    check(lib.hj_tube_check(v.numel(), ptr(prev), ptr(v), ptr(target), _lib.MASK_MIN if use_min else _lib.MASK_MAX,
                            float(level), out.data_ptr(), stream()), "hj_tube_check")


def costates_dev(dg: DeviceGrid, Ls, Rs, stats: Stats | None):
    lib = require()
    P = [torch.empty_like(x) for x in Ls]
    check(lib.hj_costates(dg.ref, _lib.ptr_array([ptr(x) for x in Ls]), _lib.ptr_array([ptr(x) for x in Rs]),
                          _lib.ptr_array([ptr(x) for x in P]), stats.p if stats else None, stream()), "hj_costates")
    return P


def glf_delta_dev(dg: DeviceGrid, alphas, Ls, Rs, ham: torch.Tensor, want_diss: bool, stats: Stats | None):
    lib = require()
    delta = torch.empty_like(ham)
    diss = torch.empty_like(ham) if want_diss else None
    check(lib.hj_glf_delta(dg.ref, _lib.doubles(alphas, HJ_MAX_DIM), _lib.ptr_array([ptr(x) for x in Ls]),
                           _lib.ptr_array([ptr(x) for x in Rs]), ptr(ham), ptr(diss), ptr(delta),
                           stats.p if stats else None, stream()), "hj_glf_delta")
    return delta, diss


def rk_combine_dev(stage: int, dt: float, y: torch.Tensor, y0: torch.Tensor | None, delta: torch.Tensor,
                   out: torch.Tensor, stats: Stats | None = None, tag: int = 0) -> None:
    lib = require()
    check(lib.hj_rk_combine(y.numel(), int(stage), float(dt), ptr(y), ptr(y0), ptr(delta), ptr(out),
                            stats.p if stats else None, int(tag), stream()), "hj_rk_combine")


def term_dev(dg: DeviceGrid, scheme: str, dh: DeviceHam, alphas, v: torch.Tensor, stats: Stats | None):
    lib = require()
    delta = torch.empty_like(v)
    check(lib.hj_term(dg.ref, _lib.SCHEME_CODES[scheme], dh.ref, _lib.doubles(alphas, HJ_MAX_DIM), ptr(v),
                      ptr(delta), stats.p if stats else None, stream()), "hj_term")
    return delta


def stage_dev(dg: DeviceGrid, scheme: str, dh: DeviceHam, alphas_c, dt: float, stage: int, y_in: torch.Tensor,
              y0: torch.Tensor | None, y_out: torch.Tensor, mask_prev: torch.Tensor | None = None,
              mask: int = 0, stats: Stats | None = None, tag: int = 0, lib=None, strm=None,
              part: int = 0, planes: tuple[int, int] | None = None) -> None:
    """One fused TVD-RK stage (hj_stage; hj_stage_part when ``part`` is
    PART_CORE / PART_RIM).  ``alphas_c`` is a ctypes double[5]."""
    lib = lib or require()
    if planes is not None:
        rc = lib.hj_stage_planes(dg.ref, _lib.SCHEME_CODES[scheme], dh.ref, alphas_c, float(dt), int(stage),
                                 ptr(y_in), ptr(y0), ptr(y_out), ptr(mask_prev), int(mask),
                                 stats.p if stats else None, int(tag), int(planes[0]), int(planes[1]),
                                 strm if strm is not None else stream())
        if rc:
            check(rc, "hj_stage_planes")
        return
    if part:
        rc = lib.hj_stage_part(dg.ref, _lib.SCHEME_CODES[scheme], dh.ref, alphas_c, float(dt), int(stage),
                               ptr(y_in), ptr(y0), ptr(y_out), ptr(mask_prev), int(mask),
                               stats.p if stats else None, int(tag), int(part),
                               strm if strm is not None else stream())
        if rc:
            check(rc, "hj_stage_part")
        return
    rc = lib.hj_stage(dg.ref, _lib.SCHEME_CODES[scheme], dh.ref, alphas_c, float(dt), int(stage), ptr(y_in),
                      ptr(y0), ptr(y_out), ptr(mask_prev), int(mask), stats.p if stats else None, int(tag),
                      strm if strm is not None else stream())
    if rc:
        check(rc, "hj_stage")
