"""ctypes binding of libhjb200.so (C ABI declared in include/hjb200.h).

This module is the only place that touches the shared library.  Loading is
lazy; every entry point raises if the library or a CUDA device is missing —
the package has no CPU fallback for the grid-update path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

HJ_MAX_DIM = 5

# status codes
HJ_OK, HJ_EINVAL, HJ_ECUDA = 0, -1, -2
# boundary kinds
BC_CODES = {"periodic": 0, "extrapolate": 1, "dirichlet": 2}
# schemes (spatial.py:260-266)
SCHEME_CODES = {"first": 0, "eno2": 1, "eno3": 2, "weno5": 3, "weno5_fma": 4}
EPS_CODES = {"squared": 0, "raw": 1}
# Hamiltonian kinds
HAM_ADVECTION, HAM_ROCKETS, HAM_ROCKETS_EXTREMAL, HAM_AIR3D, HAM_DI4 = range(5)
# stage kinds
STAGE_DELTA, STAGE_EULER, STAGE_RK2_AVG, STAGE_RK3_QUARTER, STAGE_RK3_THIRD = range(5)
MASK_NONE, MASK_MIN, MASK_MAX = range(3)
SHAPE_SPHERE, SHAPE_CYLINDER, SHAPE_ELLIPSOID, SHAPE_BOX = range(4)
CSG_UNION, CSG_INTERSECT, CSG_COMPLEMENT, CSG_DIFFERENCE = range(4)
NF_INPUT, NF_DERIV, NF_HAM, NF_DELTA, NF_OUTPUT = 1, 2, 4, 8, 16
FLAG_HAM_NONZERO = 32
NF_MASK = 31
PART_ALL, PART_CORE, PART_RIM = range(3)   # hj_stage_part (hjb200.h HJ_PART_*)
HALO_MIN = 3          # hjb200.h HJ_HALO_MIN: exchanged planes per side of a slab buffer
DD_UID_BYTES = 128    # hjb200.h HJ_DD_UID_BYTES
HJ_ENCCL = -3


class HjGrid(ctypes.Structure):
    _fields_ = [
        ("dim", c_int32),
        ("batch", c_int32),
        ("n", c_int64 * HJ_MAX_DIM),
        ("h", c_double * HJ_MAX_DIM),
        ("bc", c_int32 * HJ_MAX_DIM),
        ("bc_value", c_double * HJ_MAX_DIM),
        ("nodes", c_void_p * HJ_MAX_DIM),
        ("halo_lo", c_int32),
        ("halo_hi", c_int32),
        ("halo", c_int32),
        ("_pad", c_int32),
        ("batch_stride", c_int64),
    ]


class HjHam(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32),
        ("_pad", c_int32),
        ("p", c_double * 16),
        ("tab", c_void_p * 4),
    ]


class HjStats(ctypes.Structure):
    _fields_ = [
        ("lo_key", c_int64 * HJ_MAX_DIM),
        ("hi_key", c_int64 * HJ_MAX_DIM),
        ("nonfinite", c_uint32),
        ("first_bad_tag", c_int32),
    ]


STATS_BYTES = ctypes.sizeof(HjStats)

_LIB = None
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhjb200.so")
# HJ_LIB=check selects the bounds-checking build (libhjb200_check.so, build.py --check)
if os.environ.get("HJ_LIB") == "check":
    _LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhjb200_check.so")
# HJ_LIB_PATH: an explicit build of the library (A/B of two builds in one process tree, scripts/)
if os.environ.get("HJ_LIB_PATH"):
    _LIB_PATH = os.environ["HJ_LIB_PATH"]

# (name, restype, argtypes) -- must match include/hjb200.h
_SIGNATURES = [
    ("hj_version", c_int, []),
    ("hj_last_error", ctypes.c_char_p, []),
    ("hj_launch_count", c_uint64, []),
    ("hj_extend_ghost", c_int, [POINTER(HjGrid), c_int, c_void_p, c_void_p, c_void_p]),
    ("hj_derivs", c_int, [POINTER(HjGrid), c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hj_weno5_workspace", c_int, [POINTER(HjGrid), c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    ("hj_stage", c_int, [POINTER(HjGrid), c_int, POINTER(HjHam), POINTER(c_double), c_double, c_int,
                         c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int32, c_void_p]),
    ("hj_stage_part", c_int, [POINTER(HjGrid), c_int, POINTER(HjHam), POINTER(c_double), c_double, c_int,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int32, c_int, c_void_p]),
    ("hj_stage_planes", c_int, [POINTER(HjGrid), c_int, POINTER(HjHam), POINTER(c_double), c_double, c_int,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int32, c_int64, c_int64,
                                c_void_p]),
    ("hj_term", c_int, [POINTER(HjGrid), c_int, POINTER(HjHam), POINTER(c_double), c_void_p, c_void_p,
                        c_void_p, c_void_p]),
    ("hj_costates", c_int, [POINTER(HjGrid), POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p),
                            c_void_p, c_void_p]),
    ("hj_glf_delta", c_int, [POINTER(HjGrid), POINTER(c_double), POINTER(c_void_p), POINTER(c_void_p),
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hj_rk_combine", c_int, [c_int64, c_int, c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_int32, c_void_p]),
    ("hj_init_shape", c_int, [POINTER(HjGrid), c_int, POINTER(c_double), c_int, c_void_p, c_void_p]),
    ("hj_csg", c_int, [c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hj_mask", c_int, [c_int64, c_void_p, c_void_p, c_int, c_void_p]),
    ("hj_count_below", c_int, [c_int64, c_void_p, c_double, c_void_p, c_void_p]),
    ("hj_stats_reset", c_int, [c_void_p, c_void_p]),
    ("hj_bounds_violations", c_int64, []),
    ("hj_eval_hamiltonian", c_int, [POINTER(HjGrid), POINTER(HjHam), POINTER(c_void_p), c_void_p, c_void_p]),
    ("hj_integrate", c_int, [POINTER(HjGrid), c_int, POINTER(HjHam), POINTER(c_double), c_int, c_double, c_double,
                             c_double, c_double, c_int, c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                             c_int, c_void_p, POINTER(c_double), POINTER(c_void_p), c_void_p]),
    ("hj_tube_check", c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_int, c_double, c_void_p, c_void_p]),
    ("hj_check_division", c_int, [c_int64, c_uint64, c_void_p, c_void_p]),
    ("hj_fp64_probe", c_int, [c_int, c_int, c_void_p, c_void_p]),
    ("hj_set_stage_kernel", c_int, [c_int]),
    ("hj_divided_differences", c_int, [POINTER(HjGrid), c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p]),
    # multi-GPU slabs (hj_dd.cu)
    ("hj_dd_nccl_version", c_int, []),
    ("hj_dd_unique_id", c_int, [c_void_p]),
    ("hj_dd_init", c_int, [c_void_p, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    ("hj_dd_stage", c_int, [c_void_p, POINTER(HjGrid), c_int, POINTER(HjHam), POINTER(c_double), c_double, c_int,
                            c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int32, c_int, c_void_p]),
    ("hj_dd_exchange", c_int, [c_void_p, POINTER(HjGrid), c_void_p, c_void_p]),
    ("hj_dd_reduce_stats", c_int, [c_void_p, c_void_p, c_void_p]),
    ("hj_dd_gather", c_int, [c_void_p, c_void_p, c_int64, c_void_p, POINTER(c_int64), c_int, c_void_p]),
    ("hj_dd_stats", c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64)]),
    ("hj_dd_free", c_int, [c_void_p]),
]

EXPORTED_SYMBOLS = tuple(name for name, _, _ in _SIGNATURES)


class LibraryMissing(RuntimeError):
    pass


def library_path() -> str:
    return _LIB_PATH


def load(path: str | None = None):
    """Load and type the shared library (no CUDA call is made here)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or _LIB_PATH
    if not os.path.exists(p):
        raise LibraryMissing(
            f"libhjb200.so not built at {p}; run `python -c 'import __graft_entry__ as e; e.build()'`"
        )
    lib = ctypes.CDLL(p)
    for name, res, args in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map an HJ status code to the reference's exception types."""
    if rc == HJ_OK:
        return
    msg = (load().hj_last_error() or b"").decode()
    if rc == HJ_EINVAL:
        raise ValueError(msg or f"{what}: invalid argument")
    if rc == HJ_ENCCL:
        raise RuntimeError(f"{what}: {msg or 'NCCL failure'} (NCCL, status {rc})")
    raise RuntimeError(f"{what}: {msg or 'CUDA failure'} (status {rc})")


def launch_count() -> int:
    return int(load().hj_launch_count())


def decode_key(k: int) -> float:
    """Inverse of the device's order-preserving double -> int64 map."""
    import struct

    k = int(k)
    if k < 0:
        k ^= 0x7FFFFFFFFFFFFFFF
    return struct.unpack("<d", struct.pack("<q", k))[0]


def ptr_array(ptrs) -> "ctypes.Array":
    arr = (c_void_p * HJ_MAX_DIM)()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def doubles(values, n: int | None = None) -> "ctypes.Array":
    vals = [float(x) for x in values]
    arr = (c_double * max(n or len(vals), 1))()
    for i, x in enumerate(vals):
        arr[i] = x
    return arr
