"""Build libhjb200.so in-tree with nvcc for sm_100a.

Each .cu translation unit compiles in parallel to build/obj/*.o; the shared
library is linked into the package directory so it travels with the repo
snapshot to the GPU box.  --fmad=false is part of the numerical contract:
it keeps every multiply and add separately rounded, as NumPy does.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import re
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libhjb200.so")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
         f"-I{INCLUDE}", "--expt-relaxed-constexpr"]


def _deps(src: str) -> list[str]:
    """Headers a translation unit includes, transitively (quoted includes)."""
    seen: set[str] = set()
    todo = [src]
    while todo:
        f = todo.pop()
        with open(f) as fh:
            for line in fh:
                m = re.match(r'\s*#\s*include\s+"([^"]+)"', line)
                if m:
                    h = os.path.normpath(os.path.join(os.path.dirname(f), m.group(1)))
                    if os.path.exists(h) and h not in seen:
                        seen.add(h)
                        todo.append(h)
    return sorted(seen)


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src: str, verbose: bool, check: bool = False) -> str:
    obj = os.path.join(OBJ + ("_check" if check else ""), os.path.basename(src)[:-3] + ".o")
    if _stale(obj, [src, *_deps(src)]):
        cmd = [NVCC, *ARCH, *FLAGS, *(["-DHJ_CHECK_BOUNDS"] if check else []), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False, jobs: int | None = None, check: bool = False) -> str:
    """Compile (incrementally) and link libhjb200.so; returns its path.
    check=True builds libhjb200_check.so instead: the same kernels with every
    global access of the stage kernels tested against its field's extent
    (-DHJ_CHECK_BOUNDS; tests and scripts/bounds_check.py only)."""
    os.makedirs(OBJ + ("_check" if check else ""), exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or max(1, min(len(sources), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, check), sources))
    lib = LIB.replace(".so", "_check.so") if check else LIB
    if _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", lib + ".tmp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, check="--check" in sys.argv))
