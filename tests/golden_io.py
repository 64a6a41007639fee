"""Load tests/golden/*.npz fixtures (written by tests/golden/make_golden.py
from the reference) and rebuild their grids without the reference."""
from __future__ import annotations

import json
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases(name: str):
    """Yield (meta, arrays) for every case in tests/golden/<name>."""
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta):
        prefix = f"c{i}_"
        arrays = {k[len(prefix):]: z[k] for k in z.files if k.startswith(prefix)}
        yield m, arrays


def case_list(name: str):
    return list(cases(name))


def spec_grid(spec: dict):
    """A duck-typed grid following create_grid's node rules (grid.py:159-166)
    -- for the oracle, which must not depend on the product package."""
    lo = np.asarray(spec["mins"], dtype=np.float64)
    hi = np.asarray(spec["maxs"], dtype=np.float64)
    n = tuple(int(c) for c in spec["counts"])
    dim = len(n)
    per = set(spec["periodic"])
    spacings = np.empty(dim)
    nodes, bcs = [], []
    for i in range(dim):
        if i in per:
            spacings[i] = (hi[i] - lo[i]) / n[i]
            nodes.append(lo[i] + spacings[i] * np.arange(n[i]))
            bcs.append(SimpleNamespace(kind="periodic", value=0.0))
        else:
            spacings[i] = (hi[i] - lo[i]) / (n[i] - 1)
            nodes.append(np.linspace(lo[i], hi[i], n[i]))
            bcs.append(SimpleNamespace(kind="extrapolate", value=0.0))
    for k, v in spec.get("dirichlet", {}).items():
        bcs[int(k)] = SimpleNamespace(kind="dirichlet", value=float(v))
    return SimpleNamespace(dim=dim, counts=n, spacings=spacings, axis_nodes=tuple(nodes), boundary=tuple(bcs),
                           mins=lo, maxs=hi)


def package_grid(spec: dict):
    """The same grid through the package's create_grid / with_boundary."""
    import paper_2411_03501_b200 as hj

    g = hj.create_grid(spec["mins"], spec["maxs"], spec["counts"], periodic_axes=set(spec["periodic"]))
    for k, v in spec.get("dirichlet", {}).items():
        g = hj.with_boundary(g, int(k), hj.dirichlet(v))
    return g
