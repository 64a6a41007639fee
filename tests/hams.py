"""Oracle-side Hamiltonian descriptors for the golden cases (test helper).

Constants follow the reference (RocketParams defaults, reachability.py:33-47;
rockets_partials, reachability.py:139-157) and the builder fixtures pinned in
tests/golden/make_golden.py (AIR3D, DI4)."""
from __future__ import annotations

import numpy as np

from oracle import hjoracle as orc

ROCKET = dict(a=1.0, grav=32.0, u_min=-1.0, u_max=1.0)
AIR3D = dict(va=5.0, vb=5.0, a_in=1.0, b_in=1.0)
DI4 = dict(u_bar=1.0, d_bar=0.5)


def rockets_alphas(g, p=ROCKET):
    x_max = float(max(abs(g.mins[0]), abs(g.maxs[0])))
    a, grav = p["a"], p["grav"]
    return np.array([a + abs(p["u_max"]) * x_max,
                     max(abs(grav), abs(grav - 2.0 * a)) + abs(p["u_min"]) * x_max,
                     abs(p["u_max"]) + abs(p["u_min"])])


def air3d_alphas(g, vbc, vbs, p=AIR3D):
    x, y = g.axis_nodes[0], g.axis_nodes[1]
    return np.array([float(np.max(np.abs(-p["va"] + vbc))) + p["a_in"] * float(np.max(np.abs(y))),
                     float(np.max(np.abs(vbs))) + p["a_in"] * float(np.max(np.abs(x))),
                     p["a_in"] + p["b_in"]])


def di4_alphas(g, p=DI4):
    s = p["u_bar"] + p["d_bar"]
    return np.array([float(np.max(np.abs(g.axis_nodes[2]))), float(np.max(np.abs(g.axis_nodes[3]))), s, s])


def oracle_ham(name, g, meta=None, arrays=None):
    meta = meta or {}
    arrays = arrays or {}
    if name == "advection":
        c = np.asarray(meta["speeds"], dtype=np.float64)
        return orc.Ham("advection", c, alphas=np.abs(c))
    if name in ("rockets", "rockets_extremal"):
        tabs = (arrays["cos"], arrays["sin"]) if "cos" in arrays else (
            np.cos(g.axis_nodes[2]), np.sin(g.axis_nodes[2]))
        p = ROCKET
        return orc.Ham(name, (p["a"], p["grav"], p["u_min"], p["u_max"]), tabs, rockets_alphas(g))
    if name == "air3d":
        p = AIR3D
        vbc, vbs = (arrays["cos"], arrays["sin"]) if "cos" in arrays else (
            p["vb"] * np.cos(g.axis_nodes[2]), p["vb"] * np.sin(g.axis_nodes[2]))
        return orc.Ham("air3d", (p["va"], p["vb"], p["a_in"], p["b_in"]), (vbc, vbs), air3d_alphas(g, vbc, vbs))
    if name == "di4":
        p = DI4
        return orc.Ham("di4", (p["u_bar"], p["d_bar"]), (), di4_alphas(g))
    raise KeyError(name)
