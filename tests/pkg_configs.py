"""Package-side term configs for golden cases (test helper).

Trig tables are taken from the fixture (the reference's own np.cos/np.sin
bits, computed where the goldens were made) so that a different host CPU on
the GPU box cannot change the inputs."""
from __future__ import annotations

import numpy as np

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200.problems import Air3DHamiltonian, Air3DParams
from paper_2411_03501_b200.reachability import RocketsHamiltonian, RocketsPartials


class _FixedRockets(RocketsHamiltonian):
    def __init__(self, params, route, cos, sin):
        super().__init__(params, route)
        self._tabs = (np.asarray(cos), np.asarray(sin))

    def tables(self, g):
        return self._tabs


class _FixedAir3D(Air3DHamiltonian):
    def __init__(self, params, cos, sin):
        super().__init__(params)
        self._tabs = (np.asarray(cos), np.asarray(sin))

    def tables(self, g):
        return self._tabs


def package_config(name, scheme, meta=None, arrays=None, rocket_params=None):
    meta = meta or {}
    arrays = arrays or {}
    if name == "advection":
        return hj.advection_term_config(meta["speeds"], scheme=scheme)
    if name in ("rockets", "rockets_extremal"):
        p = rocket_params or hj.RocketParams()
        route = "published" if name == "rockets" else "extremal"
        return hj.TermConfig(hamiltonian=_FixedRockets(p, route, arrays["cos"], arrays["sin"]),
                             partials=RocketsPartials(p), derivative_scheme=scheme)
    if name == "air3d":
        base = hj.air3d_term_config(scheme=scheme)
        return hj.TermConfig(hamiltonian=_FixedAir3D(Air3DParams(), arrays["cos"], arrays["sin"]),
                             partials=base.partials, derivative_scheme=scheme)
    if name == "di4":
        return hj.di4_term_config(scheme=scheme)
    raise KeyError(name)
