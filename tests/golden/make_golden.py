"""Generate golden vectors by running the REFERENCE itself (run here only).

    python tests/golden/make_golden.py [/root/reference]

The reference package (/root/reference/pkg/src/hjls, pure Python + NumPy) is
imported under the alias ``hjls_ref`` and exercised on small seeded inputs;
inputs and outputs land in tests/golden/*.npz.  These fixtures pin the CPU
oracle (oracle/hjoracle.c) in the CPU test suite and the CUDA path in the
GPU suite.  /root/reference does not exist on the GPU box, so nothing there
calls this script -- it only reads the committed .npz files.

Air3D and the 4-D double-integrator pair are not in the reference
(SPEC.md:15).  They are plugged into the reference's own TermConfig /
term_lax_friedrichs / ode_cfl_k / solve_brt API here with the operation order
pinned below; the package's device Hamiltonians (hj_ham.cuh) mirror it.
"""
from __future__ import annotations

import importlib.util
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def load_reference(root: str):
    src = os.path.join(root, "pkg", "src", "hjls")
    spec = importlib.util.spec_from_file_location(
        "hjls_ref", os.path.join(src, "__init__.py"), submodule_search_locations=[src]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["hjls_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


# ----------------------------------------------------------------- builder fixtures (pinned op order)
AIR3D = dict(va=5.0, vb=5.0, a_in=1.0, b_in=1.0, mins=(-6.0, -10.0, 0.0), maxs=(20.0, 10.0, 2 * math.pi),
             radius=5.0)
DI4 = dict(u_bar=1.0, d_bar=0.5, mins=(-8.0, -8.0, -4.0, -4.0), maxs=(8.0, 8.0, 4.0, 4.0), radius=2.0)


def air3d_tables(g, p=AIR3D):
    psi = g.axis_nodes[2]
    return p["vb"] * np.cos(psi), p["vb"] * np.sin(psi)


def air3d_alphas(g, p=AIR3D):
    vbc, vbs = air3d_tables(g, p)
    x, y = g.axis_nodes[0], g.axis_nodes[1]
    return np.array([
        float(np.max(np.abs(-p["va"] + vbc))) + p["a_in"] * float(np.max(np.abs(y))),
        float(np.max(np.abs(vbs))) + p["a_in"] * float(np.max(np.abs(x))),
        p["a_in"] + p["b_in"],
    ])


def air3d_config(ref, scheme, p=AIR3D):
    def ham(t, g, v, pc):
        x = g.axis_nodes[0].reshape(-1, 1, 1)
        y = g.axis_nodes[1].reshape(1, -1, 1)
        vbc, vbs = air3d_tables(g, p)
        vbc = vbc.reshape(1, 1, -1)
        vbs = vbs.reshape(1, 1, -1)
        p1, p2, p3 = (f.values for f in pc)
        return ref.ScalarField(-(-p["va"] * p1 + vbc * p1 + vbs * p2
                                 + p["a_in"] * np.abs(y * p1 - x * p2 - p3) - p["b_in"] * np.abs(p3)))

    def partials(t, g, v, ranges, axis):
        return float(air3d_alphas(g, p)[axis])

    return ref.TermConfig(hamiltonian=ham, partials=partials, derivative_scheme=scheme)


def di4_alphas(g, p=DI4):
    wx, wy = g.axis_nodes[2], g.axis_nodes[3]
    s = p["u_bar"] + p["d_bar"]
    return np.array([float(np.max(np.abs(wx))), float(np.max(np.abs(wy))), s, s])


def di4_config(ref, scheme, p=DI4):
    def ham(t, g, v, pc):
        wx = g.axis_nodes[2].reshape(1, 1, -1, 1)
        wy = g.axis_nodes[3].reshape(1, 1, 1, -1)
        p1, p2, p3, p4 = (f.values for f in pc)
        return ref.ScalarField(-(p1 * wx + p2 * wy + (p["d_bar"] - p["u_bar"]) * (np.abs(p3) + np.abs(p4))))

    def partials(t, g, v, ranges, axis):
        return float(di4_alphas(g, p)[axis])

    return ref.TermConfig(hamiltonian=ham, partials=partials, derivative_scheme=scheme)


def di4_target(ref, g, p=DI4):
    d2 = np.zeros(g.counts)
    for axis in (0, 1):
        d2 += (ref.mesh_coordinates(g, axis).values - 0.0) ** 2
    return ref.ScalarField(np.sqrt(d2) - p["radius"])


def brt_clone(ref, g, target, cfg, horizon, steps, order, opts=None):
    """solve_brt (reachability.py:218-254) with a selectable integrator order,
    for dims/orders that ReachProblem / solve_brt do not accept."""
    integ = {1: ref.ode_cfl_1, 2: ref.ode_cfl_2, 3: ref.ode_cfl_3}[order]
    mask = np.minimum if cfg.approximation_sign == "over" else np.maximum

    def rhs(t, y, c):
        return ref.term_lax_friedrichs(t, y, c, g)

    snaps, times, nsteps = [target], [0.0], []
    v = target
    for k in range(1, steps + 1):
        t0, t1 = times[-1], horizon * k / steps
        res = integ(rhs, (t0, t1), v, opts or ref.IntegratorOptions(), cfg)
        v = ref.ScalarField(mask(res.y_final.values, snaps[-1].values))
        snaps.append(v)
        times.append(t1)
        nsteps.append(res.steps_taken)
    return snaps, times, nsteps


# ----------------------------------------------------------------- helpers
class Store:
    def __init__(self):
        self.arrays = {}
        self.meta = []

    def case(self, meta: dict, **arrays):
        i = len(self.meta)
        self.meta.append(meta)
        for k, v in arrays.items():
            self.arrays[f"c{i}_{k}"] = np.asarray(v)

    def save(self, name):
        path = os.path.join(HERE, name)
        np.savez_compressed(path, meta=np.array(json.dumps(self.meta)), **self.arrays)
        print(f"{name}: {len(self.meta)} cases, {os.path.getsize(path)} bytes")


def gspec(mins, maxs, counts, periodic=(), dirichlet=None):
    return dict(mins=list(map(float, mins)), maxs=list(map(float, maxs)), counts=list(map(int, counts)),
                periodic=sorted(periodic), dirichlet={str(k): float(v) for k, v in (dirichlet or {}).items()})


def make_grid(ref, spec):
    g = ref.create_grid(spec["mins"], spec["maxs"], spec["counts"], periodic_axes=set(spec["periodic"]))
    for k, v in spec["dirichlet"].items():
        g = ref.with_boundary(g, int(k), ref.dirichlet(v))
    return g


def fields(rng, g, kinds=("random", "sdf", "smooth")):
    out = {}
    X = [ref_mesh(g, a) for a in range(g.dim)]
    for kind in kinds:
        if kind == "random":
            out[kind] = rng.standard_normal(g.counts)
        elif kind == "sdf":
            d2 = sum((X[a] - 0.3 * (a + 1)) ** 2 for a in range(g.dim))
            out[kind] = np.sqrt(d2) - 0.7 + 0.2 * np.abs(X[0])  # kinks + a cone
        else:
            out[kind] = sum(np.sin(1.3 * X[a] + 0.5 * a) for a in range(g.dim)) + 0.1 * X[-1] ** 3
    return out


def ref_mesh(g, axis):
    shape = [1] * g.dim
    shape[axis] = g.counts[axis]
    return np.broadcast_to(g.axis_nodes[axis].reshape(shape), g.counts).copy()


GRIDS = [
    gspec((-1.0,), (2.0,), (17,)),
    gspec((-math.pi,), (math.pi,), (16,), periodic={0}),
    gspec((0.0,), (1.0,), (13,), dirichlet={0: 0.75}),
    gspec((-1.0, 0.0), (1.0, 2.0), (9, 11), periodic={1}),
    gspec((-1.0, -2.0), (1.0, 2.0), (10, 8), dirichlet={0: -1.5}),
    gspec((-1.0, -1.0, 0.0), (1.0, 1.5, 2 * math.pi), (7, 8, 9), periodic={2}),
    gspec((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), (8, 7, 6), periodic={0}, dirichlet={1: 2.0}),
    gspec((-1.0, -1.0, -1.0, -1.0), (1.0, 1.0, 1.0, 1.0), (6, 5, 7, 6), periodic={3}),
]


def gen_grid_and_ghost(ref, rng):
    st = Store()
    for spec in GRIDS + [gspec((0.0,), (1.0,), (4,), periodic={0}), gspec((0.0, 0.0, 0.0), (1.0, 1.0, 1.0),
                                                                           (4, 5, 6), periodic={1})]:
        g = make_grid(ref, spec)
        v = rng.standard_normal(g.counts)
        for w in (1, 2, 3):
            if any(g.is_periodic(a) and w > g.counts[a] for a in range(g.dim)):
                continue
            ext = ref.extend_with_ghost_cells(g, ref.ScalarField(v), w).values
            arrays = {"v": v, "ext": ext, "spacings": g.spacings}
            for a in range(g.dim):
                arrays[f"nodes{a}"] = g.axis_nodes[a]
            st.case(dict(grid=spec, width=w), **arrays)
    st.save("ghost.npz")


def gen_derivs(ref, rng):
    st = Store()
    for spec in GRIDS:
        g = make_grid(ref, spec)
        for kind, v in fields(rng, g).items():
            f = ref.ScalarField(v)
            for scheme in ("first", "eno2", "eno3", "weno5"):
                for axis in range(g.dim):
                    pair = ref.derivative_pair(g, f, axis, scheme)
                    st.case(dict(grid=spec, field=kind, scheme=scheme, axis=axis, eps_mode="squared"),
                            v=v, left=pair.left.values, right=pair.right.values)
            for axis in range(g.dim):
                pair = ref.upwind_first_weno5(g, f, axis, eps_mode="raw")
                st.case(dict(grid=spec, field=kind, scheme="weno5", axis=axis, eps_mode="raw"),
                        v=v, left=pair.left.values, right=pair.right.values)
    # exact-arithmetic fields from the reference tests (ties in the ENO picks)
    g = ref.create_grid((0.0,), (16.0,), (17,))
    for v in (g.axis_nodes[0] ** 2, 3.0 * g.axis_nodes[0] - 0.5, np.abs(g.axis_nodes[0] - 8.0)):
        for scheme in ("first", "eno2", "eno3", "weno5"):
            pair = ref.derivative_pair(g, ref.ScalarField(v), 0, scheme)
            st.case(dict(grid=gspec((0.0,), (16.0,), (17,)), field="exact", scheme=scheme, axis=0,
                         eps_mode="squared"), v=v, left=pair.left.values, right=pair.right.values)
    st.save("derivs.npz")


def gen_workspace_divdiff(ref, rng):
    st = Store()
    for spec in (GRIDS[1], GRIDS[3], GRIDS[5]):
        g = make_grid(ref, spec)
        v = rng.standard_normal(g.counts)
        f = ref.ScalarField(v)
        for axis in range(g.dim):
            for side in ("left", "right"):
                for eps_mode in ("squared", "raw"):
                    ws = ref.weno5_workspace(g, f, axis, side=side, eps_mode=eps_mode)
                    st.case(dict(grid=spec, axis=axis, side=side, eps_mode=eps_mode, kind="workspace"), v=v,
                            **{k: getattr(ws, k) for k in ("sigma1", "sigma2", "sigma3", "alpha1", "alpha2",
                                                          "alpha3", "eps", "w1", "w2", "w3")})
            for order in (1, 2, 3):
                for width in (None, 3):
                    t = ref.divided_differences(g, f, axis, order=order, width=width)
                    arrays = {"v": v, "d0": t.d0, "d1": t.d1}
                    if t.d2 is not None:
                        arrays["d2"] = t.d2
                    if t.d3 is not None:
                        arrays["d3"] = t.d3
                    st.case(dict(grid=spec, axis=axis, order=order, width=width, kind="divdiff"), **arrays)
    st.save("spatial_extra.npz")


def term_configs(ref, scheme):
    rp = ref.RocketParams()
    return {
        "rockets": (ref.rockets_term_config(rp, scheme=scheme, hamiltonian="published"), 3),
        "rockets_extremal": (ref.rockets_term_config(rp, scheme=scheme, hamiltonian="extremal"), 3),
        "air3d": (air3d_config(ref, scheme), 3),
    }


def gen_term(ref, rng):
    st = Store()
    specs = {
        "advection": [gspec((-math.pi,), (math.pi,), (16,), periodic={0}),
                      gspec((0.0, 0.0), (1.0, 2.0), (9, 10), periodic={0, 1}),
                      gspec((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), (7, 6, 8), periodic={2}),
                      gspec((-1.0,) * 4, (1.0,) * 4, (5, 6, 5, 6))],
        "rockets": [gspec((-64.0, -64.0, -math.pi), (64.0, 64.0, math.pi), (9, 8, 10), periodic={2})],
        "air3d": [gspec(AIR3D["mins"], AIR3D["maxs"], (9, 10, 8), periodic={2})],
        "di4": [gspec(DI4["mins"], DI4["maxs"], (6, 5, 6, 7))],
    }
    speeds = {1: [2.0], 2: [3.0, -0.5], 3: [1.25, -0.75, 0.5], 4: [1.0, -2.0, 0.5, 0.25]}
    for scheme in ("first", "eno2", "eno3", "weno5"):
        cases = []
        for spec in specs["advection"]:
            g = make_grid(ref, spec)
            cases.append(("advection", spec, g, ref.advection_term_config(speeds[g.dim], scheme=scheme),
                          dict(speeds=speeds[g.dim])))
        for spec in specs["rockets"]:
            g = make_grid(ref, spec)
            for name, (cfg, _) in term_configs(ref, scheme).items():
                if name == "air3d":
                    continue
                cases.append((name, spec, g, cfg, {}))
        for spec in specs["air3d"]:
            g = make_grid(ref, spec)
            cases.append(("air3d", spec, g, air3d_config(ref, scheme), {}))
        for spec in specs["di4"]:
            g = make_grid(ref, spec)
            cases.append(("di4", spec, g, di4_config(ref, scheme), {}))
        for name, spec, g, cfg, extra in cases:
            for kind, v in fields(rng, g, ("random", "sdf")).items():
                if name != "advection":
                    v = 5.0 * v
                f = ref.ScalarField(v)
                out = ref.term_lax_friedrichs(0.0, f, cfg, g)
                derivs = [ref.derivative_pair(g, f, a, scheme) for a in range(g.dim)]
                _, alphas = ref.dissipation_glf(derivs, cfg.partials, 0.0, f, g)
                ranges = [(float(min(d.left.values.min(), d.right.values.min())),
                           float(max(d.left.values.max(), d.right.values.max()))) for d in derivs]
                arrays = dict(v=v, delta=out.delta.values, step_bound=np.array(out.step_bound),
                              alphas=alphas, ranges=np.array(ranges))
                if name in ("rockets", "rockets_extremal"):
                    arrays["cos"] = np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel()
                    arrays["sin"] = np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel()
                if name == "air3d":
                    vbc, vbs = air3d_tables(g)
                    arrays["cos"], arrays["sin"] = vbc, vbs
                st.case(dict(ham=name, grid=spec, scheme=scheme, field=kind, **extra), **arrays)
    st.save("term.npz")


def gen_hamiltonians(ref, rng):
    st = Store()
    g = ref.create_grid((-64, -64, -math.pi), (64, 64, math.pi), (7, 6, 8), periodic_axes={2})
    spec = gspec((-64, -64, -math.pi), (64, 64, math.pi), (7, 6, 8), periodic={2})
    params = ref.RocketParams()
    p = [rng.uniform(-2, 2, g.counts) for _ in range(3)]
    pf = [ref.ScalarField(x) for x in p]
    st.case(dict(ham="rockets", grid=spec), p0=p[0], p1=p[1], p2=p[2],
            H=ref.rockets_hamiltonian(0.0, g, None, pf, params).values,
            cos=np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel(),
            sin=np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel())
    st.case(dict(ham="rockets_extremal", grid=spec), p0=p[0], p1=p[1], p2=p[2],
            H=ref.rockets_hamiltonian_extremal(0.0, g, None, pf, params).values,
            cos=np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel(),
            sin=np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel())
    partials = [ref.rockets_partials(0.0, g, None, None, a, params) for a in range(3)]
    st.case(dict(ham="rockets_partials", grid=spec), alphas=np.array(partials))
    st.save("hamiltonian.npz")


def gen_integrate(ref, rng):
    st = Store()
    # advection, the reference's own integrator tests' setup
    g = ref.create_grid((0.0,), (2 * math.pi,), (40,), periodic_axes={0})
    spec = gspec((0.0,), (2 * math.pi,), (40,), periodic={0})
    y0 = np.sin(g.axis_nodes[0])
    for order, integ in ((1, ref.ode_cfl_1), (2, ref.ode_cfl_2), (3, ref.ode_cfl_3)):
        for scheme in ("first", "eno2", "weno5"):
            cfg = ref.advection_term_config([1.0], scheme=scheme)
            res = integ(lambda t, y, c: ref.term_lax_friedrichs(t, y, c, g), (0.0, 0.7), ref.ScalarField(y0),
                        ref.IntegratorOptions(cfl_factor=0.5), cfg)
            st.case(dict(ham="advection", speeds=[1.0], grid=spec, scheme=scheme, order=order, t0=0.0, t1=0.7,
                         cfl=0.5, max_step=None), y0=y0, y=res.y_final.values,
                    info=np.array([res.t_final, res.steps_taken, res.min_dt, res.max_dt]))
    # air3d, a few steps each order
    spec = gspec(AIR3D["mins"], AIR3D["maxs"], (11, 12, 10), periodic={2})
    g = make_grid(ref, spec)
    target = ref.cylinder(g, 2, (0.0, 0.0, 0.0), AIR3D["radius"])
    for order, integ in ((1, ref.ode_cfl_1), (2, ref.ode_cfl_2), (3, ref.ode_cfl_3)):
        for scheme in ("eno2", "weno5"):
            cfg = air3d_config(ref, scheme)
            res = integ(lambda t, y, c: ref.term_lax_friedrichs(t, y, c, g), (0.0, 0.05),
                        target, ref.IntegratorOptions(cfl_factor=0.5, max_step=0.02), cfg)
            vbc, vbs = air3d_tables(g)
            st.case(dict(ham="air3d", grid=spec, scheme=scheme, order=order, t0=0.0, t1=0.05, cfl=0.5,
                         max_step=0.02), y0=target.values, y=res.y_final.values, cos=vbc, sin=vbs,
                    info=np.array([res.t_final, res.steps_taken, res.min_dt, res.max_dt]))
    st.save("integrate.npz")


def gen_brt(ref, rng):
    st = Store()
    # the reference's own small rockets problem (test_reachability.py:193-199)
    spec = gspec((-64.0, -64.0, -math.pi), (64.0, 64.0, math.pi), (11, 11, 11), periodic={2})
    g = make_grid(ref, spec)
    params = ref.RocketParams(capture_radius=20.0)
    target = ref.cylinder(g, 2, (0.0, 0.0, 0.0), 20.0)
    for hname in ("published", "extremal"):
        cfg = ref.rockets_term_config(params, scheme="eno2", hamiltonian=hname)
        prob = ref.ReachProblem(grid=g, target=target, params=params, term_config=cfg, horizon=0.4,
                                global_steps=2)
        res = ref.solve_brt(prob)
        st.case(dict(ham="rockets" if hname == "published" else "rockets_extremal", grid=spec, scheme="eno2",
                     order=3, horizon=0.4, steps=2, radius=20.0, params=dict(capture_radius=20.0)),
                target=target.values, snaps=np.stack([s.values for s in res.snapshots]),
                times=np.array(res.times), cos=np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel(),
                sin=np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel())
    # Air3D through the reference solve_brt (RK3), WENO5 and ENO2
    spec = gspec(AIR3D["mins"], AIR3D["maxs"], (15, 15, 12), periodic={2})
    g = make_grid(ref, spec)
    target = ref.cylinder(g, 2, (0.0, 0.0, 0.0), AIR3D["radius"])
    vbc, vbs = air3d_tables(g)
    for scheme in ("weno5", "eno2", "eno3"):
        cfg = air3d_config(ref, scheme)
        prob = ref.ReachProblem(grid=g, target=target, params=ref.RocketParams(), term_config=cfg, horizon=0.3,
                                global_steps=3)
        res = ref.solve_brt(prob)
        st.case(dict(ham="air3d", grid=spec, scheme=scheme, order=3, horizon=0.3, steps=3), target=target.values,
                snaps=np.stack([s.values for s in res.snapshots]), times=np.array(res.times), cos=vbc, sin=vbs)
    # C1-style: Air3D ENO2 + odeCFL2 (solve_brt clone with RK2), 2 of the 8 intervals of [0, 2.8]
    spec = gspec(AIR3D["mins"], AIR3D["maxs"], (21, 21, 12), periodic={2})
    g = make_grid(ref, spec)
    target = ref.cylinder(g, 2, (0.0, 0.0, 0.0), AIR3D["radius"])
    vbc, vbs = air3d_tables(g)
    snaps, times, nsteps = brt_clone(ref, g, target, air3d_config(ref, "eno2"), 0.7, 2, order=2)
    st.case(dict(ham="air3d", grid=spec, scheme="eno2", order=2, horizon=0.7, steps=2), target=target.values,
            snaps=np.stack([s.values for s in snaps]), times=np.array(times), cos=vbc, sin=vbs,
            nsteps=np.array(nsteps))
    # 4-D double-integrator pair, ENO2 + RK3 and WENO5 + RK3
    spec = gspec(DI4["mins"], DI4["maxs"], (7, 7, 6, 6))
    g = make_grid(ref, spec)
    target = di4_target(ref, g)
    for scheme in ("eno2", "weno5"):
        snaps, times, nsteps = brt_clone(ref, g, target, di4_config(ref, scheme), 0.5, 2, order=3)
        st.case(dict(ham="di4", grid=spec, scheme=scheme, order=3, horizon=0.5, steps=2), target=target.values,
                snaps=np.stack([s.values for s in snaps]), times=np.array(times), nsteps=np.array(nsteps))
    st.save("brt.npz")


def gen_shapes(ref, rng):
    st = Store()
    spec = gspec((-2.0, -1.0, -math.pi), (2.0, 3.0, math.pi), (9, 10, 8), periodic={2})
    g = make_grid(ref, spec)
    sph = ref.sphere(g, (0.1, 0.5, 0.2), 1.2)
    cyl = ref.cylinder(g, 2, (0.0, 1.0, 0.0), 1.5)
    cyl0 = ref.cylinder(g, 0, (0.0, 1.0, 0.3), 0.9)
    ell = ref.ellipsoid(g, (1.0, 4.0, 9.0), 2.0)
    box = ref.hyper_rectangle(g, (-1.0, 0.0, -1.0), (0.5, 2.0, 1.5))
    st.case(dict(grid=spec, kind="shapes"), sphere=sph.values, cylinder=cyl.values, cylinder0=cyl0.values,
            ellipsoid=ell.values, box=box.values,
            union=ref.csg_union(sph, box).values, intersect=ref.csg_intersect(sph, box).values,
            complement=ref.csg_complement(cyl).values, difference=ref.csg_difference(box, sph).values,
            mesh0=ref.mesh_coordinates(g, 0).values, mesh2=ref.mesh_coordinates(g, 2).values,
            vol=np.array([ref.sublevel_volume(g, sph), ref.sublevel_volume(g, box, level=0.3)]))
    spec4 = gspec(DI4["mins"], DI4["maxs"], (6, 7, 5, 6))
    g4 = make_grid(ref, spec4)
    st.case(dict(grid=spec4, kind="di4_target"), target=di4_target(ref, g4).values)
    st.save("shapes.npz")


# plug-in contract (term.py:29-30 TermConfig callables) exercised through the
# integrator: range-dependent partials on the rockets Hamiltonian (two-pass
# GLF, each stage with its own costate ranges, term.py:71-83), Python-lambda
# Hamiltonians, and the error contract of _rhs (integrator.py:59-66).
# The formulas are restated in tests/test_gpu_plugins.py.
def range_partials(ref, params):
    def partials(t, g, v, ranges, i):
        base = ref.rockets_partials(t, g, v, ranges, i, params)
        return base + 0.01 * (abs(ranges[i][0]) + abs(ranges[i][1]))
    return partials


def lambda_ham(t, g, v, p):
    # a nonlinear Hamiltonian written the way the reference's tests write them
    x = np.asarray(g.axis_nodes[0]).reshape((-1,) + (1,) * (g.dim - 1))
    h = 0.5 * p[0].values * p[0].values - 0.25 * p[1].values + 0.1 * x * p[g.dim - 1].values
    return type(p[0])(h)


def lambda_partials(t, g, v, ranges, i):
    return max(abs(ranges[i][0]), abs(ranges[i][1])) + 0.5


def gen_plugins(ref, rng):
    st = Store()
    params = ref.RocketParams()
    spec = gspec((-64.0, -64.0, -math.pi), (64.0, 64.0, math.pi), (9, 8, 10), periodic={2})
    g = make_grid(ref, spec)
    target = ref.cylinder(g, 2, (0.0, 0.0, 0.0), 15.0)
    for scheme in ("eno2", "weno5"):
        base = ref.rockets_term_config(params, scheme=scheme)
        cfg = ref.TermConfig(hamiltonian=base.hamiltonian, partials=range_partials(ref, params),
                             derivative_scheme=scheme)
        res = ref.ode_cfl_3(lambda t, y, c: ref.term_lax_friedrichs(t, y, c, g), (0.0, 0.05), target,
                            ref.IntegratorOptions(cfl_factor=0.5), cfg)
        st.case(dict(kind="rockets_range_partials", grid=spec, scheme=scheme, t1=0.05), y0=target.values,
                y=res.y_final.values, info=np.array([res.t_final, res.steps_taken, res.min_dt, res.max_dt]),
                cos=np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel(),
                sin=np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel())
    spec2 = gspec((-1.0, -1.0), (1.0, 2.0), (12, 14), periodic={1})
    g2 = make_grid(ref, spec2)
    y0 = np.sin(np.pi * ref_mesh(g2, 0)) * np.cos(ref_mesh(g2, 1)) + 0.1 * ref_mesh(g2, 1)
    for scheme in ("first", "eno3", "weno5"):
        cfg = ref.TermConfig(hamiltonian=lambda_ham, partials=lambda_partials, derivative_scheme=scheme)
        res = ref.ode_cfl_3(lambda t, y, c: ref.term_lax_friedrichs(t, y, c, g2), (0.0, 0.08),
                            ref.ScalarField(y0), ref.IntegratorOptions(cfl_factor=0.4), cfg)
        st.case(dict(kind="lambda_ham", grid=spec2, scheme=scheme, t1=0.08, cfl=0.4), y0=y0,
                y=res.y_final.values, info=np.array([res.t_final, res.steps_taken, res.min_dt, res.max_dt]))
    # the error contract: what the reference raises, verbatim
    errs = {
        "invalid_bound": ref.TermConfig(hamiltonian=lambda_ham, partials=lambda *a: -1.0, derivative_scheme="eno2"),
        "nan_hamiltonian": ref.TermConfig(hamiltonian=lambda t, g, v, p: np.full(p[0].values.shape, np.nan),
                                          partials=lambda *a: 1.0, derivative_scheme="eno2"),
    }
    for name, cfg in errs.items():
        try:
            ref.ode_cfl_3(lambda t, y, c: ref.term_lax_friedrichs(t, y, c, g2), (0.0, 0.08), ref.ScalarField(y0),
                          ref.IntegratorOptions(cfl_factor=0.4), cfg)
            raise AssertionError(f"{name}: the reference did not raise")
        except (RuntimeError, ValueError) as err:
            st.case(dict(kind="error", name=name, grid=spec2, error=type(err).__name__, message=str(err)), y0=y0)
    # the same invalid bound on a REGISTERED Hamiltonian (rockets), range-dependent partials
    base = ref.rockets_term_config(params, scheme="eno2")
    cfg = ref.TermConfig(hamiltonian=base.hamiltonian, partials=lambda t, g, v, r, i: -2.0 if i == 1 else 1.0,
                         derivative_scheme="eno2")
    try:
        ref.ode_cfl_3(lambda t, y, c: ref.term_lax_friedrichs(t, y, c, g), (0.0, 0.05), target,
                      ref.IntegratorOptions(), cfg)
        raise AssertionError("rockets invalid bound: the reference did not raise")
    except (RuntimeError, ValueError) as err:
        st.case(dict(kind="error", name="rockets_invalid_bound", grid=spec, error=type(err).__name__,
                     message=str(err)), y0=target.values, cos=np.cos(g.axis_nodes[2].reshape(1, 1, -1)).ravel(),
                sin=np.sin(g.axis_nodes[2].reshape(1, 1, -1)).ravel())
    st.save("plugins.npz")


def main():
    root = sys.argv[1] if len(sys.argv) > 1 else "/root/reference"
    ref = load_reference(root)
    if len(sys.argv) > 2:   # e.g. `make_golden.py /root/reference plugins`: one generator only
        globals()[f"gen_{sys.argv[2]}"](ref, np.random.default_rng(20241103))
        return
    rng = np.random.default_rng(20241103)
    gen_grid_and_ghost(ref, rng)
    gen_derivs(ref, rng)
    gen_workspace_divdiff(ref, rng)
    gen_term(ref, rng)
    gen_hamiltonians(ref, rng)
    gen_integrate(ref, rng)
    gen_brt(ref, rng)
    gen_shapes(ref, rng)
    gen_plugins(ref, np.random.default_rng(20241103))


if __name__ == "__main__":
    main()
