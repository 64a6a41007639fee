"""Conditioning probe for the tolerance-mode WENO5: full-horizon Air3D tubes,
exact vs fma vs exact with a 1-ulp perturbed target; per-snapshot L-inf rel
and where the largest difference sits."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import sys
import numpy as np
import paper_2411_03501_b200 as hj

n = int(sys.argv[1]) if len(sys.argv) > 1 else 301
g = hj.air3d_grid(n)
target = hj.cylinder(g, 2, (0.0, 0.0, 0.0), 5.0)
pert = hj.ScalarField(np.nextafter(target.values, np.inf))
ex = hj.solve_tube(g, target, hj.air3d_term_config(scheme="weno5"), 2.8, 8, order=3)
fm = hj.solve_tube(g, target, hj.air3d_term_config(scheme="weno5_fma"), 2.8, 8, order=3)
pe = hj.solve_tube(g, pert, hj.air3d_term_config(scheme="weno5"), 2.8, 8, order=3)
for name, other in (("fma", fm), ("exact+1ulp", pe)):
    for k, (a, b) in enumerate(zip(other.snapshots, ex.snapshots)):
        a, b = a.values, b.values
        d = np.abs(a - b)
        scale = np.max(np.abs(b))
        i = np.unravel_index(np.argmax(d), d.shape)
        print(f"{name:11s} snap {k} linf_rel {d.max()/scale:.3e}  n>1e-12rel {int(np.sum(d > 1e-12*scale)):8d} "
              f"at {i} V={b[i]:.6g} prevV={ex.snapshots[max(k-1,0)].values[i]:.6g} "
              f"signdiff(|V|>=1e-9) {int(np.sum((np.sign(a)!=np.sign(b)) & (np.abs(b)>=1e-9)))}", flush=True)
