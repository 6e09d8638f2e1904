"""Development aid: FP64 V-cycle vs the oracle for smoother degree / depth combinations."""
import sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
from oracle import simp_oracle as O
dims = (8, 4, 4)
g = P.build_cantilever(*dims)
rho = P.make_state("uniform", *dims, vf=0.5, seed=42)
op = P.FineOperator(g, P.simp_modulus(rho, 3.0))
og, E, ke = O.problem(*dims, kind="uniform", vf=0.5, p=3.0, seed=42)
r = P.SplitMix64(7).gaussian(g.n_free)
for deg in (2, 3):
    for lev in (2, 3):
        for kind in ("chebyshev", "jacobi"):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                h = P.build_hierarchy(op, lev, "fp64", P.SmootherConfig(kind=kind, degree=deg))
            oh = O.Hier(og, E, ke, lev, "fp64", smoother=(kind, deg, 1 / 30, 0.5))
            a, b = h.vcycle(r), oh.vcycle(r)
            print(kind, "deg", deg, "levels", lev, "rel", np.linalg.norm(a - b) / np.linalg.norm(b),
                  "lams", [l.lam_max for l in h.levels], [l.lam for l in oh.levels])
