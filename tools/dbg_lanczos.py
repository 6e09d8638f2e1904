"""Development aid: Lanczos kappa sensitivity (native vs generic path, perturbed start)."""
import sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
dims = (8, 4, 4)
g = P.build_cantilever(*dims)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", *dims, vf=0.5, seed=42), 3.0))
for deg, lev in ((2, 3), (3, 2), (3, 3)):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, lev, "fp64", P.SmootherConfig(kind="chebyshev", degree=deg))
    nat = P.lanczos_kappa_eff(P.PreconditionedOperator(op, h), g.n_free, 40, 0)
    gen = P.lanczos_kappa_eff(lambda v: h.vcycle(op.matvec(v)), g.n_free, 40, 0)
    gen2 = P.lanczos_kappa_eff(lambda v: h.vcycle(op.matvec(v)) * (1 + 1e-15), g.n_free, 40, 0)
    print(deg, lev, nat.kappa_eff, gen.kappa_eff, gen2.kappa_eff, nat.lambda_min, gen.lambda_min)
