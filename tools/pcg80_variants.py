"""Development aid: V-cycle differences between the pcg80 variants at N^3
(brick Chronopoulos-Gear default, brick Hestenes-Stiefel SG_PCG80_HS=1,
contiguous-range kernel SG_PCG80_RANGE=1) and per-variant coarsest time."""
import ctypes, os, sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
r = P.SplitMix64(5).gaussian(g.n_free)
out = {}
for name, env in (("pipe", {}), ("cg", {"SG_PCG80_CG": "1"}), ("hs", {"SG_PCG80_HS": "1"}), ("range", {"SG_PCG80_RANGE": "1"})):
    for k in ("SG_PCG80_CG", "SG_PCG80_HS", "SG_PCG80_RANGE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, 4, "fp32")
    out[name] = h.vcycle(r)
    t = ctypes.c_double()
    _native.check(_native.load().sg_hier_profile(h._hh, 3, 20, ctypes.byref(t), _dev.stream()))
    print(f"{name:6s} coarsest {t.value*1e3:8.1f} us")
    b = g.load[g.free_dofs]
    rep = P.pcg(op.matvec, h.vcycle, b, P.SolverConfig(tol=1e-6, maxiter=200))
    print(f"       pcg iters {rep.iterations} true res {rep.final_true_residual:.4e} hist[-1] {rep.residual_history[-1]:.6e}")
for a, b in (("pipe", "range"), ("cg", "range"), ("hs", "range"), ("pipe", "hs")):
    d = np.linalg.norm(out[a] - out[b]) / np.linalg.norm(out[b])
    print(f"vcycle rel diff {a} vs {b}: {d:.3e}")
