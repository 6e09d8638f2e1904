"""Development aid: fixed cost of the coarsest pcg80 launch -- steps 0/1/80, after
the L2-flush memset (3), after another coarsest solve (8), after the restriction (9)."""
import ctypes, sys, warnings
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
for steps in (0, 1, 80):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, 4, "fp32", coarse_pcg_steps=steps)
    res = []
    for what in (3, 8, 9):
        out = ctypes.c_double()
        _native.check(_native.load().sg_hier_profile(h._hh, what, 20, ctypes.byref(out), _dev.stream()))
        res.append(out.value * 1e3)
    print(f"steps {steps:3d}: after memset {res[0]:7.1f} us, after pcg80 {res[1]:7.1f} us, "
          f"after restrict {res[2]:7.1f} us")
