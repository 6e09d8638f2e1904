"""Development aid: coarsest pcg80 cost vs step count (isolates per-step cost)."""
import ctypes, sys, warnings
sys.path.insert(0, ".")
import torch
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
for steps in (0, 1, 10, 80):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, 4, "fp32", coarse_pcg_steps=steps)
    out = ctypes.c_double()
    _native.check(_native.load().sg_hier_profile(h._hh, 3, 10, ctypes.byref(out), _dev.stream()))
    print(f"pcg steps {steps:3d}: coarsest solve {out.value*1e3:8.1f} us")
