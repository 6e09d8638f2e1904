"""Development aid: per-phase timing of one pcg80 step (block 0, %globaltimer)."""
import ctypes, sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
lib = _native.load()
lib.sg_hier_pcg80_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
h.vcycle(np.ones(g.n_free))
names = ["phaseA", "reduceA", "phaseB", "reduceB"]
for rep in range(3):
    t = np.zeros(9, dtype=np.int64)
    _native.check(lib.sg_hier_pcg80_trace(h._hh, t.ctypes.data, _dev.stream()))
    d = np.diff(t)
    print(" ".join(f"{n}={v/1e3:.2f}us" for n, v in zip(names, d[:4])), f"total={(t[4]-t[0])/1e3:.2f}us")
