"""Development aid: device time of the hot kernels at N^3 via sg_hier_profile
(L2 flushed before every repetition), plus the same without the flush."""
import ctypes, sys, warnings
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
lib = _native.load()
for what, name in ((0, "fine_apply_fp32"), (1, "fine_apply_fp64"), (2, "level1_spmv"), (3, "coarsest"), (4, "vcycle")):
    out = ctypes.c_double()
    _native.check(lib.sg_hier_profile(h._hh, what, 20, ctypes.byref(out), _dev.stream()))
    print(f"{name:18s} {out.value*1e3:9.1f} us")
