"""Development aid: one launch each of the level-0 P32 kernels at N^3 on seeded
gaussian inputs (sg_hier_profile targets 0 plain apply, 6 apply + Chebyshev step,
7 apply + residual), for an ncu capture of exactly these three launches."""
import ctypes, sys, warnings
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
lib = _native.load()
import torch
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()  # (ncu --profile-from-start off: these launches only)
for what, name in ((0, "plain apply"), (6, "apply + Chebyshev step"), (7, "apply + residual"), (1, "FP64 apply")):
    out = ctypes.c_double()
    _native.check(lib.sg_hier_profile(h._hh, what, reps, ctypes.byref(out), _dev.stream()))
    print(f"{name:24s} {out.value*1e3:9.1f} us")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
