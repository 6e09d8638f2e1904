"""Development aid: BF16EMU fine apply at N^3 -- record-fed tcgen05 kernel vs the
per-element one (SG_BF16_TC1=1 in the environment) -- CUDA-event time per launch
(sg_hier_profile target 5, L2 flushed), and max deviation from the dense
CUDA-core kernel."""
import ctypes, sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("binary", N, N, N, vf=0.5, seed=3), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "bf16")
out = ctypes.c_double()
_native.check(_native.load().sg_hier_profile(h._hh, 5, 20, ctypes.byref(out), _dev.stream()))
print(f"BF16 apply {N}^3: {out.value * 1e3:.1f} us")
