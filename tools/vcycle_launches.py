"""Development aid: one V-cycle at N^3 (after warm-up) for an ncu launch list."""
import sys, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
r = P.SplitMix64(5).gaussian(g.n_free)
h.vcycle(r)
import torch
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
h.vcycle(r)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
