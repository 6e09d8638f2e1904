"""Development aid: wall time of build_hierarchy (fp32 policy) at N^3, repeated."""
import sys, time, warnings
sys.path.insert(0, ".")
import torch
import paper_2604_26441_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, 4, "fp32")
    torch.cuda.synchronize()
    print(f"build {i}: {time.perf_counter() - t0:.3f} s")
    del h
