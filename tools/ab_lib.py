"""Development aid: FP32 fine apply output for a grid (compare across library builds)."""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
dims = tuple(int(v) for v in sys.argv[2].split(","))
g = P.build_cantilever(*dims)
op = P.FineOperator(g, P.simp_modulus(P.make_state("random_floor", *dims, vf=0.5, seed=42), 3.0))
tag = sys.argv[3] if len(sys.argv) > 3 else "fp32"
u = P.SplitMix64(3).gaussian(g.n_free)
if tag == "fp64":
    np.save(sys.argv[1], op.matvec(u))
else:
    np.save(sys.argv[1], op.matvec_tagged(u.astype(np.float32), P.PrecisionTag.FP32))
