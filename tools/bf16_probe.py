"""Development aid: the BF16EMU level-0 apply (tcgen05 kernel) at N^3, for ncu."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_26441_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
u = torch.from_numpy(P.SplitMix64(4).gaussian(g.n_free).astype(np.float32)).cuda()
for _ in range(3):
    y = op.matvec_tagged(u, P.PrecisionTag.BF16EMU)
torch.cuda.synchronize()
