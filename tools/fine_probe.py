"""Development aid: run the fine FP32/FP64 applies at N^3 (for ncu captures)
and print CUDA-event timings of each kernel variant."""
import ctypes, os, sys, warnings
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_26441_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
u = torch.from_numpy(P.SplitMix64(4).gaussian(g.n_free).astype(np.float32)).cuda()
u64 = u.double()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for warm in (False, True):
  for tag, x in ((P.PrecisionTag.FP32, u), (P.PrecisionTag.FP64, u64)):
    y = op.matvec_tagged(x, tag)
    ts = []
    for r in range(reps):
        if not warm:
            flush.fill_(r & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        e0.record(s)
        y = op.matvec_tagged(x, tag)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{'warm' if warm else 'cold'} {tag}: median {np.median(ts):.1f} us (incl. free<->node gathers), min {min(ts):.1f}")
