"""Development aid: one FP32-GMG PCG solve at N^3 (after warm-up) inside
cudaProfilerStart/Stop, for an ncu --profile-from-start off launch list."""
import sys, warnings
sys.path.insert(0, ".")
import torch
import paper_2604_26441_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
b = torch.from_numpy(g.load[g.free_dofs]).cuda()
cfg = P.SolverConfig(tol=1e-6, maxiter=200)
P.pcg(op.matvec, h.vcycle, b, cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
rep = P.pcg(op.matvec, h.vcycle, b, cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("iters", rep.iterations)
