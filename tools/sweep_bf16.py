"""BASELINE configs[2]: guarded BF16-GMG (FGMRES) vs the Lanczos epsilon*kappa screen
on the binary sweep (bench/runner.py:319-343 cell recipe: FP64 hierarchy probe,
BF16 hierarchy FGMRES).  python tools/sweep_bf16.py 80 [--restart 50 --maxiter 500]
"""
import argparse, json, sys, time, warnings
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("N", type=int)
ap.add_argument("--restart", type=int, default=50)
ap.add_argument("--maxiter", type=int, default=500)
ap.add_argument("--cells", default="all")
args = ap.parse_args()
N = args.N
for vf in (0.2, 0.5, 0.8):
    for p in (1.5, 3.0, 4.5):
        g = P.build_cantilever(N, N, N)
        op = P.FineOperator(g, P.simp_modulus(P.make_state("binary", N, N, N, vf=vf, floor=1e-2, seed=42), p))
        b = g.load[g.free_dofs]
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            h64 = P.build_hierarchy(op, 4, "fp64")
            probe = P.lanczos_kappa_eff(P.PreconditionedOperator(op, h64), g.n_free, 40, 0)
            h16 = P.build_hierarchy(op, 4, "bf16")
        t1 = time.perf_counter()
        rep = P.fgmres(op.matvec, h16.vcycle, b, P.SolverConfig(method="fgmres", tol=1e-6,
                                                                 maxiter=args.maxiter, restart=args.restart))
        print(json.dumps({"vf": vf, "p": p, "kappa_eff": round(probe.kappa_eff, 4),
                          "eps_kappa": round(probe.eps_kappa, 4), "screen": P.bf16_screen(probe),
                          "iters": rep.iterations, "conv": rep.converged, "kind": rep.failure_kind,
                          "true": rep.final_true_residual, "probe_s": round(t1 - t0, 3),
                          "solve_s": round(rep.wall_time, 3)}), flush=True)
