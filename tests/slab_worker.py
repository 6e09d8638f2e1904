"""One rank of the multi-process slab tests (launched by tests/test_slab_*.py).

usage: python tests/slab_worker.py MODE OUT_JSON   (RANK / WORLD_SIZE /
MASTER_ADDR / MASTER_PORT in the environment; gloo backend)

MODE comm  -- CPU: TorchSlabComm halo / allreduce / allgather against a known
              global vector.
MODE solve -- GPU (all ranks on cuda:0): SlabSolver matvec, V-cycle and PCG
              against the single-process native path on the same problem.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def _comm_case(out):
    from paper_2604_26441_b200.slab import TorchSlabComm, slab_plan
    rank, world = dist.get_rank(), dist.get_world_size()
    res = {}
    for nz, n_dist in ((8, 2), (12, 2), (7, 1)):
        plan = slab_plan(nz, world, n_dist)
        psz = [3 * 5 * 4, 3 * 3 * 3][:n_dist]
        full_planes = [nz + 1, nz // 2 + 1][:n_dist]
        comm = TorchSlabComm(plan, psz, full_planes)
        for lvl in range(n_dist):
            w = plan[lvl][rank]
            ps = psz[lvl]
            glob = torch.arange(full_planes[lvl] * ps, dtype=torch.float64) * 0.5 + lvl
            win = glob[w.w0 * ps:(w.w1 + 1) * ps].clone()
            own = slice((w.o0 - w.w0) * ps, (w.o1 - w.w0) * ps)
            ghost = torch.ones_like(win, dtype=torch.bool)
            ghost[own] = False
            win[ghost] = -1.0  # stale ghosts
            comm.halo(lvl, win)
            ok_halo = bool(torch.equal(win, glob[w.w0 * ps:(w.w1 + 1) * ps]))
            full = torch.full_like(glob, float("nan"))
            comm.allgather(lvl, win, full)
            ok_gather = bool(torch.equal(full, glob))
            res[f"{nz}_{n_dist}_{lvl}"] = [ok_halo, ok_gather]
        vals = torch.tensor([1.0 + rank, 0.1 * (rank + 1), -rank], dtype=torch.float64)
        comm.allreduce(vals)
        exp = torch.zeros(3, dtype=torch.float64)
        for r in range(world):
            exp += torch.tensor([1.0 + r, 0.1 * (r + 1), -r], dtype=torch.float64)
        res[f"sum_{nz}"] = bool(torch.equal(vals, exp))
    return res


def _solve_case(out):
    import paper_2604_26441_b200 as P
    from paper_2604_26441_b200.slab import SlabSolver
    rank = dist.get_rank()
    res = {}
    cases = [(16, 8, 8, "uniform", 3.0, "fp32"), (24, 8, 12, "binary", 3.0, "fp32"),
             (16, 8, 16, "binary", 1.5, "bf16")]
    for nx, ny, nz, kind, p, policy in cases:
        g = P.build_cantilever(nx, ny, nz)
        E = P.simp_modulus(P.make_state(kind, nx, ny, nz, vf=0.5, floor=1e-2, seed=42), p)
        op = P.FineOperator(g, E)
        h = P.build_hierarchy(op, 4, policy)
        b = g.load[g.free_dofs]
        rng = np.random.default_rng(7)
        x = rng.standard_normal(g.n_free)
        cfg = P.SolverConfig(tol=1e-6, maxiter=200)
        key = f"{nx}x{ny}x{nz}_{kind}_{policy}"
        for n_dist in (1, 2):
            s = SlabSolver(op, h, n_dist=n_dist, transport=os.environ.get("SLAB_TRANSPORT", "torch"))
            kx = s.matvec(x)
            vx = s.vcycle(x)
            rep = s.pcg(b, cfg)
            rep1 = P.pcg(op.matvec, h.vcycle, b, cfg)
            kx1 = op.matvec(x)
            vx1 = h.vcycle(x)
            res[f"{key}_d{n_dist}"] = {
                "matvec_equal": bool(np.array_equal(kx, kx1)),
                "matvec_rel": float(np.abs(kx - kx1).max() / np.abs(kx1).max()),
                "vcycle_equal": bool(np.array_equal(vx, vx1)),
                "vcycle_rel": float(np.abs(vx - vx1).max() / np.abs(vx1).max()),
                "iters": rep.iterations, "iters1": rep1.iterations,
                "conv": rep.converged, "conv1": rep1.converged,
                "hist_equal": rep.residual_history == rep1.residual_history,
                "hist_rel": float(max(abs(a - c) / c for a, c in
                                      zip(rep.residual_history, rep1.residual_history))),
                "x_rel": float(np.abs(rep.x - rep1.x).max() / np.abs(rep1.x).max()),
                "true_res": rep.final_true_residual,
                "halos": s.comm.n_halo if s.comm else -1,
                "gathers": s.comm.n_gather if s.comm else -1,
                "sums": s.comm.n_sum if s.comm else -1,
                "transport": s.transport,
            }
            if n_dist == 2 and policy == "fp32":
                rf = s.fgmres(b, P.SolverConfig(method="fgmres", tol=1e-6, maxiter=200, restart=32))
                rf1 = P.fgmres(op.matvec, h.vcycle, b,
                               P.SolverConfig(method="fgmres", tol=1e-6, maxiter=200, restart=32))
                res[f"{key}_d{n_dist}"].update({"fg_iters": rf.iterations,
                                                "fg_iters1": rf1.iterations,
                                                "fg_conv": rf.converged})
            s.close()
        # release_full: the hierarchy's replicated slab levels freed; the slab
        # solve must not depend on them (same x as the solve above, bit for bit)
        s = SlabSolver(op, h, n_dist=2, transport=os.environ.get("SLAB_TRANSPORT", "torch"),
                       release_full=True)
        rep_r = s.pcg(b, cfg)
        res[f"{key}_released"] = {"x_equal": bool(np.array_equal(rep_r.x, rep.x)),
                                  "iters": rep_r.iterations}
        try:
            h.vcycle(x)
            res[f"{key}_released"]["vcycle_raises"] = False
        except Exception:
            res[f"{key}_released"]["vcycle_raises"] = True
        s.close()
    return res


def main():
    mode, out = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    if mode == "solve":
        torch.cuda.set_device(0)
    res = _comm_case(out) if mode == "comm" else _solve_case(out)
    allres = [None] * dist.get_world_size()
    dist.all_gather_object(allres, res)
    if dist.get_rank() == 0:
        with open(out, "w") as f:
            json.dump(allres, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
