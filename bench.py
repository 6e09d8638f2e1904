"""Benchmark of the PCG / GMG hot path (BASELINE.json metric).

Workload (configs[3]): 100x100x100 (1M elements) cantilever, uniform rho=0.5,
p=3, FP32-GMG (policy "fp32", 4 levels requested -> 3 after the odd-dim
clamp, pcg80 coarsest), PCG to tol 1e-6, cap 200.  One step = one full PCG
solve; the hierarchy is built once outside the timed region ("setup
excluded", as the metric says).  value = seconds per solve (device time,
CUDA events on the launch stream, max over ranks); e2e = the same solve
through the public Python API with the right-hand side in host memory and
the solution copied back (H2D + D2H inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--size 100]

--impl reference times the CPU oracle port (oracle/simp_oracle.py, a numpy/
scipy restatement of the reference package, which is pure Python and so has
no compiled artefact) on the host cores: one step = one PCG iteration of the
same 100^3 problem (V-cycle + FP64 fine apply + vector updates), scaled by
the oracle's own iteration count to seconds per solve.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
import warnings

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._proc = None
        self._path = None

    def __enter__(self):
        # one long-lived nvidia-smi sampling every 200 ms into a file: no
        # process spawns or GIL traffic inside the timed region
        import tempfile
        fd, self._path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "200", "-f", self._path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self._proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        try:
            with open(self._path) as fh:
                for line in fh:
                    if line.strip():
                        self.rows.append([v.strip() for v in line.split(",")])
            os.remove(self._path)
        except Exception:
            pass

    def summary(self):
        import statistics
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def oracle_iterations(N, steps, warmup, full_solve=False):
    """Time `steps` PCG iterations (krylov.py:135-164 loop body: FP64 fine apply,
    dots, axpys, V-cycle) of the CPU oracle at N^3 after `warmup` untimed ones."""
    import numpy as np
    from oracle import simp_oracle as O
    t0 = time.perf_counter()
    g, E, ke = O.problem(N, N, N)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = O.Hier(g, E, ke, 4, "fp32")
    setup = time.perf_counter() - t0
    b = g.load[g.free]
    Kf = lambda v: O.fine_apply(g, E, ke, v, "fp64")
    full = O.pcg(Kf, h.vcycle, b, 1e-6, 200) if full_solve else None
    x = np.zeros_like(b)
    r = b.copy()
    p = h.vcycle(r)
    rz = float(r @ p)
    samples = []
    for k in range(warmup + steps):
        s = time.perf_counter()
        q = Kf(p)
        a = rz / float(p @ q)
        x = x + a * p
        r = r - a * q
        float(np.linalg.norm(r) / np.linalg.norm(b))
        z = h.vcycle(r)
        rzn = float(r @ z)
        p = z + (rzn / rz) * p
        rz = rzn
        if k >= warmup:
            samples.append(time.perf_counter() - s)
    return {"per_iter_s": sum(samples) / len(samples), "setup_s": setup,
            "iters_timed": len(samples), "full": full}


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    N = args.size
    res = oracle_iterations(N, args.steps, args.warmup, full_solve=True)
    full = res["full"]
    n_iters = full.iterations
    per_iter = res["per_iter_s"]
    setup = res["setup_s"]
    value = per_iter * n_iters
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_iter * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64/f32 (FP32-GMG)", "data": "synthetic",
        "config": _config(args),
        "cpu_baseline": {"value": value, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{res['iters_timed']} PCG iterations (V-cycle + FP64 apply) of the "
                                   f"{N}^3 oracle, scaled by its {n_iters}-iteration full solve"},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "oracle_setup_s": setup,
        "oracle_full_solve_s": full.wall_time,
        "oracle_iterations": n_iters,
        "oracle_converged": bool(full.converged),
    }
    print(json.dumps(line))
    return 0


METRIC = "GMG-PCG solve s at 1M elements; fine matvec achieved HBM GB/s; PCG iters"


def _config(args):
    N = args.size
    return {"workload": f"{N}x{N}x{N} uniform rho=0.5 p=3 cantilever, FP32-GMG PCG (tol 1e-6, cap 200)",
            "elements": N ** 3, "levels_requested": 4, "policy": "fp32",
            "parallelism": (f"z-slab partition x{args.gpus} (levels 0-1; {args.transport} transport: "
                            + ("device kernels over CUDA IPC mailboxes, " if args.transport == "peer" else "NCCL via torch.distributed, ")
                            + "halos + rank-ordered dot sums; coarse tail replicated)") if (args.gpus > 1 or args.slab) else "single GPU",
            "l2": "working set > 126 MB L2 (level-1 operator 258 MB, its symmetric copy 133 MB); L2 also flushed before each timed solve"}


def run_gpu(args):
    import ctypes

    import numpy as np
    import torch

    world, rank, local = _dist()
    # development knob: SG_BENCH_ONE_DEVICE=1 runs every rank on cuda:0 over
    # gloo (the multi-rank path on a one-GPU box; the peer transport maps the
    # other processes' mailboxes through IPC on the same device)
    one_dev = os.environ.get("SG_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    use_slab = world > 1 or args.slab
    if use_slab:
        import torch.distributed as dist
        if "MASTER_ADDR" not in os.environ:  # --slab on one process without torchrun
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2604_26441_b200 as P
    from paper_2604_26441_b200 import _dev, _native

    lib = _native.load()
    N = args.size
    g = P.build_cantilever(N, N, N)
    op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
    # setup: the first build in the process is "cold" (lazy module loading of
    # every kernel, cudaFuncSetAttribute, first allocations); the second "warm"
    # build is the steady-state cost of a new hierarchy (e.g. per SIMP step)
    setup = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            h = P.build_hierarchy(op, 4, "fp32")
        torch.cuda.synchronize()
        setup.append(time.perf_counter() - t0)
    setup_s = setup[1]
    b_host = np.ascontiguousarray(g.load[g.free_dofs])
    b_dev, _ = _dev.as_device(b_host)
    cfg = P.SolverConfig(tol=1e-6, maxiter=200)
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    # per-component device timings (CUDA events inside the library), taken
    # before a slab solver may release the hierarchy's replicated levels
    def prof(what, reps=10):
        out = ctypes.c_double()
        _native.check(lib.sg_hier_profile(h._hh, what, reps, ctypes.byref(out), _dev.stream()))
        return out.value

    n_free, n_elem = g.n_free, g.n_elem
    nn1 = (N // 2 + 1) ** 3
    comps = {}
    t32 = prof(0)
    t64 = prof(1)
    tl1 = prof(2)
    tco = prof(3)
    tvc = prof(4)
    tbf = prof(5)
    try:
        tch = prof(6)
    except Exception:
        tch = None
    peak, peak_kind = _peaks()
    b32 = 8 * n_free + 4 * n_elem
    b64 = 16 * n_free + 8 * n_elem
    # level-1 SpMV on the symmetric stencil copy (126 of 243 coefficients per
    # node from HBM; SG_ST64_FULL=1 selects the full 243)
    bl1 = ((243 if os.environ.get("SG_ST64_FULL") else 126) * 8 + 48) * nn1
    comps["fine_apply_fp32"] = {"ms": t32, "alg_bytes": b32, "gbs": b32 / t32 / 1e6}
    comps["fine_apply_fp64"] = {"ms": t64, "alg_bytes": b64, "gbs": b64 / t64 / 1e6}
    comps["fine_apply_bf16_tcgen05"] = {"ms": tbf, "alg_bytes": b32, "gbs": b32 / tbf / 1e6}
    if tch is not None:
        # fused apply + Chebyshev step: u, E in; b, dinv, d in; d, x' out (FP32)
        bch = 24 * n_free + 4 * n_elem
        comps["fine_apply_cheb_fused_fp32"] = {"ms": tch, "alg_bytes": bch, "gbs": bch / tch / 1e6}
    comps["level1_spmv_fp64"] = {"ms": tl1, "alg_bytes": bl1, "gbs": bl1 / tl1 / 1e6}
    comps["coarsest_pcg80"] = {"ms": tco}
    comps["vcycle"] = {"ms": tvc}
    if use_slab:
        # slab partition of levels 0-1 over the ranks (NCCL halos / dot sums),
        # coarse tail replicated (paper_2604_26441_b200/slab.py)
        from paper_2604_26441_b200.slab import SlabSolver
        try:
            slab = SlabSolver(op, h, transport=args.transport, release_full=True)
        except Exception as exc:  # e.g. no CUDA IPC between these devices: host transport
            if args.transport != "peer":
                raise
            print(f"peer transport unavailable ({exc!r}); using torch.distributed", file=sys.stderr)
            args.transport = "torch"
            slab = SlabSolver(op, h, transport="torch", release_full=True)
        solve = lambda b: slab.pcg(b, cfg)
    else:
        solve = lambda b: P.pcg(op.matvec, h.vcycle, b, cfg)

    for _ in range(args.warmup):
        rep = solve(b_dev)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = lib.sg_launch_count()
    total_ms = 0.0
    iters = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = solve(b_dev)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            iters.append(rep.iterations)
    launches = int(lib.sg_launch_count() - launches0)
    torch.cuda.synchronize()
    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cpu" if one_dev else "cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()

    # end to end through the public API with HOST buffers (the drop-in call):
    #  * "pinned": P.pcg(op.matvec, h.vcycle, b) with b a pinned host tensor (the
    #    H2D copy happens inside the call), then the solution copied into pinned
    #    host memory (D2H);
    #  * "numpy": the reference's own calling convention (krylov.py:113): numpy b
    #    in, numpy x out (pageable copies inside the call).
    # Wall clock around the call, median of >= 10 samples, L2 flushed before each.
    # The phase split (H2D / solve / D2H) is measured separately with CUDA events.
    b_pin = torch.from_numpy(b_host).pin_memory()
    x_pin = torch.empty(b_pin.shape, dtype=b_pin.dtype, pin_memory=True)
    n_e2e = max(10, args.steps)

    def wall(fn):
        out = []
        fn()  # untimed warm-up of this path
        for _ in range(n_e2e):
            flush.zero_()
            torch.cuda.synchronize()
            s = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            out.append(time.perf_counter() - s)
        return out

    def e2e_pinned():
        r = solve(b_pin)
        x_pin.copy_(r.x, non_blocking=False)

    e2e = wall(e2e_pinned)
    e2e_np = wall(lambda: solve(b_host)) if not use_slab else []
    assert np.allclose(x_pin.numpy(), rep.x.cpu().numpy())
    phases = {"h2d_ms": [], "solve_ms": [], "d2h_ms": []}
    for _ in range(n_e2e):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        bd = b_pin.to("cuda", non_blocking=True)
        ev[1].record(stream)
        r = solve(bd)
        ev[2].record(stream)
        x_pin.copy_(r.x, non_blocking=True)
        ev[3].record(stream)
        ev[3].synchronize()
        phases["h2d_ms"].append(ev[0].elapsed_time(ev[1]))
        phases["solve_ms"].append(ev[1].elapsed_time(ev[2]))
        phases["d2h_ms"].append(ev[2].elapsed_time(ev[3]))
    import statistics
    e2e_s = statistics.median(e2e)
    if world > 1:
        t = torch.tensor([e2e_s], device="cpu" if one_dev else "cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_detail = {"samples": len(e2e), "median_s": e2e_s, "min_s": min(e2e), "max_s": max(e2e),
                  "phases_median_ms": {k: statistics.median(v) for k, v in phases.items()},
                  "numpy_median_s": statistics.median(e2e_np) if e2e_np else None,
                  "numpy_note": "reference calling convention: numpy b in, numpy x out "
                                "(pageable H2D/D2H inside P.pcg)"}

    achieved = b32 / (t32 * 1e-3) / 1e9
    # DRAM bytes of one launch from the committed ncu capture (ncu cannot run
    # inside the timed process); its provenance travels with the number
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if N == 100:  # the capture is of the 100^3 launch
                traffic, traffic_src = tj.get("fine_apply_fp32_bytes"), tj.get("source")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (fine level) / f64 (coarse, outer PCG)",
        "data": "synthetic (uniform rho=0.5 cantilever, deterministic fixture)",
        "config": _config(args),
        "pcg_iters": iters[-1], "final_true_residual": rep.final_true_residual,
        "converged": bool(rep.converged), "setup_s": setup_s, "setup_cold_s": setup[0],
        "fine_matvec_gbs": achieved,
        "roofline": {"kernel": "fine_apply_fp32 (fine_pk_kernel<0>, packed FP32x2, P32 layout)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "alg_bytes_per_launch": b32, "launch_ms": t32},
        "components": comps,
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * n_free,
                "d2h_bytes_per_step": 8 * n_free + 8 * (cfg.maxiter + 1), **e2e_detail},
        "gpu_launches": launches // max(args.steps, 1),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = oracle_iterations(N, steps=2, warmup=0)
        line["cpu_baseline"] = {"value": cb["per_iter_s"] * iters[-1], "unit": "s",
                                "cores": os.cpu_count(), "kind": "port",
                                "sample": f"{cb['iters_timed']} oracle PCG iterations at {N}^3 "
                                          f"(after a {cb['setup_s']:.1f}s oracle setup), scaled by "
                                          f"{iters[-1]} iterations"}
    if rank == 0:
        print(json.dumps(line))
    if use_slab:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--size", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slab", action="store_true", help="use the slab-partitioned path even on 1 GPU")
    ap.add_argument("--transport", default="peer", choices=["peer", "torch"],
                    help="slab transport: device kernels over CUDA IPC (peer) or torch.distributed")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
