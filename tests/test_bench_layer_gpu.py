"""GPU-backed benchmark layer vs the reference's own reports.

Every experiment in tests/golden/bench_reports.json (reference payloads, see
oracle/make_golden.py) is re-run through this package's runner on the B200 and
compared field by field: identical keys, gate ids/verdicts, convergence flags,
iteration counts, levels, strings; floats within per-field tolerances (FP64
Krylov / Lanczos reductions run in a different order than numpy's).  BF16EMU
cells are the exception, as in test_gpu_parity.test_outer_solver_parity: an
fp32-ulp difference upstream of a bf16 rounding flips it (2^-8 relative), and
K amplifies such high-frequency flips, so iteration counts agree to +-2 and
residuals to their scale only.
"""

import json
import os
import subprocess
import sys
from dataclasses import replace

import pytest

pytestmark = pytest.mark.gpu

from paper_2604_26441_b200.bench import numeric_payload, run_experiment, specs  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bench_reports.json")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (rtol, atol) per float field; residual-like values only need the same scale
# (Lanczos kappa from 40 steps moves ~1e-6 with 1-ulp operator changes; the
# north star's per-entry FP32 tolerance is 1e-5)
TOL = {"kappa_eff": (1e-5, 0), "eps_kappa": (1e-5, 0), "lambda_min": (1e-5, 0),
       "lambda_max": (1e-5, 0), "compliance": (1e-8, 0), "final_true_residual": (0.5, 1e-12),
       "residual_history": (0.05, 1e-12), "error_vs_direct": (0, 1e-10)}
MEASURED_ATOL = {"M1": 2e-11, "M3": 1e-10, "M6": 1e-4, "M7": 1e-5, "M8": 1e-9}


def _golden():
    with open(GOLDEN, encoding="utf-8") as fh:
        return json.load(fh)


def _close(a, b, rtol, atol):
    return abs(a - b) <= rtol * abs(b) + atol


def _compare(ours, ref, path, key=None, gate=None, bf16=False, loose_kappa=False, loose_iters=False):
    if isinstance(ref, dict):
        assert isinstance(ours, dict) and set(ours) == set(ref), f"{path}: keys {set(ours) ^ set(ref)}"
        gid = ref.get("id", gate)
        bf16 = bf16 or ref.get("precision") == "bf16" or gid == "M7"  # M7: the BF16 solve
        # the Ritz values of an odd-degree smoother's cycle are ill-conditioned
        # (a 1e-15 change of the operator moves kappa ~1e-4 here; the reference's
        # own value sits 1.6e-3 away on the 8x4x4 depth-3 cell)
        loose_kappa = loose_kappa or ref.get("degree", 2) % 2 == 1
        # flat Jacobi-PCG (no multigrid) runs ~190 rounding-sensitive iterations
        spec = ref.get("spec") if isinstance(ref.get("spec"), dict) else {}
        loose_iters = loose_iters or ref.get("method") == "jacobi" or spec.get("method") == "jacobi"
        for k in ref:
            if not ((bf16 or loose_iters) and k == "residual_history"):
                _compare(ours[k], ref[k], f"{path}.{k}", k, gid, bf16, loose_kappa, loose_iters)
    elif isinstance(ref, list):
        assert isinstance(ours, list) and len(ours) == len(ref), f"{path}: length"
        for i, (o, r) in enumerate(zip(ours, ref)):
            _compare(o, r, f"{path}[{i}]", key, gate, bf16, loose_kappa, loose_iters)
    elif isinstance(ref, (bool, str)) or ref is None:
        assert ours == ref, f"{path}: {ours!r} != {ref!r}"
    elif (bf16 or loose_iters) and key in ("iterations", "final_true_residual", "iterations_mean",
                                           "compliance"):
        ok = abs(ours - ref) <= 2 if key.startswith("iterations") else _close(ours, ref, 0.95, 0)
        assert ok, f"{path}: {ours!r} vs {ref!r} (+-2 band)"
    elif loose_kappa and key in ("kappa_eff", "eps_kappa", "lambda_min", "lambda_max"):
        assert _close(float(ours), float(ref), 5e-3, 0), f"{path}: {ours!r} vs {ref!r}"
    elif key in ("iterations", "levels", "cells", "failures", "passes", "converged_trials",
                 "threshold", "gates_total", "gates_passed") or (key == "measured" and isinstance(ref, int)
                                                                 and gate and not gate.startswith("M6")):
        assert ours == ref, f"{path}: {ours!r} != {ref!r}"
    else:
        if key == "measured":
            rtol, atol = 1e-6, MEASURED_ATOL.get(gate.split("-")[0], 0)
        else:
            rtol, atol = TOL.get(key, (1e-12, 0))
        assert _close(float(ours), float(ref), rtol, atol), f"{path}: {ours!r} vs {ref!r}"


def _spec(over):
    conv = {k: (tuple(tuple(x) if isinstance(x, list) else x for x in v)
                if isinstance(v, list) else v) for k, v in over.items()}
    return replace(specs.ExperimentSpec(), **conv)


@pytest.mark.parametrize("name", sorted(_golden()))
def test_report_matches_reference(name):
    g = _golden()[name]
    rep = run_experiment(_spec(g["overrides"]))
    ours = json.loads(numeric_payload(rep))
    _compare(ours, json.loads(g["payload"]), name)
    assert all(x["passed"] for x in rep["gates"])
    assert rep["environment"]["device"].startswith("NVIDIA")


def test_sweep_payload_is_deterministic():
    spec = _spec({"experiment": "sweep", "grids": [[8, 4, 4]], "precisions": ["fp32", "bf16"]})
    assert numeric_payload(run_experiment(spec)) == numeric_payload(run_experiment(spec))


def test_cli_end_to_end(tmp_path):
    out = tmp_path / "r.json"
    proc = subprocess.run([sys.executable, "-m", "paper_2604_26441_b200", "solve", "--grid", "8,4,4",
                           "--trials", "2", "--warmups", "1", "--precision", "bf16", "--out", str(out)],
                          cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr
    rep = json.loads(out.read_text())
    assert rep["aggregates"]["method"] == "fgmres" and rep["aggregates"]["converged_trials"] == 2
    assert "[PASS] solve-converged" in proc.stdout
