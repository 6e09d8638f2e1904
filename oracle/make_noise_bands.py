"""Rounding-noise bands of the reference's residual histories (test infrastructure).

The reference's FP32 fine apply is OpenBLAS sgemm + ``np.add.at`` (fine_operator.py:68-77);
its FP64 dots and apply are OpenBLAS ddot / dgemm + bincount.  Any other correct
implementation rounds differently, and PCG amplifies those differences over the
iterations (at 100^3 uniform the oracle's own FP32 history moves by 1.5e-2 at entry 12
when the FP32 apply accumulates in FP64 before rounding).  A fixed 1e-4 per-entry bar
is therefore not attainable by any implementation that does not replay OpenBLAS.

This script runs the oracle port (oracle/simp_oracle.py, pinned to the reference by
tests/test_oracle_golden.py) twice per case -- as is, and with one legitimate change of
rounding order -- and records the per-entry relative distance of the two histories:

  fp32 cells  : FP32 fine apply accumulated in FP64, then rounded to FP32
                (a different but correctly rounded FP32 result per entry)
  jacobi cells: FP64 fine apply contracted with einsum instead of dgemm
                (different summation order inside the 24x24 contraction)

The GPU tests accept a history when every entry is within max(1e-4, 3 x band) of the
reference's (tests/test_baseline_configs_gpu.py), and separately require the north
star's identical verdicts, iterations within +-2 and final residual within 2x.

    OPENBLAS_NUM_THREADS=8 python oracle/make_noise_bands.py fp32 40
    OPENBLAS_NUM_THREADS=8 python oracle/make_noise_bands.py jacobi 60
    OPENBLAS_NUM_THREADS=8 python oracle/make_noise_bands.py big 100
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import simp_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")
CELLS = [(vf, p) for vf in (0.2, 0.5, 0.8) for p in (1.5, 3.0, 4.5)]
_orig = O.fine_apply


def _pert_fp32(g, E, ke, u, tag="fp64"):
    if tag != "fp32":
        return _orig(g, E, ke, u, tag)
    return _orig(g, E.astype(np.float32).astype(np.float64),
                 ke.astype(np.float32).astype(np.float64),
                 np.asarray(u, np.float32).astype(np.float64), "fp64").astype(np.float32)


def _pert_fp64(g, E, ke, u, tag="fp64"):
    if tag != "fp64":
        return _orig(g, E, ke, u, tag)
    full = np.zeros(g.n_dof)
    full[g.free] = u
    loc = np.einsum("ej,jk->ek", full[g.edofs], ke, optimize=False) * E[:, None]
    return np.bincount(g.edofs.ravel(), weights=loc.ravel(), minlength=g.n_dof)[g.free]


def _band(run, pert):
    O.fine_apply = _orig
    a = run()
    O.fine_apply = pert
    try:
        b = run()
    finally:
        O.fine_apply = _orig
    ha, hb = np.asarray(a.residual_history), np.asarray(b.residual_history)
    n = min(len(ha), len(hb))
    rel = np.abs(ha[:n] - hb[:n]) / np.abs(ha[:n])
    return {"iterations": [int(a.iterations), int(b.iterations)],
            "band": [float(v) for v in rel]}


def main(argv):
    kind, N = argv[0], int(argv[1])
    out = {}
    if kind == "fp32":
        for vf, p in CELLS:
            g, E, ke = O.problem(N, N, N, kind="binary", vf=vf, p=p)
            out[f"{vf}_{p}"] = _band(lambda: O.solve(g, E, ke, "fp32")[0], _pert_fp32)
            print(N, vf, p, out[f"{vf}_{p}"]["iterations"], max(out[f"{vf}_{p}"]["band"]),
                  flush=True)
    elif kind == "jacobi":
        for vf, p in CELLS:
            g, E, ke = O.problem(N, N, N, kind="binary", vf=vf, p=p)
            out[f"{vf}_{p}"] = _band(lambda: O.solve(g, E, ke, method="jacobi")[0], _pert_fp64)
            print(N, vf, p, max(out[f"{vf}_{p}"]["band"][:50]), flush=True)
    elif kind == "big":
        g, E, ke = O.problem(N, N, N, kind="uniform", vf=0.5, p=3.0)
        out["pcg"] = _band(lambda: O.solve(g, E, ke, "fp32")[0], _pert_fp32)
        print(N, out["pcg"]["iterations"], max(out["pcg"]["band"]), flush=True)
    else:
        raise SystemExit(__doc__)
    name = f"band_{kind}_{N}.json"
    with open(os.path.join(OUT, name), "w", encoding="utf-8") as fh:
        json.dump({"recipe": " ".join(argv), "cells": out}, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print("wrote", name)


if __name__ == "__main__":
    main(sys.argv[1:])
