"""Outer Krylov solvers: PCG and restarted flexible GMRES (reference: krylov.py:1-288).

Dispatch: when ``apply_K`` is ``FineOperator.matvec`` of this package and
``apply_M`` is ``GmgHierarchy.vcycle`` / ``wcycle`` (or the flat Jacobi
preconditioner), the whole solve runs in the native C++ driver
(``sg_pcg`` / ``sg_fgmres``): device-resident vectors, deterministic
device reductions, one small scalar read per iteration.  Arbitrary Python
callables are still accepted (the reference's tests pass lambdas); then the
Krylov arithmetic runs on the device through the sg_vec kernels and foreign
callables receive numpy arrays.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _native, _vec
from .precision import PrecisionTag

HAPPY_BREAKDOWN = 1e-14
STAGNATION_WINDOW = 50
STAGNATION_IMPROVEMENT = 0.01
_KINDS = {0: "none", 1: "cap", 2: "stagnation", 3: "non_finite"}


@dataclass(frozen=True)
class SolverConfig:
    method: str = "pcg"
    tol: float = 1e-6
    maxiter: int = 200
    restart: int = 32
    record_history: bool = True

    def __post_init__(self):
        if self.method not in ("pcg", "fgmres"):
            raise ValueError(f"unknown method {self.method!r}")
        if self.tol <= 0 or self.maxiter < 1 or self.restart < 1:
            raise ValueError("tol must be positive and iteration counts >= 1")


@dataclass
class SolveReport:
    converged: bool
    iterations: int
    final_true_residual: float
    failure_kind: str
    residual_history: list = field(default_factory=list)
    wall_time: float = 0.0
    x: object = field(default=None, repr=False)

    def to_dict(self, include_history: bool = True) -> dict:
        d = {"converged": self.converged, "iterations": self.iterations,
             "final_true_residual": self.final_true_residual,
             "failure_kind": self.failure_kind, "wall_time": self.wall_time}
        if include_history:
            d["residual_history"] = list(self.residual_history)
        return d


# ------------------------------------------------------------ dispatch
class _JacobiM:
    """Marker for flat_jacobi_pcg's 1/diag preconditioner."""

    def __init__(self, op):
        self.op = op

    def __call__(self, r):
        rd, host = _dev.as_device(r, np.float64, self.op.n_free)
        dinv = 1.0 / self.op.diagonal_device()
        return _dev.back(_vec.mul(dinv, rd), host)


def _native_pair(apply_K, apply_M):
    """(op, ktag, hier, gamma) when both callables are native, else None."""
    from .fine_operator import FineOperator
    from .hierarchy import GmgHierarchy
    op = getattr(apply_K, "__self__", None)
    if not isinstance(op, FineOperator) or getattr(apply_K, "__func__", None) is not FineOperator.matvec:
        return None
    ktag = op.precision.code
    if isinstance(apply_M, _JacobiM) and apply_M.op is op:
        return op, ktag, None, 1
    h = getattr(apply_M, "__self__", None)
    if isinstance(h, GmgHierarchy) and h._op is op:
        fn = getattr(apply_M, "__func__", None)
        if fn is GmgHierarchy.vcycle:
            return op, ktag, h, 1
        if fn is GmgHierarchy.wcycle:
            return op, ktag, h, 2
    return None


def _run_native(which, nat, b, cfg: SolverConfig):
    op, ktag, h, gamma = nat
    bd, host = _dev.as_device(b, np.float64, op.n_free)
    x = _dev.empty(op.n_free)
    hist = np.zeros(cfg.maxiter + 1)
    c = _native.SolverCfg(cfg.tol, cfg.maxiter, cfg.restart)
    rep = _native.Report()
    fn = _native.load().sg_pcg if which == "pcg" else _native.load().sg_fgmres
    _native.check(fn(op.handle, ktag, h._hh if h is not None else None, gamma, _dev.ptr(bd),
                     _dev.ptr(x), ctypes.byref(c), ctypes.byref(rep), hist.ctypes.data,
                     _dev.stream()))
    it = int(rep.iterations)
    return SolveReport(bool(rep.converged), it, float(rep.final_true_residual),
                       _KINDS[int(rep.failure_kind)],
                       [float(v) for v in hist[:it]] if cfg.record_history else [],
                       float(rep.wall_time), _dev.back(x, host))


# --------------------------------------------------------- generic path
def _apply(fn, x):
    from .smoothers import is_native
    y = fn(x) if is_native(fn) or isinstance(fn, _JacobiM) else fn(x.cpu().numpy())
    t, _ = _dev.as_device(y, np.float64, x.numel())
    return t


class _Monitor:
    def __init__(self, cfg, normb):
        self.cfg, self.normb = cfg, normb
        self.history, self.best = [], []

    def record(self, rel):
        self.history.append(rel)
        prev = self.best[-1] if self.best else math.inf
        self.best.append(min(prev, rel))
        return None if math.isfinite(rel) else "non_finite"

    def stagnant(self):
        k = len(self.best)
        if k <= STAGNATION_WINDOW:
            return False
        return not (self.best[-1] <= (1.0 - STAGNATION_IMPROVEMENT) * self.best[k - 1 - STAGNATION_WINDOW])

    def finish(self, apply_K, b, x, kind, t0, host):
        tr = _vec.norm(_vec.sub(b, _apply(apply_K, x))) / self.normb
        conv = bool(math.isfinite(tr) and tr < self.cfg.tol)
        return SolveReport(conv, len(self.history), tr, "none" if conv else kind,
                           self.history if self.cfg.record_history else [],
                           time.perf_counter() - t0, _dev.back(x, host))


def _zero_report(b, host, t0):
    return SolveReport(True, 0, 0.0, "none", [], time.perf_counter() - t0,
                       _dev.back(torch.zeros_like(b), host))


def _generic_pcg(apply_K, apply_M, b, cfg):
    t0 = time.perf_counter()
    bd, host = _dev.as_device(b, np.float64)
    normb = _vec.norm(bd)
    if normb == 0.0:
        return _zero_report(bd, host, t0)
    mon = _Monitor(cfg, normb)
    x = torch.zeros_like(bd)
    r = bd.clone()
    p = _apply(apply_M, r).clone()
    rz = _vec.dot(r, p)
    target, kind = cfg.tol, "cap"
    for _ in range(cfg.maxiter):
        q = _apply(apply_K, p)
        pq = _vec.dot(p, q)
        if not math.isfinite(pq) or pq == 0.0:
            kind = "non_finite"
            break
        a = rz / pq
        _vec.axpy(a, p, x)
        _sub_scaled(r, a, q)
        rel = _vec.norm(r) / normb
        fail = mon.record(rel)
        if fail:
            kind = fail
            break
        if rel < target:
            if _vec.norm(_vec.sub(bd, _apply(apply_K, x))) / normb < cfg.tol:
                kind = "none"
                break
            if mon.stagnant():
                kind = "stagnation"
                break
            target *= 0.1
        z = _apply(apply_M, r)
        rzn = _vec.dot(r, z)
        if not math.isfinite(rzn):
            kind = "non_finite"
            break
        p = _vec.xpby(z, rzn / rz, p)
        rz = rzn
    return mon.finish(apply_K, bd, x, kind, t0, host)


def _sub_scaled(r, a, q):
    """r <- r - a*q with the product rounded first (numpy: r - a * q)."""
    t = _vec.scale(q, a)
    _vec.sub(r, t, out=r)


def _solve_upper(R, g):
    import scipy.linalg as sla
    with np.errstate(divide="ignore", invalid="ignore"):
        try:
            y = sla.solve_triangular(R, g, lower=False, check_finite=False)
        except Exception:
            y = None
    if y is None or not np.isfinite(y).all():
        y = np.linalg.lstsq(R, g.copy(), rcond=None)[0]
    return y


def _generic_fgmres(apply_K, apply_M, b, cfg):
    t0 = time.perf_counter()
    bd, host = _dev.as_device(b, np.float64)
    normb = _vec.norm(bd)
    if normb == 0.0:
        return _zero_report(bd, host, t0)
    mon = _Monitor(cfg, normb)
    n, m = bd.numel(), cfg.restart
    x = torch.zeros_like(bd)
    kind, done = "cap", False
    while not done and len(mon.history) < cfg.maxiter:
        r = _vec.sub(bd, _apply(apply_K, x))
        beta = _vec.norm(r)
        if not math.isfinite(beta):
            kind = "non_finite"
            break
        if beta / normb < cfg.tol:
            kind = "none"
            break
        V = torch.zeros((m + 1, n), dtype=torch.float64, device=bd.device)
        Z = torch.zeros((m, n), dtype=torch.float64, device=bd.device)
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        _vec.div(r, beta, out=V[0])
        used, claimed = 0, False
        for j in range(m):
            Z[j].copy_(_apply(apply_M, V[j]))
            w = _apply(apply_K, Z[j]).clone()
            for i in range(j + 1):
                H[i, j] = _vec.dot(w, V[i])
                _sub_scaled(w, H[i, j], V[i])
            H[j + 1, j] = _vec.norm(w)
            if not np.isfinite(H[: j + 2, j]).all():
                kind, done, used = "non_finite", True, j + 1
                break
            happy = H[j + 1, j] < HAPPY_BREAKDOWN
            if not happy:
                _vec.div(w, H[j + 1, j], out=V[j + 1])
            for i in range(j):
                h0 = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = h0
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            used = j + 1
            rel = abs(g[j + 1]) / normb
            fail = mon.record(float(rel))
            if fail:
                kind, done = fail, True
                break
            if happy or rel < cfg.tol:
                claimed = True
                break
            if len(mon.history) >= cfg.maxiter:
                break
        if kind == "non_finite":
            break
        if used > 0:
            y = _solve_upper(H[:used, :used], g[:used])
            for j in range(used):
                _vec.axpy(float(y[j]), Z[j], x)
        if done:
            break
        if _vec.norm(_vec.sub(bd, _apply(apply_K, x))) / normb < cfg.tol:
            kind = "none"
            break
        if claimed and mon.stagnant():
            kind = "stagnation"
            break
        if len(mon.history) >= cfg.maxiter:
            kind = "cap"
            break
    return mon.finish(apply_K, bd, x, kind, t0, host)


def pcg(apply_K, apply_M, b, cfg: SolverConfig) -> SolveReport:
    """Left-preconditioned CG with FP64 true-residual acceptance (krylov.py:113-165)."""
    nat = _native_pair(apply_K, apply_M)
    if nat is not None:
        return _run_native("pcg", nat, b, cfg)
    return _generic_pcg(apply_K, apply_M, b, cfg)


def fgmres(apply_K, apply_M, b, cfg: SolverConfig) -> SolveReport:
    """Restarted right-preconditioned flexible GMRES (krylov.py:168-269)."""
    nat = _native_pair(apply_K, apply_M)
    if nat is not None:
        return _run_native("fgmres", nat, b, cfg)
    return _generic_fgmres(apply_K, apply_M, b, cfg)


def flat_jacobi_pcg(op, b, cfg: SolverConfig) -> SolveReport:
    """Baseline comparator: PCG preconditioned by the inverse fine diagonal."""
    return _run_native("pcg", (op, PrecisionTag.FP64.code, None, 1), b, cfg)
