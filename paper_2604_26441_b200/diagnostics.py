"""Spectral probes of the preconditioned operator (reference: diagnostics.py:1-92).

``lanczos_kappa_eff`` with the probe operator v -> h.vcycle(op.matvec(v))
of this package runs natively (``sg_lanczos``: device Krylov basis, two-pass
reorthogonalisation on the GPU); only the m x m projected matrix comes back
to the host for its eigenvalues.  Generic callables use the device vector
kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _native, _vec
from .precision import EPS_BF16
from .prng import gaussian_unit_vector

LANCZOS_STEPS = 40
_BREAKDOWN = 1e-14


@dataclass(frozen=True)
class SpectralProbe:
    m: int
    seed: int
    kappa_eff: float
    eps_kappa: float
    lambda_min: float
    lambda_max: float
    partial: bool


class PreconditionedOperator:
    """v -> M (K v) with native K = FineOperator (FP64) and M = a hierarchy cycle."""

    _sg_native = True

    def __init__(self, op, hierarchy, gamma: int = 1):
        self.op, self.h, self.gamma = op, hierarchy, gamma

    def __call__(self, v):
        from .precision import PrecisionTag
        kv = self.op.matvec_tagged(v, PrecisionTag.FP64)
        return self.h.vcycle(kv) if self.gamma == 1 else self.h.wcycle(kv)


def _ritz(H, used, m, seed, partial):
    ritz = np.sort(np.linalg.eigvals(H[:used, :used]).real)
    lo, hi = float(ritz[0]), float(ritz[-1])
    kappa = hi / lo if lo != 0.0 else np.inf
    return SpectralProbe(m, seed, float(kappa), float(EPS_BF16 * kappa), lo, hi, partial)


def lanczos_kappa_eff(apply_MK, n: int, m: int = LANCZOS_STEPS, seed: int = 0) -> SpectralProbe:
    """m-step Lanczos with full (two-pass) reorthogonalisation (diagnostics.py:38-79)."""
    if m < 2:
        raise ValueError("need at least two Lanczos steps")
    if isinstance(apply_MK, PreconditionedOperator):
        H = np.zeros((m, m))
        used, partial = ctypes.c_int(), ctypes.c_int()
        _native.check(_native.load().sg_lanczos(apply_MK.op.handle, apply_MK.h._hh, apply_MK.gamma,
                                                m, seed, H.ctypes.data, ctypes.byref(used),
                                                ctypes.byref(partial), _dev.stream()))
        return _ritz(H, used.value, m, seed, bool(partial.value))
    from .smoothers import is_native
    dev = _dev.device()
    Q = torch.zeros((m, n), dtype=torch.float64, device=dev)
    Q[0].copy_(_dev.as_device(gaussian_unit_vector(n, seed))[0])
    H = np.zeros((m, m))
    used, partial = m, False
    for j in range(m):
        y = apply_MK(Q[j]) if is_native(apply_MK) else apply_MK(Q[j].cpu().numpy())
        w, _ = _dev.as_device(y, np.float64, n)
        w = w.clone()
        for _pass in range(2):
            h = np.array([_vec.dot(Q[t], w) for t in range(j + 1)])
            H[: j + 1, j] += h
            t = torch.zeros_like(w)
            for q in range(j + 1):
                _vec.axpy(float(h[q]), Q[q], t)
            _vec.sub(w, t, out=w)
        if j == m - 1:
            break
        s = _vec.norm(w)
        if not np.isfinite(s) or s < _BREAKDOWN:
            used, partial = j + 1, True
            break
        H[j + 1, j] = s
        _vec.div(w, s, out=Q[j + 1])
    return _ritz(H, used, m, seed, partial)


def bf16_screen(probe: SpectralProbe) -> bool:
    """True iff eps_BF16 * kappa_eff < 1 (diagnostic only)."""
    return bool(probe.eps_kappa < 1.0)


def kappa_bound(rho: float) -> float:
    """(1 + rho) / (1 - rho) for a cycle contraction rho < 1."""
    if not (0.0 <= rho < 1.0):
        raise ValueError(f"spectral radius must lie in [0, 1), got {rho}")
    return (1.0 + rho) / (1.0 - rho)
