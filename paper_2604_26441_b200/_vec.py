"""Deterministic device vector arithmetic via the C ABI (sg_vec_*).

Used by the generic solver / smoother paths that accept arbitrary Python
callables: the callables may live anywhere, but the Krylov / smoother
arithmetic itself always runs in libsg_b200.so kernels on the GPU.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _dev, _native


def _dt(t):
    return 0 if t.dtype == torch.float64 else 1


def dot(a, b) -> float:
    out = ctypes.c_double()
    _native.check(_native.load().sg_vec_dot(_dt(a), a.numel(), _dev.ptr(a), _dev.ptr(b),
                                            ctypes.byref(out), _dev.stream()))
    return float(out.value)


def axpy(alpha, x, y):
    """y <- y + alpha*x (in place)."""
    _native.check(_native.load().sg_vec_axpy(_dt(y), y.numel(), float(alpha), _dev.ptr(x),
                                             _dev.ptr(y), _dev.stream()))
    return y


def xpby(x, beta, y):
    """y <- x + beta*y (in place)."""
    _native.check(_native.load().sg_vec_xpby(_dt(y), y.numel(), _dev.ptr(x), float(beta),
                                             _dev.ptr(y), _dev.stream()))
    return y


def sub(a, b, out=None):
    out = torch.empty_like(a) if out is None else out
    _native.check(_native.load().sg_vec_sub(_dt(a), a.numel(), _dev.ptr(a), _dev.ptr(b),
                                            _dev.ptr(out), _dev.stream()))
    return out


def mul(a, b, out=None):
    out = torch.empty_like(a) if out is None else out
    _native.check(_native.load().sg_vec_mul(_dt(a), a.numel(), _dev.ptr(a), _dev.ptr(b),
                                            _dev.ptr(out), _dev.stream()))
    return out


def scale(a, s, out=None):
    out = torch.empty_like(a) if out is None else out
    _native.check(_native.load().sg_vec_scale(_dt(a), a.numel(), _dev.ptr(a), float(s),
                                              _dev.ptr(out), _dev.stream()))
    return out


def div(a, s, out=None):
    out = torch.empty_like(a) if out is None else out
    _native.check(_native.load().sg_vec_div(_dt(a), a.numel(), _dev.ptr(a), float(s),
                                            _dev.ptr(out), _dev.stream()))
    return out


def norm(a) -> float:
    return math.sqrt(dot(a, a))
