"""Matrix-free fine-level operator on the B200 (reference: fine_operator.py:31-105).

Same interface as the reference ``FineOperator``; every apply runs the
sm_100a kernels of libsg_b200.so through the C ABI (``sg_fine_apply``).
Vectors may be numpy arrays (copied to and from the device, numpy returned)
or CUDA tensors (used in place, CUDA tensors returned).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _dev, _native
from .element import unit_element_stiffness
from .grid import StructuredGrid
from .precision import PrecisionTag
from .states import ModulusField

DIAGONAL_FLOOR = 1e-14
DENSE_GUARD = 20_000


class FineOperator:
    """K_ff action for one frozen modulus field on one structured grid."""

    _sg_native = True

    def __init__(self, grid: StructuredGrid, modulus: ModulusField, nu: float = 0.3,
                 precision: PrecisionTag = PrecisionTag.FP64):
        if modulus.E.shape != (grid.n_elem,):
            raise ValueError(f"modulus field must have {grid.n_elem} entries")
        self.grid = grid
        self.modulus = modulus
        self.precision = precision
        self.nu = nu
        self.ke = unit_element_stiffness(nu).ke
        lib = _native.load()
        E = np.ascontiguousarray(modulus.E, dtype=np.float64)
        ke = np.ascontiguousarray(self.ke, dtype=np.float64)
        mask = None
        if not grid.is_cantilever_mask:
            mask = np.ascontiguousarray(grid.dirichlet_mask, dtype=np.uint8)
        h = ctypes.c_void_p()
        _native.check(lib.sg_fine_create(grid.nx, grid.ny, grid.nz,
                                         mask.ctypes.data if mask is not None else None,
                                         E.ctypes.data, ke.ctypes.data, ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self._diag = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.sg_fine_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_free(self) -> int:
        return self.grid.n_free

    def matvec(self, u_free):
        return self.matvec_tagged(u_free, self.precision)

    def matvec_tagged(self, u_free, tag: PrecisionTag):
        """K_ff @ u_free under a precision tag (float64 out for FP64, float32 otherwise)."""
        if tuple(np.shape(u_free)) != (self.grid.n_free,):
            raise ValueError(f"expected free vector of length {self.grid.n_free}")
        wt = tag.working_dtype
        u, host = _dev.as_device(u_free, wt, self.grid.n_free)
        y = _dev.empty(self.grid.n_free, wt)
        _native.check(self._lib.sg_fine_apply(self._h, tag.code, _dev.ptr(u), _dev.ptr(y),
                                              _dev.stream()))
        return _dev.back(y, host)

    def diagonal_device(self):
        if self._diag is None:
            d = _dev.empty(self.grid.n_free)
            _native.check(self._lib.sg_fine_diagonal(self._h, _dev.ptr(d), _dev.stream()))
            self._diag = d
        return self._diag

    def diagonal(self) -> np.ndarray:
        """diag(K_ff), floored at 1e-14 times its mean (numpy-exact mean)."""
        return self.diagonal_device().cpu().numpy()

    def assemble_dense(self) -> np.ndarray:
        """Explicit K_ff (device assembly, ascending-element sums); oracle-sized grids only."""
        n = self.grid.n_free
        if n > DENSE_GUARD:
            raise ValueError(f"dense assembly limited to {DENSE_GUARD} free DOFs, grid has {n}")
        K = _dev.empty(n * n)
        _native.check(self._lib.sg_fine_dense(self._h, _dev.ptr(K), _dev.stream()))
        return K.cpu().numpy().reshape(n, n)

    def compliance(self, u_free) -> float:
        """f^T u of a solved state (device dot)."""
        f, _ = _dev.as_device(self.grid.load[self.grid.free_dofs])
        u, _ = _dev.as_device(u_free, np.float64, self.grid.n_free)
        out = ctypes.c_double()
        _native.check(self._lib.sg_vec_dot(0, self.grid.n_free, _dev.ptr(f), _dev.ptr(u),
                                           ctypes.byref(out), _dev.stream()))
        return float(out.value)
