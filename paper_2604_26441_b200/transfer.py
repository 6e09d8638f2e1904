"""Trilinear transfers and Galerkin coarse operators (reference: transfer.py:1-181).

Transfers are structured device kernels (P is never stored; the CSR view
``TransferPair.P`` is exported on demand).  ``assemble_level1`` and
``triple_product`` run the bit-exact device assembly / ordered SpGEMM and
return canonical scipy CSR matrices for inspection and parity checks.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _dev, _native
from .grid import CORNER_OFFSETS, StructuredGrid, make_grid


class CoarseningUnavailableError(ValueError):
    """Raised when a grid dimension is odd and cannot be halved."""


def canonical_csr(A):
    """CSR with summed duplicates, no stored zeros, sorted column indices."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    return A


def local_prolongation_patterns() -> np.ndarray:
    """(8, 24, 24): child c of a coarse element interpolated from its 8 corners."""
    pats = np.zeros((8, 24, 24))
    for c in range(8):
        child = CORNER_OFFSETS[c]
        for a in range(8):
            t = (child + CORNER_OFFSETS[a]) / 2.0
            for b in range(8):
                w = np.prod(np.where(CORNER_OFFSETS[b] == 1, t, 1.0 - t))
                if w != 0.0:
                    for ax in range(3):
                        pats[c, 3 * a + ax, 3 * b + ax] = w
    return pats


def _mask_arg(grid: StructuredGrid):
    if grid.is_cantilever_mask:
        return None, None
    m = np.ascontiguousarray(grid.dirichlet_mask, dtype=np.uint8)
    return m, m.ctypes.data


class TransferPair:
    """Prolongation between a fine grid and its 2:1 coarsening (device kernels)."""

    _sg_native = True

    def __init__(self, fine: StructuredGrid, coarse: StructuredGrid, handle=None, hier=None,
                 level=None):
        self.fine = fine
        self.coarse = coarse
        self._th = handle
        self._hier = hier
        self._level = level
        self._P = None
        self._lib = _native.load()

    @classmethod
    def _from_hierarchy(cls, h, level):
        obj = cls.__new__(cls)
        obj._th, obj._hier, obj._level, obj._P = None, h, level, None
        obj._lib = _native.load()
        return obj

    def __getattr__(self, name):
        if name in ("fine", "coarse") and self.__dict__.get("_hier") is not None:
            lv = self._hier.levels
            return lv[self._level].grid if name == "fine" else lv[self._level + 1].grid
        raise AttributeError(name)

    def __del__(self):
        th = self.__dict__.get("_th")
        if th is not None and th.value:
            try:
                self._lib.sg_transfer_destroy(th)
            except Exception:
                pass

    def _apply(self, x, transpose):
        n_in, n_out = ((self.fine.n_free, self.coarse.n_free) if transpose
                       else (self.coarse.n_free, self.fine.n_free))
        xd, host = _dev.as_device(x, np.float64, n_in)
        y = _dev.empty(n_out)
        if self._hier is not None:
            fn = self._lib.sg_hier_restrict if transpose else self._lib.sg_hier_prolong
            _native.check(fn(self._hier._hh, self._level, _dev.ptr(xd), _dev.ptr(y), _dev.stream()))
        else:
            _native.check(self._lib.sg_transfer_apply(self._th, int(transpose), _dev.ptr(xd),
                                                      _dev.ptr(y), _dev.stream()))
        return _dev.back(y, host)

    def prolong(self, xc):
        return self._apply(xc, False)

    def restrict(self, xf):
        return self._apply(xf, True)

    @property
    def P(self):
        """(fine free) x (coarse free) canonical CSR export of the structured P."""
        if self._P is None:
            import scipy.sparse as sp
            nf = self.fine.n_free
            nnz = ctypes.c_int64()
            if self._hier is not None:
                call = lambda *a: self._lib.sg_hier_transfer_csr(self._hier._hh, self._level, *a)
            else:
                call = lambda *a: self._lib.sg_transfer_csr(self._th, *a)
            indptr = np.zeros(nf + 1, dtype=np.int64)
            _native.check(call(indptr.ctypes.data, None, None, ctypes.byref(nnz)))
            indices = np.zeros(max(nnz.value, 1), dtype=np.int64)
            data = np.zeros(max(nnz.value, 1))
            _native.check(call(indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
                               ctypes.byref(nnz)))
            m = nnz.value
            self._P = sp.csr_matrix((data[:m], indices[:m].astype(np.int32), indptr.astype(np.int32)),
                                    shape=(nf, self.coarse.n_free))
            self._P.has_sorted_indices = True
        return self._P


def build_transfer(fine: StructuredGrid) -> TransferPair:
    """Transfer pair for one 2:1 coarsening of `fine` (injection boundary mask)."""
    if fine.nx % 2 or fine.ny % 2 or fine.nz % 2:
        raise CoarseningUnavailableError(
            f"grid ({fine.nx},{fine.ny},{fine.nz}) has an odd dimension")
    lib = _native.load()
    m, mp = _mask_arg(fine)
    th = ctypes.c_void_p()
    _native.check(lib.sg_transfer_create(fine.nx, fine.ny, fine.nz, mp, ctypes.byref(th)))
    cx, cy, cz = fine.nx // 2, fine.ny // 2, fine.nz // 2
    cmask = np.zeros(3 * (cx + 1) * (cy + 1) * (cz + 1), dtype=np.uint8)
    _native.check(lib.sg_transfer_coarse_mask(th, cmask.ctypes.data))
    coarse = make_grid(cx, cy, cz, cmask.astype(bool))
    return TransferPair(fine, coarse, handle=th)


def assemble_level1(op, t: TransferPair):
    """Galerkin P^T K P of the fine operator, element-wise on the device (bit-exact CSR)."""
    import scipy.sparse as sp
    from .hierarchy import galerkin_tables
    fine, coarse = t.fine, t.coarse
    if (op.grid.nx, op.grid.ny, op.grid.nz) != (fine.nx, fine.ny, fine.nz):
        raise ValueError("transfer pair was built for a different grid")
    lib = _native.load()
    cap = 4096
    codes = np.zeros(cap, dtype=np.uint32)
    nc = ctypes.c_int()
    _native.check(lib.sg_fine_boundary_codes(op.handle, codes.ctypes.data, cap, ctypes.byref(nc)))
    codes = codes[: nc.value]
    triples, diffs = galerkin_tables(op.ke, codes)
    n = coarse.n_free
    indptr = np.zeros(n + 1, dtype=np.int64)
    nnz = ctypes.c_int64()
    args = (op.handle, triples.ctypes.data, codes.ctypes.data if codes.size else None,
            diffs.ctypes.data if codes.size else None, int(codes.size))
    _native.check(lib.sg_level1_csr(*args, indptr.ctypes.data, None, None, ctypes.byref(nnz)))
    indices = np.zeros(max(nnz.value, 1), dtype=np.int64)
    data = np.zeros(max(nnz.value, 1))
    _native.check(lib.sg_level1_csr(*args, indptr.ctypes.data, indices.ctypes.data,
                                    data.ctypes.data, ctypes.byref(nnz)))
    m = nnz.value
    K = sp.csr_matrix((data[:m], indices[:m].astype(np.int32), indptr.astype(np.int32)),
                      shape=(n, n))
    K.has_sorted_indices = True
    return K


def triple_product(P, K):
    """Exact P^T K P in canonical CSR form with scipy's summation order (device SpGEMM)."""
    from ._spgemm import ptap
    if K.shape[0] != K.shape[1] or K.shape[1] != P.shape[0]:
        raise ValueError(f"dimension mismatch: K {K.shape}, P {P.shape}")
    return ptap(P, K)
