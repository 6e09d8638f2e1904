"""General sparse triple product P^T (K P) on the device (sg_ptap_csr).

Used by ``transfer.triple_product`` for arbitrary scipy CSR inputs; the
hierarchy itself never goes through here (its levels are structured stencils,
csrc/sg_galerkin.cu).  Summation order = scipy's csr_matmat / csc_matmat, so
the result equals ``canonical_csr(P.T @ (K @ P))`` bit for bit.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _dev, _native


def _csr_arrays(A):
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    return (np.ascontiguousarray(A.indptr, dtype=np.int64),
            np.ascontiguousarray(A.indices, dtype=np.int64),
            np.ascontiguousarray(A.data, dtype=np.float64), A.shape)


def ptap(P, K):
    import scipy.sparse as sp
    Pp, Pj, Px, (nf, nc) = _csr_arrays(P)
    Kp, Kj, Kx, _ = _csr_arrays(K)
    lib = _native.load()
    res = ctypes.c_void_p()
    nnz = ctypes.c_int64()
    _native.check(lib.sg_ptap_csr(nf, nc, Pp.ctypes.data, Pj.ctypes.data, Px.ctypes.data,
                                  Kp.ctypes.data, Kj.ctypes.data, Kx.ctypes.data,
                                  ctypes.byref(res), ctypes.byref(nnz), _dev.stream()))
    try:
        Cp = np.zeros(nc + 1, dtype=np.int64)
        Cj = np.zeros(max(nnz.value, 1), dtype=np.int64)
        Cx = np.zeros(max(nnz.value, 1))
        _native.check(lib.sg_csr_result_get(res, Cp.ctypes.data, Cj.ctypes.data, Cx.ctypes.data))
    finally:
        lib.sg_csr_result_free(res)
    m = nnz.value
    C = sp.csr_matrix((Cx[:m], Cj[:m].astype(np.int32), Cp.astype(np.int32)), shape=(nc, nc))
    C.has_sorted_indices = True
    return C
