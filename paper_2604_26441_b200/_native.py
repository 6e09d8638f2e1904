"""ctypes binding of include/sg_api.h (the C-ABI of libsg_b200.so).

There is no fallback: if the library cannot be loaded, or no CUDA device is
present, every compute entry point raises.  The library is built in-tree by
``paper_2604_26441_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libsg_b200.so")

c_int, c_i64, c_u64, c_double, c_void_p = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER


class HierParams(C.Structure):
    _fields_ = [("levels", c_int), ("policy", c_int), ("smoother_kind", c_int),
                ("degree", c_int), ("alpha", c_double), ("omega", c_double),
                ("coarse_smooth_steps", c_int), ("cholesky_cutoff", c_int),
                ("coarse_pcg_steps", c_int), ("power_seed", c_u64)]


class HierInfo(C.Structure):
    _fields_ = [("n_levels", c_int), ("clamped", c_int), ("coarsest_dense", c_int),
                ("eps", c_double)]


class LevelInfo(C.Structure):
    _fields_ = [("nx", c_int), ("ny", c_int), ("nz", c_int), ("tag", c_int),
                ("n_free", c_i64), ("nnz", c_i64), ("lam_max", c_double)]


class SolverCfg(C.Structure):
    _fields_ = [("tol", c_double), ("maxiter", c_int), ("restart", c_int)]


class Report(C.Structure):
    _fields_ = [("converged", c_int), ("iterations", c_int),
                ("final_true_residual", c_double), ("failure_kind", c_int),
                ("wall_time", c_double)]


HALO_FN = C.CFUNCTYPE(c_int, c_void_p, c_int, c_void_p, c_int, c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(c_int, c_void_p, c_void_p, c_int, c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p)


class Comm(C.Structure):
    """sg_comm: host callbacks of the slab partition (include/sg_api.h)."""
    _fields_ = [("ctx", c_void_p), ("halo", HALO_FN), ("allreduce", ALLREDUCE_FN),
                ("allgather", ALLGATHER_FN)]


# name: (restype, argtypes) -- mirrors include/sg_api.h
SIGNATURES = {
    "sg_last_error": (C.c_char_p, []),
    "sg_version": (c_int, []),
    "sg_fine_create": (c_int, [c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, P(c_void_p)]),
    "sg_fine_destroy": (None, [c_void_p]),
    "sg_fine_n_free": (c_i64, [c_void_p]),
    "sg_fine_apply": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_fine_apply_nodes": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_fine_n_nodes": (c_i64, [c_void_p]),
    "sg_launch_count": (c_u64, []),
    "sg_fine_diagonal": (c_int, [c_void_p, c_void_p, c_void_p]),
    "sg_fine_dense": (c_int, [c_void_p, c_void_p, c_void_p]),
    "sg_fine_boundary_codes": (c_int, [c_void_p, c_void_p, c_int, P(c_int)]),
    "sg_hier_create": (c_int, [c_void_p, P(HierParams), c_void_p, c_void_p, c_void_p, c_int,
                               c_void_p, c_int, c_void_p, P(c_void_p)]),
    "sg_hier_destroy": (None, [c_void_p]),
    "sg_hier_get_info": (c_int, [c_void_p, P(HierInfo)]),
    "sg_hier_level_info": (c_int, [c_void_p, c_int, P(LevelInfo)]),
    "sg_hier_level_csr": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_hier_level_mask": (c_int, [c_void_p, c_int, c_void_p]),
    "sg_hier_level_diag": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "sg_hier_cycle": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_hier_level_apply": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_hier_level_smooth": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_hier_prolong": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_hier_restrict": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_hier_coarsest_solve": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_hier_profile": (c_int, [c_void_p, c_int, c_int, P(c_double), c_void_p]),
    "sg_hier_transfer_csr": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, P(c_i64)]),
    "sg_transfer_create": (c_int, [c_int, c_int, c_int, c_void_p, P(c_void_p)]),
    "sg_transfer_destroy": (None, [c_void_p]),
    "sg_transfer_coarse_mask": (c_int, [c_void_p, c_void_p]),
    "sg_transfer_apply": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_transfer_csr": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, P(c_i64)]),
    "sg_level1_csr": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                              c_void_p, P(c_i64)]),
    "sg_ptap_csr": (c_int, [c_i64, c_i64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                            c_void_p, P(c_void_p), P(c_i64), c_void_p]),
    "sg_csr_result_get": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_csr_result_free": (None, [c_void_p]),
    "sg_hier_pcg80_trace": (c_int, [c_void_p, c_void_p, c_void_p]),
    "sg_plan_brick": (c_int, [c_int, c_int, c_int, c_int, c_void_p]),
    "sg_plan_p32": (c_int, [c_int, c_int, c_int, c_int, c_void_p]),
    "sg_plan_p32_bs": (c_int, [c_int, c_int, c_int, c_int, c_int, c_void_p]),
    "sg_pcg": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p, P(SolverCfg),
                       P(Report), c_void_p, c_void_p]),
    "sg_fgmres": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p, P(SolverCfg),
                          P(Report), c_void_p, c_void_p]),
    "sg_lanczos": (c_int, [c_void_p, c_void_p, c_int, c_int, c_u64, c_void_p, P(c_int),
                           P(c_int), c_void_p]),
    "sg_dist_create": (c_int, [c_void_p, c_int, c_void_p, P(Comm), c_void_p, P(c_void_p)]),
    "sg_dist_destroy": (None, [c_void_p]),
    "sg_dist_create_peer": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_void_p,
                                    P(c_void_p)]),
    "sg_dist_peer_handle": (c_int, [c_void_p, c_void_p, P(c_u64)]),
    "sg_dist_peer_open": (c_int, [c_void_p, c_void_p, c_void_p]),
    "sg_dist_release_full": (c_int, [c_void_p, c_void_p]),
    "sg_plan_halo": (c_int, [c_int, c_void_p, c_void_p, c_int]),
    "sg_dist_solve": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, P(SolverCfg),
                              P(Report), c_void_p, c_void_p]),
    "sg_dist_apply": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "sg_vec_dot": (c_int, [c_int, c_i64, c_void_p, c_void_p, P(c_double), c_void_p]),
    "sg_vec_axpy": (c_int, [c_int, c_i64, c_double, c_void_p, c_void_p, c_void_p]),
    "sg_vec_xpby": (c_int, [c_int, c_i64, c_void_p, c_double, c_void_p, c_void_p]),
    "sg_vec_sub": (c_int, [c_int, c_i64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_vec_mul": (c_int, [c_int, c_i64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_vec_scale": (c_int, [c_int, c_i64, c_void_p, c_double, c_void_p, c_void_p]),
    "sg_vec_div": (c_int, [c_int, c_i64, c_void_p, c_double, c_void_p, c_void_p]),
    "sg_vec_bf16": (c_int, [c_i64, c_void_p, c_void_p, c_void_p]),
    "sg_make_state": (c_int, [c_int, c_int, c_int, c_int, c_double, c_double, c_u64, c_void_p,
                              c_void_p]),
}

_lib = None


class NativeError(RuntimeError):
    """Raised when the sm_100a library is missing or a call fails."""


def load():
    """Load libsg_b200.so (no fallback: raises NativeError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                          "(python -m paper_2604_26441_b200.build)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != 0:
        msg = load().sg_last_error()
        raise NativeError(msg.decode() if msg else "sg call failed")


def call(name, *args):
    """Invoke an sg_* function and raise on a nonzero status."""
    st = getattr(load(), name)(*args)
    check(st)
    return st
