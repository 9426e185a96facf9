"""ctypes binding of libarrabit.so (include/arrabit.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels.  There is no CPU
fallback — if the shared library is missing or fails to load, import fails."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ARRABIT_LIB", os.path.join(HERE, "libarrabit.so"))  # override: tuning variants

ARR_OK, ARR_EINVAL, ARR_ENOMEM, ARR_ECUDA, ARR_ECUSOLVER, ARR_ENCCL, ARR_ENUMERIC = 0, 1, 2, 3, 5, 6, 7
STATUS_NAMES = {0: "ARR_OK", 1: "ARR_EINVAL", 2: "ARR_ENOMEM", 3: "ARR_ECUDA", 5: "ARR_ECUSOLVER", 6: "ARR_ENCCL",
                7: "ARR_ENUMERIC"}

# Every symbol include/arrabit.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "eig_init", "eig_init_w", "eig_destroy", "eig_last_error", "eig_workspace_bytes", "eig_launch_count",
    "eig_gershgorin_lower", "eig_set_interval", "eig_set_degree", "eig_set_filter", "eig_set_mode", "filter_step", "spmm", "gram", "gemm",
    "orthonormalize", "arr_project", "arr_project_p", "residuals", "eig_solve", "eig_solve_host",
    "eig_set_timing", "eig_phase_times", "eig_kernel_times", "eig_set_schedule", "eig_set_stencil", "eig_stencil_active", "eig_stencil_abytes", "eig_last_spmm_kernel",
    "eig_init_dist", "eig_init_colsplit", "comm_get_nccl_id", "comm_init_nccl", "comm_init_local_group", "comm_rank_size", "comm_destroy",
]


class arr_csr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class arr_dist(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("n_ghost", ctypes.c_int64),
                ("npeers", ctypes.c_int32), ("peer", ctypes.c_void_p), ("send_off", ctypes.c_void_p),
                ("send_rows", ctypes.c_void_p), ("recv_off", ctypes.c_void_p),
                ("int_row0", ctypes.c_void_p), ("int_len", ctypes.c_void_p), ("n_int_tiles", ctypes.c_int64),
                ("bnd_row0", ctypes.c_void_p), ("bnd_len", ctypes.c_void_p), ("n_bnd_tiles", ctypes.c_int64)]


class arr_solve_opts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("maxit", ctypes.c_int32), ("s_max", ctypes.c_int32),
                ("exits", ctypes.c_int32), ("inner", ctypes.c_int32), ("adapt", ctypes.c_int32),
                ("gn", ctypes.c_int32), ("grid", ctypes.c_int64 * 3), ("log", ctypes.c_void_p),
                ("log_cap", ctypes.c_int32), ("range_digits", ctypes.c_double)]


class arr_solve_info(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int32), ("outer", ctypes.c_int32), ("sweeps", ctypes.c_int32),
                ("last_rank", ctypes.c_int32), ("maxres", ctypes.c_double), ("a", ctypes.c_double),
                ("b", ctypes.c_double), ("spmm_blocks", ctypes.c_int64), ("exit_rule", ctypes.c_int32),
                ("p_final", ctypes.c_int32), ("d_final", ctypes.c_int32), ("locked", ctypes.c_int32)]


_lib = None


def load(path: str | None = None):
    """Load libarrabit.so (raises OSError if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    # ARRABIT_LIB: an alternative build of the same library (e.g. the bounds-checked
    # libarrabit_checked.so, build.py --checked); never a CPU path
    path = path or os.environ.get("ARRABIT_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise OSError(f"libarrabit.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    pvp = ctypes.POINTER(ctypes.c_void_p)
    pf64 = ctypes.POINTER(ctypes.c_double)
    pi32 = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "eig_init": ([pvp, ctypes.POINTER(arr_csr), i32, i32, i32, vp], ctypes.c_int),
        "eig_init_w": ([pvp, ctypes.POINTER(arr_csr), i32, i32, i32, i32, vp], ctypes.c_int),
        "eig_init_dist": ([pvp, ctypes.POINTER(arr_csr), i32, i32, i32, i32, ctypes.POINTER(arr_dist), vp, vp],
                          ctypes.c_int),
        "eig_init_colsplit": ([pvp, ctypes.POINTER(arr_csr), i32, i32, i32, i32, ctypes.POINTER(arr_csr),
                               ctypes.POINTER(arr_dist), vp, vp, vp, vp], ctypes.c_int),
        "comm_get_nccl_id": ([ctypes.c_char_p], ctypes.c_int),
        "comm_init_nccl": ([pvp, ctypes.c_char_p, i32, i32], ctypes.c_int),
        "comm_init_local_group": ([pvp, i32], ctypes.c_int),
        "comm_rank_size": ([vp, pi32, pi32], ctypes.c_int),
        "comm_destroy": ([vp], ctypes.c_int),
        "eig_destroy": ([vp], ctypes.c_int),
        "eig_last_error": ([vp], ctypes.c_char_p),
        "eig_workspace_bytes": ([vp], ctypes.c_size_t),
        "eig_launch_count": ([vp], ctypes.c_uint64),
        "eig_gershgorin_lower": ([vp, pf64], ctypes.c_int),
        "eig_set_interval": ([vp, f64, f64], ctypes.c_int),
        "eig_set_degree": ([vp, i32], ctypes.c_int),
        "eig_set_stencil": ([vp, i64, i64, i64], ctypes.c_int),
        "eig_stencil_active": ([vp], ctypes.c_int32),
        "eig_stencil_abytes": ([vp], ctypes.c_int32),
        "eig_last_spmm_kernel": ([vp], ctypes.c_char_p),
        "eig_set_filter": ([vp, i32], ctypes.c_int),
        "eig_set_mode": ([vp, i32], ctypes.c_int),
        "eig_set_timing": ([vp, i32], ctypes.c_int),
        "eig_set_schedule": ([vp, vp, vp, i64], ctypes.c_int),
        "eig_phase_times": ([vp, pf64, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "eig_kernel_times": ([vp, pf64, pf64, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "filter_step": ([vp, vp, i64, i32, vp], ctypes.c_int),
        "spmm": ([vp, f64, f64, vp, i64, vp, i64, i32], ctypes.c_int),
        "gram": ([vp, vp, i64, i32, vp, i64, i32, vp, i64], ctypes.c_int),
        "gemm": ([vp, f64, vp, i64, i32, vp, i64, i32, f64, vp, i64, vp, i64], ctypes.c_int),
        "orthonormalize": ([vp, vp, i64, i32, pi32], ctypes.c_int),
        "arr_project": ([vp, vp, i64, vp, i64, pf64, pi32], ctypes.c_int),
        "arr_project_p": ([vp, i32, vp, i64, vp, i64, pf64, pi32], ctypes.c_int),
        "residuals": ([vp, vp, i64, pf64, i32, pf64], ctypes.c_int),
        "eig_solve": ([vp, vp, i64, ctypes.POINTER(arr_solve_opts), pf64, pf64,
                       ctypes.POINTER(arr_solve_info)], ctypes.c_int),
        "eig_solve_host": ([i64, i64, vp, vp, vp, i32, i32, i32, i32, vp, ctypes.POINTER(arr_solve_opts), pf64, pf64,
                            vp, ctypes.POINTER(arr_solve_info), vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib
