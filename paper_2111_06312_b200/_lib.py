"""ctypes declarations of include/isvd.h (argument marshalling only).

The shared library is ``libisvd.so`` next to this file, built by
``paper_2111_06312_b200._build`` for sm_100a.  There is no fallback: if the
library is missing or cannot be loaded, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libisvd.so")

ISVD_OK = 0
STATUS_NAMES = {
    0: "ISVD_OK", 1: "ISVD_ERR_INVALID_ARG", 2: "ISVD_ERR_SHAPE", 3: "ISVD_ERR_RANK", 4: "ISVD_ERR_INDEX",
    5: "ISVD_ERR_NONFINITE", 6: "ISVD_ERR_OOM", 7: "ISVD_ERR_CUDA", 8: "ISVD_ERR_NCCL", 9: "ISVD_ERR_NOT_PD",
    10: "ISVD_ERR_BUSY", 11: "ISVD_ERR_UNSUPPORTED",
}

ISVD_PTR_DEVICE = 1
ISVD_GRAPH_SYMMETRIC = 2
ISVD_GRAPH_VALIDATE = 4
ISVD_BORROW = 8

ISVD_OP_POWER_SUM = 1
ISVD_OP_STACKED_PROPAGATION = 2

ISVD_BASIS_DEFAULT = 0
ISVD_BASIS_T_ROW = 1
ISVD_BASIS_AHAT_SYM = 2

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]

ISVD_SVD_OMEGA_PROVIDED = 1
ISVD_SVD_HOST_OUTPUT = 2
ISVD_SVD_NO_GRAPH = 4
ISVD_SVD_FORCE_CHOL_FAIL = 8
ISVD_SVD_PROFILE = 16


class OpDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("num_terms", C.c_int32),
        ("weights", C.POINTER(C.c_double)),
        ("lambda_ones", C.c_double),
        ("lambda_adj", C.c_double),
        ("X", C.c_void_p),
        ("d", C.c_int64),
        ("ldx", C.c_int64),
        ("x_flags", C.c_uint32),
        ("Y", C.c_void_p),
        ("y", C.c_int64),
        ("ldy", C.c_int64),
        ("lr_powers", C.c_int32),
        ("y_flags", C.c_uint32),
        ("basis", C.c_int32),
        ("pad0", C.c_int32),
        ("rows", C.POINTER(C.c_int64)),
        ("n_rows", C.c_int64),
    ]


class SvdParams(C.Structure):
    _fields_ = [
        ("k", C.c_int32),
        ("oversampling", C.c_int32),
        ("power_iters", C.c_int32),
        ("seed", C.c_uint64),
        ("flags", C.c_uint32),
        ("omega", C.c_void_p),
    ]


class SvdReport(C.Structure):
    _fields_ = [
        ("l", C.c_int32),
        ("ld", C.c_int32),
        ("chol_fallbacks", C.c_int32),
        ("jacobi_sweeps", C.c_int32),
        ("world", C.c_int32),
        ("kernel_launches", C.c_int32),
        ("ms_total", C.c_double),
        ("spmm_steps", C.c_int32),
        ("pad0", C.c_int32),
        ("ms_spmm", C.c_double),
        ("spmm_alg_bytes", C.c_double),
        ("ms_products", C.c_double),
        ("ms_orth", C.c_double),
        ("ms_small", C.c_double),
        ("ms_comm", C.c_double),
        ("gram_probe_fallbacks", C.c_int32),
        ("gram_probe_skipped", C.c_int32),
        ("ms_allgather", C.c_double),
        ("ms_allgather_hidden", C.c_double),
    ]


# name -> (restype, argtypes); every entry point of include/isvd.h
SIGNATURES = {
    "isvd_abi_version": (C.c_int, []),
    "isvd_status_string": (C.c_char_p, [C.c_int]),
    "isvd_last_error": (C.c_char_p, [C.c_void_p]),
    "isvd_partition": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "isvd_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_size_t]),
    "isvd_ctx_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(Allocator), C.c_void_p, C.c_int, C.c_int,
                                  C.POINTER(C.c_void_p)]),
    "isvd_sim_group_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "isvd_sim_group_destroy": (C.c_int, [C.c_void_p]),
    "isvd_ctx_create_sim": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(Allocator), C.c_void_p, C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "isvd_ctx_destroy": (C.c_int, [C.c_void_p]),
    "isvd_graph_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "isvd_graph_destroy": (C.c_int, [C.c_void_p]),
    "isvd_graph_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64)]),
    "isvd_op_define": (C.c_int, [C.c_void_p, C.POINTER(OpDesc), C.POINTER(C.c_void_p)]),
    "isvd_op_shape": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "isvd_op_destroy": (C.c_int, [C.c_void_p]),
    "isvd_matmul": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64]),
    "isvd_matmul_T": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64]),
    "isvd_svd": (C.c_int, [C.c_void_p, C.POINTER(SvdParams), C.c_void_p, C.c_int64, C.POINTER(C.c_double),
                           C.c_void_p, C.c_int64, C.POINTER(SvdReport)]),
    "isvd_sample_omega": (C.c_int, [C.c_void_p, C.POINTER(SvdParams), C.c_void_p, C.c_int64]),
    "isvd_embeddings": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                  C.POINTER(C.c_double), C.c_void_p, C.c_int64]),
    "isvd_spectral_kernel": (C.c_int, [C.POINTER(C.c_double), C.c_int64, C.c_double, C.c_double,
                                       C.POINTER(C.c_double)]),
    "isvd_least_norm": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_double),
                                  C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                  C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]),
}

_lib = None


def load():
    """Load libisvd.so (raises if absent: there is no CPU or eager fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2111_06312_b200._build` "
            "(nvcc, sm_100a). The isvd path has no fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class IsvdError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{where}: {name}" + (f" ({detail})" if detail else ""))


def check(status: int, where: str, ctx=None):
    if status != ISVD_OK:
        detail = ""
        if ctx is not None:
            detail = (load().isvd_last_error(ctx) or b"").decode(errors="replace")
        raise IsvdError(status, where, detail)
