"""ctypes binding of libmcfunm_cuda.so (declared in include/mcfunm_cuda.h).

This is the reference-side binding a maintainer would add:
plain pointers and sizes, no torch types cross the boundary.  Loading fails
loudly -- there is no CPU fallback on the product path."""

from __future__ import annotations

import ctypes as C
import os

from .errors import BY_CODE, McfunmError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCFUNM_CUDA_LIB", os.path.join(_HERE, "lib", "libmcfunm_cuda.so"))

MCF_STATS_LEN = 4
MCF_FLAG_TIME_KERNELS = 1
MCF_FLAG_RETURN_ONLY = 2
MCF_FLAG_WALK_GROUP = 4
MCF_EDGES_DROP_LOOPS = 1
MCF_EDGES_ADD_REVERSE = 2
MCF_EDGES_FAIL_ON_DUPLICATES = 4


def group_flags(groups: int, index: int) -> int:
    """MCF_GROUP_FLAGS(G, g) of include/mcfunm_cuda.h: only walks w = g mod G."""
    return MCF_FLAG_WALK_GROUP | (((groups - 1) & 0xFF) << 8) | ((index & 0xFF) << 16)

P = C.c_void_p
I64 = C.c_int64


class McfCsr(C.Structure):
    _fields_ = [("n", I64), ("nnz", I64), ("row_ptr", P), ("col_ids", P), ("vals", P),
                ("csc_ptr", P), ("csc_rows", P), ("csc_vals", P)]


class McfGraphInfo(C.Structure):
    _fields_ = [("n", I64), ("nnz", I64), ("n_uniform_rows", I64), ("n_empty_rows", I64),
                ("n_negative", I64), ("max_degree", I64), ("max_row_abs_sum", C.c_double),
                ("col_norm_total", C.c_double), ("walk_layout", I64)]


class McfWalkParams(C.Structure):
    _fields_ = [("max_steps", I64), ("weight_cutoff", C.c_double), ("seed", C.c_uint64),
                ("zeta", P), ("walk_capacity", I64), ("flags", C.c_int32)]


# name -> (restype, argtypes); exactly the symbols include/mcfunm_cuda.h declares
SIGNATURES = {
    "mcf_version": (C.c_char_p, []),
    "mcf_last_error": (C.c_char_p, []),
    "mcf_kernel_launches": (I64, []),
    "mcf_graph_kernel_times": (C.c_int, [P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(I64), C.c_int]),
    "mcf_graph_create": (C.c_int, [C.POINTER(McfCsr), P, C.POINTER(P)]),
    "mcf_graph_destroy": (C.c_int, [P]),
    "mcf_graph_get_info": (C.c_int, [P, C.POINTER(McfGraphInfo)]),
    "mcf_graph_tables": (C.c_int, [P, P, P, P, P]),
    "mcf_allocate_walks": (C.c_int, [P, I64, P, P, P]),
    "mcf_spmv": (C.c_int, [P, C.c_double, P, C.c_double, P, P, P, I64, I64, P]),
    "mcf_spmv_peer": (C.c_int, [P, C.c_double, P, C.c_double, P, P, P, C.c_int, P, C.c_int, I64, I64, P]),
    "mcf_peer_alloc": (C.c_int, [I64, C.POINTER(P), P]),
    "mcf_peer_open": (C.c_int, [P, C.POINTER(P)]),
    "mcf_peer_close": (C.c_int, [P]),
    "mcf_peer_free": (C.c_int, [P]),
    "mcf_walk_action": (C.c_int, [P, C.POINTER(McfWalkParams), P, I64, I64, P, P, P, P, P]),
    "mcf_funm_action": (C.c_int, [P, C.POINTER(McfWalkParams), C.c_int64, P, P, P, C.c_double, C.c_double, P, P, P, P, P, P]),
    "mcf_replay_action": (C.c_int, [P, C.POINTER(McfWalkParams), P, I64, I64, P, P, P, P, P, P]),
    "mcf_walk_diag": (C.c_int, [P, C.POINTER(McfWalkParams), P, I64, I64, P, P, P]),
    "mcf_replay_diag": (C.c_int, [P, C.POINTER(McfWalkParams), P, I64, I64, P, P, P, P, P]),
    "mcf_diag_combine": (C.c_int, [P, C.c_double, C.c_double, P, P, I64, I64, P]),
    "mcf_diag_combine_peer": (C.c_int, [P, C.c_double, C.c_double, P, P, C.c_int, P, C.c_int, I64, I64, P]),
    "mcf_walk_qdense": (C.c_int, [P, C.POINTER(McfWalkParams), P, I64, I64, P, I64, P, P]),
    "mcf_column_costs": (C.c_int, [P, P, I64, C.c_int, P, P]),
    "mcf_gen_rmat_keys": (C.c_int, [C.c_int, I64, C.c_double, C.c_double, C.c_double, C.c_uint64, P, P]),
    "mcf_gen_chung_lu_keys": (C.c_int, [P, I64, I64, C.c_uint64, P, P]),
    "mcf_edges_to_csr": (C.c_int, [P, I64, I64, C.c_int, P, P, I64, C.POINTER(I64), P]),
    "mcf_csr_compact": (C.c_int, [I64, P, P, I64, P, P, C.POINTER(I64), P]),
    "mcf_funm_full": (C.c_int, [P, C.POINTER(McfWalkParams), P, C.c_double, C.c_double, P, I64, I64, P, P]),
    "mcf_diag_variance": (C.c_int, [P, P, C.c_int, P, P, I64, I64, P]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen the library and bind every declared symbol (no device needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise McfunmError(f"libmcfunm_cuda.so not found at {path}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib


def lib():
    return load_library()


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().mcf_last_error().decode(errors="replace")
        raise BY_CODE.get(rc, McfunmError)(f"{what}: {msg}" if what else msg)
