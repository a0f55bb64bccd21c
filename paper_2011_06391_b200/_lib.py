"""ctypes binding of libfusedmm_cuda's C ABI (include/fusedmm_cuda.h).

This is the same binding a Python maintainer of the reference would add
(INTEGRATION.md). There is no fallback: if the in-tree library is missing the
import fails loudly with the build command.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("FMM_CUDA_LIB", _PKG / "lib" / "libfusedmm_cuda.so"))
GEN_PATH = _PKG / "lib" / "libfmm_gen.so"

# status codes
FMM_OK, FMM_E_INVAL, FMM_E_UNSUPPORTED, FMM_E_CUDA, FMM_E_NCCL, FMM_E_OOM, FMM_E_LOGIC = range(7)
# flags
FMM_HOST_PTRS = 0
FMM_DEVICE_PTRS = 1 << 0
FMM_ASYNC = 1 << 1
FMM_EXACT = 1 << 2
FMM_FAST = 1 << 3
FMM_EXCHANGE_COPIES = 1 << 4
FMM_PEERS_ALL = 1 << 5


class fmm_opspec(C.Structure):
    _fields_ = [("vop", C.c_int32), ("rop", C.c_int32), ("sop", C.c_int32),
                ("mop", C.c_int32), ("aop", C.c_int32), ("alpha", C.c_float), ("k", C.c_float),
                ("mlp_wx", C.c_float), ("mlp_wy", C.c_float), ("mlp_b", C.c_float)]


class fmm_stats(C.Structure):
    _fields_ = [("aux_bytes", C.c_uint64), ("threads", C.c_int32), ("pattern", C.c_int32),
                ("exact", C.c_int32), ("launches", C.c_int32), ("kernel_ms", C.c_float),
                ("total_ms", C.c_float)]


class fmm_graph_info(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64),
                ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("nonempty_rows", C.c_int64), ("max_degree", C.c_int64),
                ("split_rows", C.c_int64), ("split_chunks", C.c_int64),
                ("shards", C.c_int32), ("has_values", C.c_int32),
                ("exchange_rows", C.c_int64), ("exchange_rows_all", C.c_int64)]


# every symbol include/fusedmm_cuda.h declares: name -> (restype, argtypes)
_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_FP = C.POINTER(C.c_float)
SIGNATURES = {
    "fmm_version": (C.c_char_p, []),
    "fmm_status_string": (C.c_char_p, [C.c_int]),
    "fmm_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(_P)]),
    "fmm_destroy": (C.c_int, [_P]),
    "fmm_last_error": (C.c_char_p, [_P]),
    "fmm_device_count": (C.c_int, []),
    "fmm_set_stream": (C.c_int, [_P, C.c_int, _P]),
    "fmm_reset_stream": (C.c_int, [_P, C.c_int]),
    "fmm_set_variant": (C.c_int, [_P, C.c_int]),
    "fmm_get_variant": (C.c_int, [_P]),
    "fmm_pattern_of": (C.c_int, [C.POINTER(fmm_opspec), C.POINTER(C.c_int32)]),
    "fmm_part1d": (C.c_int, [C.c_int64, _I64P, C.c_int, _I64P]),
    "fmm_part1d_weighted": (C.c_int, [C.c_int64, _I64P, C.c_int, C.c_double, _I64P]),
    "fmm_set_row_weight": (C.c_int, [_P, C.c_double]),
    "fmm_plan_pieces": (C.c_int, [C.c_int64, C.c_int64, _I64P, _I64P, C.c_int64, C.c_int64, _I64P, _I64P, _I64P,
                                  _I64P, _I64P, C.c_int64]),
    "fmm_graph_upload": (C.c_int, [_P, C.c_int64, C.c_int64, _I64P, _I64P, _FP, C.c_int64,
                                   C.c_int64, C.POINTER(_P)]),
    "fmm_graph_free": (C.c_int, [_P]),
    "fmm_graph_update_values": (C.c_int, [_P, _FP]),
    "fmm_fingerprint": (C.c_uint64, [_P, C.c_size_t]),
    "fmm_graph_column_use": (C.c_int, [_P, _P]),
    "fmm_graph_set_peer_mask": (C.c_int, [_P, _P, C.c_int]),
    "fmm_graph_get_info": (C.c_int, [_P, C.POINTER(fmm_graph_info)]),
    "fmm_graph_shard_bounds": (C.c_int, [_P, _I64P]),
    "fmm_run": (C.c_int, [_P, _P, C.POINTER(fmm_opspec), C.c_int64, _P, C.c_int64, _P, _P,
                          C.c_uint32, C.POINTER(fmm_stats)]),
    "fmm_iterate": (C.c_int, [_P, _P, C.POINTER(fmm_opspec), C.c_int64, _P, C.c_int,
                              C.c_uint32, C.POINTER(fmm_stats)]),
    "fmm_sync": (C.c_int, [_P]),
    "fmm_run_unfused": (C.c_int, [_P, _P, C.POINTER(fmm_opspec), C.c_int64, _P, C.c_int64, _P, _P,
                                  C.c_uint32, C.POINTER(fmm_stats)]),
    "fmm_host_alloc": (C.c_int, [C.POINTER(_P), C.c_size_t]),
    "fmm_host_free": (C.c_int, [_P]),
    "fmm_run_peers": (C.c_int, [_P, _P, C.POINTER(fmm_opspec), C.c_int64, _P, C.c_int64, _P, _P,
                                C.POINTER(_P), C.c_int, C.c_uint32, C.POINTER(fmm_stats)]),
    "fmm_ipc_handle": (C.c_int, [_P, _P, C.POINTER(C.c_uint64)]),
    "fmm_ipc_open": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "fmm_ipc_close": (C.c_int, [_P]),
    "fmm_csr_from_coo": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, _I64P, _I64P, _FP, _I64P,
                                   _I64P, _FP, _I64P]),
    "fmm_read_matrix_market": (C.c_int, [C.c_char_p, C.c_int, _I64P, _I64P, _I64P, C.POINTER(_I64P),
                                         C.POINTER(_I64P), C.POINTER(_FP), C.c_char_p, C.c_size_t]),
    "fmm_write_matrix_market": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, _I64P, _I64P, _FP]),
    "fmm_free": (None, [_P]),
    "fmm_csr_sym_unique": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _I64P, _I64P, C.c_int, C.c_int,
                                     _I64P, _I64P, _I64P]),
    "fmm_rmat_device": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                  C.c_int, _I64P, _I64P, _FP, _I64P, _I64P, _I64P]),
    "fmm_mt64_window": (C.c_int, [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]),
}

_lib = None
_gen = None


def lib() -> C.CDLL:
    """Load libfusedmm_cuda.so; raise (never fall back) when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"libfusedmm_cuda.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2011_06391_b200.build` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def gen() -> C.CDLL:
    global _gen
    if _gen is None:
        if not GEN_PATH.exists():
            raise ImportError(f"libfmm_gen.so not found at {GEN_PATH}; run the build")
        G = C.CDLL(str(GEN_PATH))
        G.fmmgen_free.argtypes = [_P]
        G.fmmgen_er_fixed.argtypes = [C.c_int64, C.c_int, C.c_uint64, _I64P, _I64P, _FP, _FP,
                                      C.c_int64]
        G.fmmgen_rmat_sym.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_uint64, C.POINTER(_I64P), C.POINTER(_I64P), _I64P]
        G.fmmgen_rmat_stream.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_uint64, _I64P, _I64P]
        G.fmmgen_lattice.argtypes = [C.c_int64, C.c_uint64, C.POINTER(_I64P), C.POINTER(_I64P),
                                     _I64P, _FP]
        G.fmmgen_normal_fill.argtypes = [_FP, C.c_int64, C.c_double, C.c_uint64]
        G.fmmgen_uniform_fill.argtypes = [_FP, C.c_int64, C.c_double, C.c_double, C.c_uint64]
        _gen = G
    return _gen
