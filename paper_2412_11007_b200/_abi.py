"""ctypes declarations of the C-ABI in include/tcs/tcs.h.

The shared library is built in-tree (``make lib`` -> libtcsparse_b200.so
next to this file).  Loading fails loudly when it is missing: there is no
CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TCS_LIB_PATH: load an experimental build instead (tools/build_variant.sh)
LIB_PATH = os.environ.get("TCS_LIB_PATH") or os.path.join(_HERE, "libtcsparse_b200.so")

(TCS_OK, TCS_ERR_ARGUMENT, TCS_ERR_SHAPE, TCS_ERR_FORMAT, TCS_ERR_CUDA, TCS_ERR_NCCL, TCS_ERR_OOM, TCS_ERR_PARSE,
 TCS_ERR_IO) = range(9)
TCS_MAP_DIRECT, TCS_MAP_COALESCED = 0, 1
TCS_CFG_COUNT_ACCESS = 0x4
TCS_FP16, TCS_TF32 = 0, 1
TCS_DTYPE_F16, TCS_DTYPE_F32 = 0, 1
TCS_MEBCRS_OWN_STRUCTURE, TCS_MEBCRS_OWN_VALUES = 1, 2

u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)


class tcs_csr(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class tcs_mebcrs(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("vector_height", C.c_uint32),
                ("k", C.c_uint32), ("precision", C.c_int), ("value_dtype", C.c_int),
                ("num_windows", C.c_uint64), ("num_vectors", C.c_uint64),
                ("row_pointers", C.c_void_p), ("column_indices", C.c_void_p), ("values", C.c_void_p),
                ("flags", C.c_uint32), ("max_window_vectors", C.c_uint32),
                ("num_blocks", C.c_uint64), ("num_groups16", C.c_uint64), ("plan", C.c_void_p)]


class tcs_srbcrs(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("vector_height", C.c_uint32),
                ("k", C.c_uint32), ("precision", C.c_int), ("value_dtype", C.c_int),
                ("num_windows", C.c_uint64), ("num_padded", C.c_uint64),
                ("row_pointer_pairs", C.c_void_p), ("column_indices", C.c_void_p), ("values", C.c_void_p),
                ("impl", C.c_void_p)]


TCS_SR_PADDING = 0xFFFFFFFF


class tcs_kernel_config(C.Structure):
    _fields_ = [("precision", C.c_int), ("vector_height", C.c_uint32), ("mapping", C.c_int),
                ("flags", C.c_uint32)]


class tcs_counters(C.Structure):
    _fields_ = [("mma_invocations", C.c_uint64), ("transactions", C.c_uint64),
                ("transaction_bytes", C.c_uint64), ("useful_bytes", C.c_uint64)]


class tcs_cost(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("mma_count", "zero_fill", "access_bytes", "transactions",
                                          "exec_transactions", "exec_transaction_bytes", "exec_useful_bytes",
                                          "footprint_me", "footprint_sr", "padded_vectors")]


class tcs_dist(C.Structure):
    _fields_ = [("comm", C.c_void_p), ("rank", C.c_int), ("world", C.c_int), ("timeout_ms", C.c_int64)]


TCS_DIST_BROADCAST_B, TCS_DIST_ALLGATHER_C = 0x1, 0x2

EXPORTS = {
    # include/tcs/tcs_dist.h
    "tcs_dist_init": (C.c_int, [C.POINTER(tcs_dist), C.c_void_p, C.c_int64]),
    "tcs_shard_windows": (C.c_int, [C.POINTER(tcs_csr), C.c_int, C.c_void_p, C.c_void_p]),
    "tcs_mebcrs_encode_shard": (C.c_int, [C.POINTER(tcs_csr), C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                          C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_dist_broadcast": (C.c_int, [C.POINTER(tcs_dist), C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]),
    "tcs_spmm_sharded": (C.c_int, [C.POINTER(tcs_dist), C.c_void_p, C.c_uint64, C.POINTER(tcs_mebcrs), C.c_void_p,
                                   C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_uint32, C.c_void_p,
                                   C.c_int64, C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters), C.c_void_p]),
    "tcs_dist_wait": (C.c_int, [C.POINTER(tcs_dist), C.c_void_p, C.c_int64]),
    "tcs_spmm_sharded_csr_host": (C.c_int, [C.POINTER(tcs_dist), C.POINTER(tcs_csr), C.c_int, C.c_void_p, C.c_int64,
                                            C.c_int, C.c_void_p, C.POINTER(tcs_kernel_config),
                                            C.POINTER(tcs_counters), C.c_void_p]),
    # include/tcs/tcs.h
    # name: (restype, argtypes)
    "tcs_version": (C.c_char_p, []),
    "tcs_last_error": (C.c_char_p, []),
    "tcs_launch_count": (C.c_uint64, []),
    "tcs_round_values": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "tcs_mebcrs_encode": (C.c_int, [C.POINTER(tcs_csr), C.c_int, C.c_int, C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_encode_v": (C.c_int, [C.POINTER(tcs_csr), C.c_int, C.c_int, C.c_uint32, C.POINTER(tcs_mebcrs),
                                      C.c_void_p]),
    "tcs_spmm_baseline16": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                      C.c_void_p, C.c_int64, C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters),
                                      C.c_void_p]),
    "tcs_srbcrs_encode": (C.c_int, [C.POINTER(tcs_csr), C.c_int, C.c_int, C.POINTER(tcs_srbcrs), C.c_void_p]),
    "tcs_srbcrs_from_mebcrs": (C.c_int, [C.POINTER(tcs_mebcrs), C.POINTER(tcs_srbcrs), C.c_void_p]),
    "tcs_srbcrs_upload": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(tcs_srbcrs), C.c_void_p]),
    "tcs_srbcrs_download": (C.c_int, [C.POINTER(tcs_srbcrs), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tcs_srbcrs_free": (C.c_int, [C.POINTER(tcs_srbcrs), C.c_void_p]),
    "tcs_srbcrs_decode": (C.c_int, [C.POINTER(tcs_srbcrs), C.POINTER(tcs_csr), C.c_void_p]),
    "tcs_spmm_srbcrs": (C.c_int, [C.POINTER(tcs_srbcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_void_p, C.c_int64, C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters),
                                  C.c_void_p]),
    "tcs_spmm_srbcrs_host": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.POINTER(tcs_kernel_config),
                                       C.POINTER(tcs_counters), C.c_void_p]),
    "tcs_mebcrs_cost": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_uint64, C.c_int64, C.c_int, C.POINTER(tcs_cost),
                                  C.c_void_p]),
    "tcs_matrix_market_parse": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(tcs_csr), C.c_void_p]),
    "tcs_matrix_market_read": (C.c_int, [C.c_char_p, C.POINTER(tcs_csr), C.c_void_p]),
    "tcs_matrix_market_write": (C.c_int, [C.c_char_p, C.POINTER(tcs_csr)]),
    "tcs_csr_free_host": (C.c_int, [C.POINTER(tcs_csr)]),
    "tcs_coo_to_csr": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.POINTER(tcs_csr), C.c_void_p]),
    "tcs_csr_free": (C.c_int, [C.POINTER(tcs_csr), C.c_void_p]),
    "tcs_mebcrs_write": (C.c_int, [C.c_char_p, C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_read": (C.c_int, [C.c_char_p, C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_prepare": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_validate": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_free": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_decode": (C.c_int, [C.POINTER(tcs_mebcrs), C.POINTER(tcs_csr), C.c_void_p]),
    "tcs_csr_download": (C.c_int, [C.POINTER(tcs_csr), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tcs_spmm": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                           C.c_void_p, C.c_int64, C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters),
                           C.c_void_p]),
    "tcs_sddmm": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                            C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.POINTER(tcs_mebcrs), C.c_int,
                            C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters), C.c_void_p]),
    "tcs_mebcrs_row_softmax": (C.c_int, [C.POINTER(tcs_mebcrs), C.POINTER(tcs_mebcrs), C.c_float,
                                         C.POINTER(tcs_mebcrs), C.c_int, C.c_void_p]),
    "tcs_sddmm_row_softmax": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, C.c_int,
                                        C.POINTER(tcs_mebcrs), C.c_int, C.POINTER(tcs_kernel_config), C.c_void_p]),
    "tcs_agnn_aggregate": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_float, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p,
                                     C.c_int64, C.POINTER(tcs_kernel_config), C.c_void_p]),
    "tcs_agnn_attend": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_float, C.c_float, C.c_void_p, C.c_int64, C.POINTER(tcs_kernel_config),
                                  C.c_void_p]),
    "tcs_rows_normalize": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_int64, C.c_int, C.c_float, C.c_void_p]),
    "tcs_mebcrs_encode_host": (C.c_int, [C.POINTER(tcs_csr), C.c_int, C.c_int, C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_mebcrs_download": (C.c_int, [C.POINTER(tcs_mebcrs), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tcs_mebcrs_upload": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(tcs_mebcrs), C.c_void_p]),
    "tcs_spmm_host": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_int64, C.c_int64, C.c_void_p, C.POINTER(tcs_kernel_config),
                                C.POINTER(tcs_counters), C.c_void_p]),
    "tcs_sddmm_host": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                 C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters), C.c_void_p]),
    "tcs_spmm_csr_host": (C.c_int, [C.POINTER(tcs_csr), C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters), C.c_void_p]),
    "tcs_spmm_baseline16_csr_host": (C.c_int, [C.POINTER(tcs_csr), C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                               C.POINTER(tcs_kernel_config), C.POINTER(tcs_counters),
                                               C.c_void_p]),
}

_lib = None


def load():
    """Loads libtcsparse_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make lib` (or __graft_entry__.build())")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
