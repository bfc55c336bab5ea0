"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end of the CPU oracle.

Two libraries sit behind this module:

* ``liboracle.so`` -- the CPU restatement in ``oracle/oracle.cpp`` (each
  function cites the reference file:line it follows).
* ``_ref/libtcsref.so`` -- the reference's own headers compiled unmodified
  behind a C-ABI shim (``oracle/ref_shim.cpp``), built here where
  ``/root/reference`` exists and shipped prebuilt to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package; the product library never
does (and has no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_u32p = C.POINTER(C.c_uint32)
_f32p = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)

FP16, TF32 = 0, 1
K_OF = {FP16: 8, TF32: 4}


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load(name):
    path = os.path.join(_HERE, name)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    return C.CDLL(path)


_orc = None
_ref = None


def lib():
    global _orc
    if _orc is None:
        _orc = _load("liboracle.so")
        _orc.orc_round_fp16.restype = C.c_float
        _orc.orc_round_fp16.argtypes = [C.c_float]
        _orc.orc_round_tf32.restype = C.c_float
        _orc.orc_round_tf32.argtypes = [C.c_float]
        _orc.orc_generate_random_sparse.restype = C.c_int64
        _orc.orc_generate_random_sparse.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                                    C.c_int, C.POINTER(_u32p), C.POINTER(_u32p),
                                                    C.POINTER(_f32p)]
        _orc.orc_generate_random_dense.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _f32p]
        _orc.orc_mebcrs_row_pointers.restype = C.c_int64
        _orc.orc_mebcrs_row_pointers.argtypes = [C.c_uint64, _u32p, _u32p, _u32p]
        _orc.orc_mebcrs_fill.argtypes = [C.c_uint64, _u32p, _u32p, _f32p, C.c_uint32, _u32p, _u32p, _f32p]
        _orc.orc_mebcrs_row_pointers_v.restype = C.c_int64
        _orc.orc_mebcrs_row_pointers_v.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _u32p]
        _orc.orc_mebcrs_fill_v.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, C.c_uint32, _u32p, _u32p,
                                           _f32p]
        _orc.orc_spmm_v.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, _u32p, _u32p, _f32p, _f32p,
                                    C.c_uint64, C.c_uint64, _f32p, C.c_uint64, C.c_int]
        _orc.orc_mebcrs_to_dense.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, _u32p, _u32p, _f32p, _f32p]
        _orc.orc_spmm.argtypes = [C.c_uint64, C.c_uint32, C.c_int, _u32p, _u32p, _f32p, _f32p,
                                  C.c_uint64, C.c_uint64, _f32p, C.c_uint64, C.c_int]
        _orc.orc_sddmm.argtypes = [C.c_uint64, C.c_uint32, C.c_int, _u32p, _u32p, _f32p, _f32p,
                                   C.c_uint64, _f32p, C.c_uint64, C.c_uint64, _f32p]
        _orc.orc_count_mma_spmm.restype = C.c_uint64
        _orc.orc_count_mma_spmm.argtypes = [C.c_uint64, _u32p, C.c_uint32, C.c_uint64]
        _orc.orc_count_mma_sddmm.restype = C.c_uint64
        _orc.orc_count_mma_sddmm.argtypes = [C.c_uint64, _u32p, C.c_uint32, C.c_uint64]
        _orc.orc_num_threads.restype = C.c_int
        _orc.orc_set_num_threads.argtypes = [C.c_int]
        _orc.orc_mt19937.argtypes = [C.c_uint32, C.c_uint64, _u32p]
        _orc.orc_round_array.argtypes = [C.c_int, _f32p, _f32p, C.c_uint64]
        _orc.orc_free.argtypes = [C.c_void_p]
    return _orc


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref", "libtcsref.so"))


def ref():
    global _ref
    if _ref is None:
        _ref = _load(os.path.join("_ref", "libtcsref.so"))
        _ref.ref_round_fp16.restype = C.c_float
        _ref.ref_round_fp16.argtypes = [C.c_float]
        _ref.ref_round_tf32.restype = C.c_float
        _ref.ref_round_tf32.argtypes = [C.c_float]
        _ref.ref_generate_random_sparse.restype = C.c_int64
        _ref.ref_generate_random_sparse.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                                    C.c_int, C.POINTER(_u32p), C.POINTER(_u32p),
                                                    C.POINTER(_f32p)]
        _ref.ref_generate_random_dense.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _f32p]
        _ref.ref_encode_mebcrs.restype = C.c_int64
        _ref.ref_encode_mebcrs.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, C.c_int,
                                           C.POINTER(_u32p), C.POINTER(_u32p), C.POINTER(_f32p)]
        _ref.ref_decode_mebcrs.restype = C.c_int64
        _ref.ref_decode_mebcrs.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _u32p, _u32p, _f32p,
                                           C.POINTER(_u32p), C.POINTER(_u32p), C.POINTER(_f32p)]
        _ref.ref_spmm.restype = C.c_int
        _ref.ref_spmm.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _u32p, _u32p, _f32p, _f32p,
                                  C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_int, _f32p, _u64p]
        _ref.ref_sddmm.restype = C.c_int
        _ref.ref_sddmm.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _u32p, _u32p, _f32p, _f32p,
                                   C.c_uint64, _f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                   _f32p, _u64p]
        _ref.ref_partition_windows.restype = C.c_int64
        _ref.ref_partition_windows.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, C.c_uint64, C.c_uint64,
                                               C.POINTER(_u32p), C.POINTER(_u32p)]
        _ref.ref_spmm_baseline16.restype = C.c_int
        _ref.ref_spmm_baseline16.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, _f32p, C.c_uint64,
                                             C.c_uint64, C.c_int, C.c_uint64, _f32p, _u64p]
        _ref.ref_cli.restype = C.c_int
        _ref.ref_cli.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int, _u64p, C.c_int,
                                 C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_void_p)]
        _ref.ref_parse_matrix_market.restype = C.c_int64
        _ref.ref_parse_matrix_market.argtypes = [C.c_char_p, C.c_uint64, _u64p, _u64p, C.POINTER(_u32p),
                                                 C.POINTER(_u32p), C.POINTER(_f32p), C.POINTER(C.c_void_p)]
        _ref.ref_read_mebcrs.restype = C.c_int64
        _ref.ref_read_mebcrs.argtypes = [C.c_char_p, _u64p, _u64p, C.POINTER(C.c_int), C.POINTER(_u32p),
                                         C.POINTER(_u32p), C.POINTER(_f32p), C.POINTER(C.c_void_p)]
        _ref.ref_encode_srbcrs.restype = C.c_int64
        _ref.ref_encode_srbcrs.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, C.c_int,
                                           C.POINTER(_u32p), C.POINTER(_u32p), C.POINTER(_f32p)]
        _ref.ref_spmm_srbcrs.restype = C.c_int
        _ref.ref_spmm_srbcrs.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _u32p, _u32p, _f32p, _f32p, C.c_uint64,
                                         C.c_uint64, C.c_int, _f32p, _u64p]
        _ref.ref_sddmm_output_offsets.restype = C.c_uint64
        _ref.ref_sddmm_output_offsets.argtypes = [C.c_uint64, C.c_int]
        _ref.ref_free.argtypes = [C.c_void_p]
        _ref.ref_dense_new.restype = C.c_void_p
        _ref.ref_dense_new.argtypes = [C.c_uint64, C.c_uint64, _f32p]
        _ref.ref_dense_free.argtypes = [C.c_void_p]
        _ref.ref_time_encode_spmm.restype = C.c_double
        _ref.ref_time_encode_spmm.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, C.c_int, C.c_void_p,
                                              _f32p]
        _ref.ref_time_encode_sddmm.restype = C.c_double
        _ref.ref_time_encode_sddmm.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f32p, C.c_int, _f32p,
                                               C.c_uint64, C.c_void_p, _f32p, C.c_uint64]
    return _ref


def _p(a, t):
    return a.ctypes.data_as(t)


def _take(lib_, ptr, n, dtype):
    out = np.ctypeslib.as_array(ptr, shape=(max(n, 1),))[:n].astype(dtype, copy=True)
    lib_free = lib_.orc_free if hasattr(lib_, "orc_free") else lib_.ref_free
    lib_free(C.cast(ptr, C.c_void_p))
    return out


class Csr:
    """CSR matrix (inc/matrix.hpp:20-49): u32 row_ptr / col_idx, f32 values."""

    def __init__(self, rows, cols, row_ptr, col_idx, values):
        self.rows, self.cols = int(rows), int(cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint32)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.uint32)
        self.values = np.ascontiguousarray(values, dtype=np.float32)

    @property
    def nnz(self):
        return int(self.col_idx.shape[0])

    def to_dense(self):
        d = np.zeros((self.rows, self.cols), np.float32)
        r = np.repeat(np.arange(self.rows), np.diff(self.row_ptr.astype(np.int64)))
        d[r, self.col_idx] = self.values
        return d

    @staticmethod
    def from_dense(d):
        d = np.asarray(d, np.float32)
        rows, cols = d.shape
        r, c = np.nonzero(d)
        rp = np.zeros(rows + 1, np.uint32)
        np.cumsum(np.bincount(r, minlength=rows), out=rp[1:])
        return Csr(rows, cols, rp, c.astype(np.uint32), d[r, c])

    @staticmethod
    def from_coords(rows, cols, coords):
        """csr_from_coords (inc/matrix.hpp:100-128): duplicates summed, explicit zeros kept."""
        acc = {}
        for r, c, v in coords:
            acc[(r, c)] = acc.get((r, c), np.float32(0)) + np.float32(v)
        keys = sorted(acc)
        rp = np.zeros(rows + 1, np.uint32)
        for r, _ in keys:
            rp[r + 1] += 1
        rp = np.cumsum(rp).astype(np.uint32)
        return Csr(rows, cols, rp, [c for _, c in keys], [acc[k] for k in keys])


class MeBcrs:
    """ME-BCRS (inc/mebcrs.hpp:23-78) with f32 values (reference storage)."""

    def __init__(self, rows, cols, precision, row_pointers, column_indices, values, vector_height=8):
        self.rows, self.cols, self.precision = int(rows), int(cols), int(precision)
        self.vector_height = int(vector_height)
        self.k = K_OF[self.precision]
        self.row_pointers = np.ascontiguousarray(row_pointers, dtype=np.uint32)
        self.column_indices = np.ascontiguousarray(column_indices, dtype=np.uint32)
        self.values = np.ascontiguousarray(values, dtype=np.float32)

    @property
    def num_windows(self):
        return self.row_pointers.shape[0] - 1

    @property
    def nv(self):
        return int(self.column_indices.shape[0])


# ---------------------------------------------------------------- restatement
def generate_random_sparse(rows, cols, density, seed, real=False) -> Csr:
    rp, ci, v = _u32p(), _u32p(), _f32p()
    nnz = lib().orc_generate_random_sparse(rows, cols, density, seed, int(real),
                                           C.byref(rp), C.byref(ci), C.byref(v))
    if nnz < 0:
        raise ValueError("ArgumentError: bad generator arguments")
    o = lib()
    return Csr(rows, cols, _take(o, rp, rows + 1, np.uint32), _take(o, ci, nnz, np.uint32),
               _take(o, v, nnz, np.float32))


def generate_random_dense(rows, cols, seed, real=False) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    lib().orc_generate_random_dense(rows, cols, seed, int(real), _p(out, _f32p))
    return out


def encode_mebcrs(m: Csr, precision: int, vector_height: int = 8) -> MeBcrs:
    vh = vector_height
    W = (m.rows + vh - 1) // vh
    rp = np.empty(W + 1, np.uint32)
    nv = lib().orc_mebcrs_row_pointers_v(m.rows, vh, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p), _p(rp, _u32p))
    ci = np.empty(max(nv, 1), np.uint32)
    vals = np.empty(max(vh * nv, 1), np.float32)
    lib().orc_mebcrs_fill_v(m.rows, vh, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p), _p(m.values, _f32p),
                            K_OF[precision], _p(rp, _u32p), _p(ci, _u32p), _p(vals, _f32p))
    return MeBcrs(m.rows, m.cols, precision, rp, ci[:nv], vals[:vh * nv], vector_height=vh)


class SrBcrs:
    """ref srbcrs.hpp:17-38 (host arrays)."""

    def __init__(self, rows, cols, precision, row_pointer_pairs, column_indices, values):
        self.rows, self.cols, self.precision = rows, cols, precision
        self.k = K_OF[precision]
        self.row_pointer_pairs = np.ascontiguousarray(row_pointer_pairs, np.uint32)
        self.column_indices = np.ascontiguousarray(column_indices, np.uint32)
        self.values = np.ascontiguousarray(values, np.float32)


SR_PADDING = 0xFFFFFFFF  # ref kPaddingSentinel (srbcrs.hpp:12)


def encode_srbcrs(me: MeBcrs) -> SrBcrs:
    """Restatement of ref encode_srbcrs's padding loop (srbcrs.hpp:49-70),
    vectorised: window w keeps its nv_w columns and gains ceil(nv_w/k)*k -
    nv_w sentinel columns; block b is re-laid from width_b to k columns,
    zeros past width_b."""
    k, rp = me.k, me.row_pointers.astype(np.int64)
    W = len(rp) - 1
    nvw = np.diff(rp)
    padded = (nvw + k - 1) // k * k
    start = np.zeros(W + 1, np.int64)
    np.cumsum(padded, out=start[1:])
    P = int(start[-1])
    pairs = np.empty(2 * W, np.uint32)
    pairs[0::2], pairs[1::2] = start[:-1], start[1:]
    ci = np.full(P, SR_PADDING, np.uint32)
    vals = np.zeros(8 * P, np.float32)
    w_of = np.repeat(np.arange(W), nvw)                       # window of every stored vector
    j = np.arange(len(me.column_indices)) - rp[w_of]         # slot within its window
    ci[start[w_of] + j] = me.column_indices
    b, jj = j // k, j % k
    width = np.minimum(k, nvw[w_of] - b * k)
    for r in range(8):
        vals[8 * (start[w_of] + b * k) + r * k + jj] = me.values[8 * (rp[w_of] + b * k) + r * width + jj]
    return SrBcrs(me.rows, me.cols, me.precision, pairs, ci, vals)


def mebcrs_to_dense(me: MeBcrs) -> np.ndarray:
    d = np.empty((me.rows, me.cols), np.float32)
    lib().orc_mebcrs_to_dense(me.rows, me.cols, me.k, _p(me.row_pointers, _u32p),
                              _p(me.column_indices, _u32p), _p(me.values, _f32p), _p(d, _f32p))
    return d


def spmm(me: MeBcrs, B: np.ndarray, strict=False) -> np.ndarray:
    B = np.ascontiguousarray(B, np.float32)
    N = B.shape[1]
    Cm = np.zeros((me.rows, N), np.float32)
    lib().orc_spmm_v(me.rows, me.vector_height, me.k, me.precision, _p(me.row_pointers, _u32p),
                     _p(me.column_indices, _u32p), _p(me.values, _f32p), _p(B, _f32p), N, N, _p(Cm, _f32p), N,
                     int(strict))
    return Cm


def sddmm(mask: MeBcrs, A: np.ndarray, Bt: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, np.float32)
    Bt = np.ascontiguousarray(Bt, np.float32)
    F = A.shape[1]
    out = np.zeros(max(8 * mask.nv, 1), np.float32)
    lib().orc_sddmm(mask.rows, mask.k, mask.precision, _p(mask.row_pointers, _u32p),
                    _p(mask.column_indices, _u32p), _p(mask.values, _f32p), _p(A, _f32p), F,
                    _p(Bt, _f32p), F, F, _p(out, _f32p))
    return out[:8 * mask.nv]


def count_mma_spmm(me: MeBcrs, N: int) -> int:
    return int(lib().orc_count_mma_spmm(me.num_windows, _p(me.row_pointers, _u32p), me.k, N))


def count_mma_sddmm(me: MeBcrs, F: int) -> int:
    return int(lib().orc_count_mma_sddmm(me.num_windows, _p(me.row_pointers, _u32p), me.k, F))


def mt19937(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    lib().orc_mt19937(seed, n, _p(out, _u32p))
    return out


class Mt:
    """Sequential std::mt19937 stream (replays reference tests' draw order)."""

    def __init__(self, seed):
        self.seed, self.n = seed, 0
        self.buf = mt19937(seed, 1 << 16)

    def __call__(self):
        if self.n == self.buf.shape[0]:
            self.buf = mt19937(self.seed, 2 * self.buf.shape[0])
        v = int(self.buf[self.n])
        self.n += 1
        return v


def round_array(x: np.ndarray, precision: int) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    lib().orc_round_array(precision, _p(x, _f32p), _p(out, _f32p), x.size)
    return out


def round_fp16(x: float) -> float:
    return lib().orc_round_fp16(x)


def round_tf32(x: float) -> float:
    return lib().orc_round_tf32(x)


# ------------------------------------------------------ the reference itself
class Ref:
    """The unmodified reference (oracle/_ref/libtcsref.so)."""

    @staticmethod
    def generate_random_sparse(rows, cols, density, seed, real=False) -> Csr:
        r = ref()
        rp, ci, v = _u32p(), _u32p(), _f32p()
        nnz = r.ref_generate_random_sparse(rows, cols, density, seed, int(real),
                                           C.byref(rp), C.byref(ci), C.byref(v))
        if nnz < 0:
            raise ValueError("ArgumentError")
        return Csr(rows, cols, _take(r, rp, rows + 1, np.uint32), _take(r, ci, nnz, np.uint32),
                   _take(r, v, nnz, np.float32))

    @staticmethod
    def generate_random_dense(rows, cols, seed, real=False):
        out = np.empty((rows, cols), np.float32)
        ref().ref_generate_random_dense(rows, cols, seed, int(real), _p(out, _f32p))
        return out

    @staticmethod
    def encode_mebcrs(m: Csr, precision: int) -> MeBcrs:
        r = ref()
        rp, ci, v = _u32p(), _u32p(), _f32p()
        nv = r.ref_encode_mebcrs(m.rows, m.cols, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p),
                                 _p(m.values, _f32p), precision, C.byref(rp), C.byref(ci), C.byref(v))
        if nv < 0:
            raise ValueError("encode failed")
        W = (m.rows + 7) // 8
        return MeBcrs(m.rows, m.cols, precision, _take(r, rp, W + 1, np.uint32),
                      _take(r, ci, nv, np.uint32), _take(r, v, 8 * nv, np.float32))

    @staticmethod
    def decode_mebcrs(me: MeBcrs) -> Csr:
        r = ref()
        rp, ci, v = _u32p(), _u32p(), _f32p()
        nnz = r.ref_decode_mebcrs(me.rows, me.cols, me.precision, _p(me.row_pointers, _u32p),
                                  _p(me.column_indices, _u32p), _p(me.values, _f32p),
                                  C.byref(rp), C.byref(ci), C.byref(v))
        if nnz < 0:
            raise ValueError("FormatError")
        return Csr(me.rows, me.cols, _take(r, rp, me.rows + 1, np.uint32), _take(r, ci, nnz, np.uint32),
                   _take(r, v, nnz, np.float32))

    @staticmethod
    def spmm(me: MeBcrs, B, mapping=1, cfg_precision=None, vector_height=8):
        B = np.ascontiguousarray(B, np.float32)
        Cm = np.zeros((me.rows, B.shape[1]), np.float32)
        cnt = C.c_uint64(0)
        rc = ref().ref_spmm(me.rows, me.cols, me.precision, _p(me.row_pointers, _u32p),
                            _p(me.column_indices, _u32p), _p(me.values, _f32p), _p(B, _f32p),
                            B.shape[0], B.shape[1],
                            me.precision if cfg_precision is None else cfg_precision,
                            vector_height, mapping, _p(Cm, _f32p), C.byref(cnt))
        if rc:
            raise ValueError({1: "ArgumentError", 2: "ShapeError"}.get(rc, "error"))
        return Cm, int(cnt.value)

    @staticmethod
    def sddmm(mask: MeBcrs, A, Bt, cfg_precision=None):
        A = np.ascontiguousarray(A, np.float32)
        Bt = np.ascontiguousarray(Bt, np.float32)
        out = np.zeros(max(8 * mask.nv, 1), np.float32)
        cnt = C.c_uint64(0)
        rc = ref().ref_sddmm(mask.rows, mask.cols, mask.precision, _p(mask.row_pointers, _u32p),
                             _p(mask.column_indices, _u32p), _p(mask.values, _f32p), _p(A, _f32p),
                             A.shape[0], _p(Bt, _f32p), Bt.shape[0], A.shape[1], Bt.shape[1],
                             mask.precision if cfg_precision is None else cfg_precision,
                             _p(out, _f32p), C.byref(cnt))
        if rc:
            raise ValueError({1: "ArgumentError", 2: "ShapeError"}.get(rc, "error"))
        return out[:8 * mask.nv], int(cnt.value)

    @staticmethod
    def encode_srbcrs(m: Csr, precision: int) -> "SrBcrs":
        r = ref()
        pp, ci, v = _u32p(), _u32p(), _f32p()
        n = r.ref_encode_srbcrs(m.rows, m.cols, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p), _p(m.values, _f32p),
                                precision, C.byref(pp), C.byref(ci), C.byref(v))
        if n < 0:
            raise ValueError("encode failed")
        W = (m.rows + 7) // 8
        return SrBcrs(m.rows, m.cols, precision, _take(r, pp, 2 * W, np.uint32), _take(r, ci, n, np.uint32),
                      _take(r, v, 8 * n, np.float32))

    @staticmethod
    def spmm_srbcrs(sr: "SrBcrs", B, cfg_precision=None):
        B = np.ascontiguousarray(B, np.float32)
        Cm = np.zeros((sr.rows, B.shape[1]), np.float32)
        cnt = C.c_uint64(0)
        rc = ref().ref_spmm_srbcrs(sr.rows, sr.cols, sr.precision, _p(sr.row_pointer_pairs, _u32p),
                                   _p(sr.column_indices, _u32p), _p(sr.values, _f32p), _p(B, _f32p), B.shape[0],
                                   B.shape[1], sr.precision if cfg_precision is None else cfg_precision,
                                   _p(Cm, _f32p), C.byref(cnt))
        if rc:
            raise ValueError({1: "ArgumentError", 2: "ShapeError"}.get(rc, "error"))
        return Cm, int(cnt.value)

    @staticmethod
    def partition_windows(m: Csr, vector_height: int, k: int):
        """(row_pointers, column_indices) of ref partition_windows (partition.hpp:40-66)."""
        r = ref()
        rp, ci = _u32p(), _u32p()
        nv = r.ref_partition_windows(m.rows, m.cols, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p),
                                     _p(m.values, _f32p), vector_height, k, C.byref(rp), C.byref(ci))
        if nv < 0:
            raise ValueError("ArgumentError")
        W = (m.rows + vector_height - 1) // vector_height
        return _take(r, rp, W + 1, np.uint32), _take(r, ci, nv, np.uint32)

    @staticmethod
    def spmm_baseline16(m: Csr, B, precision: int, vector_height: int = 16):
        B = np.ascontiguousarray(B, np.float32)
        Cm = np.zeros((m.rows, B.shape[1]), np.float32)
        cnt = C.c_uint64(0)
        rc = ref().ref_spmm_baseline16(m.rows, m.cols, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p),
                                       _p(m.values, _f32p), _p(B, _f32p), B.shape[0], B.shape[1], precision,
                                       vector_height, _p(Cm, _f32p), C.byref(cnt))
        if rc:
            raise ValueError({1: "ArgumentError", 2: "ShapeError"}.get(rc, "error"))
        return Cm, int(cnt.value)

    @staticmethod
    def _str(ptr):
        if not ptr:
            return None
        out = C.cast(ptr, C.c_char_p).value.decode()
        ref().ref_free(ptr)
        return out

    @staticmethod
    def cli(cmd, input="", dir="", output="", precision=0, mapping=1, n=(), vector_height=8, seed=1,
            verify=False, real=False, json=False):
        """The reference CLI (inc/cli.hpp run_convert/spmm/sddmm/stats/bench):
        returns (exit code, stdout text, stderr text)."""
        code = {"convert": 0, "spmm": 1, "sddmm": 2, "stats": 3, "bench": 4}[cmd]
        ns = np.ascontiguousarray(list(n) or [0], np.uint64)
        o, e = C.c_void_p(), C.c_void_p()
        rc = ref().ref_cli(code, str(input).encode(), str(dir).encode(), str(output).encode(), precision, mapping,
                           _p(ns, _u64p), len(n), vector_height, seed, int(verify), int(real), int(json),
                           C.byref(o), C.byref(e))
        return rc, Ref._str(o.value), Ref._str(e.value)

    @staticmethod
    def parse_matrix_market(text):
        """Csr, or raises ValueError(ParseError message)."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        r = ref()
        rows, cols = C.c_uint64(), C.c_uint64()
        rp, ci, v, err = _u32p(), _u32p(), _f32p(), C.c_void_p()
        nnz = r.ref_parse_matrix_market(b, len(b), C.byref(rows), C.byref(cols), C.byref(rp), C.byref(ci),
                                        C.byref(v), C.byref(err))
        if nnz < 0:
            raise ValueError(Ref._str(err.value))
        return Csr(rows.value, cols.value, _take(r, rp, rows.value + 1, np.uint32), _take(r, ci, nnz, np.uint32),
                   _take(r, v, nnz, np.float32))

    @staticmethod
    def read_mebcrs(path):
        r = ref()
        rows, cols, prec = C.c_uint64(), C.c_uint64(), C.c_int()
        rp, ci, v, err = _u32p(), _u32p(), _f32p(), C.c_void_p()
        nv = r.ref_read_mebcrs(str(path).encode(), C.byref(rows), C.byref(cols), C.byref(prec), C.byref(rp),
                               C.byref(ci), C.byref(v), C.byref(err))
        if nv < 0:
            raise ValueError(Ref._str(err.value))
        W = (rows.value + 7) // 8
        return MeBcrs(rows.value, cols.value, prec.value, _take(r, rp, W + 1, np.uint32), _take(r, ci, nv, np.uint32),
                      _take(r, v, 8 * nv, np.float32))

    @staticmethod
    def sddmm_output_offsets(lane, kind):
        return int(ref().ref_sddmm_output_offsets(lane, kind))

    @staticmethod
    def round_fp16(x):
        return ref().ref_round_fp16(x)

    @staticmethod
    def round_tf32(x):
        return ref().ref_round_tf32(x)


def spmm_csr_rows(m: Csr, B: np.ndarray, precision: int, rows=None) -> np.ndarray:
    """Reference SpMM result (inc/spmm.hpp:126-163) computed from the CSR
    (orc_spmm_csr_rows): all rows, or the rows listed in ``rows``."""
    B = np.ascontiguousarray(B, np.float32)
    N = B.shape[1]
    sel = None if rows is None else np.ascontiguousarray(rows, np.uint64)
    n = m.rows if sel is None else sel.size
    Cm = np.zeros((n, N), np.float32)
    lib().orc_spmm_csr_rows(C.c_uint64(m.rows), precision, _p(m.row_ptr, _u32p), _p(m.col_idx, _u32p),
                            _p(m.values, _f32p), _p(B, _f32p), C.c_uint64(B.shape[0]), C.c_uint64(N),
                            C.c_uint64(N), None if sel is None else _p(sel, _u64p), C.c_uint64(n),
                            _p(Cm, _f32p), C.c_uint64(N))
    return Cm


def sddmm_csr_rows(m: Csr, precision: int, rp: np.ndarray, ci: np.ndarray, A: np.ndarray, Bt: np.ndarray,
                   rows=None):
    """Reference SDDMM values (inc/sddmm.hpp:102-132) of the CSR entries of
    ``rows`` (all rows if None), in CSR order, with each entry's slot in the
    ME-BCRS value array of (rp, ci) (orc_sddmm_csr_rows).  Returns
    (dot[f32], pos[u64]); pos = 2^64-1 marks an entry missing from (rp, ci)."""
    A = np.ascontiguousarray(A, np.float32)
    Bt = np.ascontiguousarray(Bt, np.float32)
    # rp = ci = None: dot products only, no ME-BCRS positions (pos stays 0)
    rp = None if rp is None else np.ascontiguousarray(rp, np.uint32)
    ci = None if ci is None else np.ascontiguousarray(ci, np.uint32)
    sel = np.arange(m.rows, dtype=np.uint64) if rows is None else np.ascontiguousarray(rows, np.uint64)
    lens = (m.row_ptr[sel.astype(np.int64) + 1].astype(np.uint64) - m.row_ptr[sel.astype(np.int64)].astype(np.uint64))
    eoff = np.zeros(sel.size + 1, np.uint64)
    np.cumsum(lens, out=eoff[1:])
    dot = np.zeros(max(int(eoff[-1]), 1), np.float32)
    pos = np.zeros(max(int(eoff[-1]), 1), np.uint64)
    lib().orc_sddmm_csr_rows(C.c_uint64(m.rows), precision, K_OF[precision], _p(m.row_ptr, _u32p),
                             _p(m.col_idx, _u32p), _p(m.values, _f32p), None if rp is None else _p(rp, _u32p),
                             None if ci is None else _p(ci, _u32p), _p(A, _f32p),
                             C.c_uint64(A.shape[1]), _p(Bt, _f32p), C.c_uint64(Bt.shape[1]), C.c_uint64(A.shape[1]),
                             _p(sel, _u64p), C.c_uint64(sel.size), _p(eoff, _u64p), _p(dot, _f32p), _p(pos, _u64p))
    n = int(eoff[-1])
    return dot[:n], pos[:n]
