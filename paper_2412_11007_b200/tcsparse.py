"""Python front end of the B200 FlashSparse path, mirroring the reference's
C++ API (``tcsparse::encode_mebcrs / spmm / sddmm``, ref
proj/include/tcsparse) on torch CUDA tensors.

Every call goes through the C-ABI (include/tcs/tcs.h) into
libtcsparse_b200.so; torch supplies device memory and the current stream
only.  Errors are raised as the reference's exception types
(ref errors.hpp): ArgumentError, ShapeError, FormatError; CUDA failures as
CudaError.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import torch

from . import _abi


class TcsError(RuntimeError):
    pass


class ArgumentError(TcsError, ValueError):
    """ref errors.hpp:36 (std::invalid_argument)."""


class ShapeError(TcsError):
    """ref errors.hpp:30."""


class FormatError(TcsError):
    """ref errors.hpp:24."""


class ParseError(TcsError):
    """ref errors.hpp:11-22 (malformed MatrixMarket; message carries "line N: ")."""


class FileError(TcsError, OSError):
    """A container / output file cannot be opened or written."""


class CudaError(TcsError):
    pass


_ERR = {_abi.TCS_ERR_ARGUMENT: ArgumentError, _abi.TCS_ERR_SHAPE: ShapeError, _abi.TCS_ERR_FORMAT: FormatError,
        _abi.TCS_ERR_CUDA: CudaError, _abi.TCS_ERR_OOM: CudaError, _abi.TCS_ERR_NCCL: CudaError,
        _abi.TCS_ERR_PARSE: ParseError, _abi.TCS_ERR_IO: FileError}


def _check(rc: int):
    if rc != _abi.TCS_OK:
        msg = _abi.load().tcs_last_error().decode()
        raise _ERR.get(rc, TcsError)(msg)


class Precision(enum.IntEnum):
    """ref precision.hpp:13."""
    fp16 = 0
    tf32 = 1


class ThreadMapping(enum.IntEnum):
    """ref access_pattern.hpp:15."""
    direct = 0
    coalesced = 1


@dataclass
class KernelConfig:
    """ref spmm.hpp:17-21."""
    precision: Precision = Precision.fp16
    vector_height: int = 8
    mapping: ThreadMapping = ThreadMapping.coalesced
    path: str = "auto"  # SpMM instruction path: auto | mma_sync | tcgen05 (tcs.h TCS_CFG_PATH_*)
    static_mask: bool = False  # SDDMM: mask values fixed across calls -> cached liveness bytes (TCS_CFG_STATIC_MASK)
    tf32_f32_gather: bool = False  # TF32 SpMM ablation: gather f32 B, no 2.5-byte repack (TCS_CFG_TF32_F32_GATHER)

    def _c(self):
        flags = ({"auto": 0, "mma_sync": 1, "tcgen05": 2}[self.path] | (8 if self.static_mask else 0)
                 | (0x10 if self.tf32_f32_gather else 0))
        return _abi.tcs_kernel_config(int(self.precision), int(self.vector_height), int(self.mapping), flags)


@dataclass
class KernelCounters:
    """ref spmm.hpp:23-28."""
    mma_invocations: int = 0
    transactions: int = 0
    transaction_bytes: int = 0
    useful_bytes: int = 0

    @staticmethod
    def _from(c):
        return KernelCounters(c.mma_invocations, c.transactions, c.transaction_bytes, c.useful_bytes)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, name: str) -> torch.Tensor:
    """Device operands go to the kernels as raw pointers on the current
    device's stream: anything else would fault (host memory) or run against
    another device's memory pool."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ArgumentError(f"{name} must be a CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        raise ArgumentError(f"{name} is on {t.device}, the current device is cuda:{torch.cuda.current_device()}")
    return t


_TORCH_OF_TAG = {_abi.TCS_DTYPE_F16: torch.float16, _abi.TCS_DTYPE_F32: torch.float32}


def _out_rows(out: torch.Tensor, rows: int, n: int, name: str = "out") -> torch.Tensor:
    """Caller-supplied f32 output [>= rows, >= n] with unit column stride."""
    _dev(out, name)
    if out.dtype != torch.float32 or out.dim() != 2 or out.stride(1) != 1 or out.shape[0] < rows \
            or out.shape[1] < n:
        raise ArgumentError(f"{name} must be a float32 [>= {rows}, >= {n}] tensor with unit column stride")
    return out


def _out_values(v: torch.Tensor, nv: int, tag: int, name: str = "out_values") -> torch.Tensor:
    """Caller-supplied ME-BCRS value array: 8 * nv contiguous elements of the
    output dtype (the kernels write 8 * nv * width bytes)."""
    _dev(v, name)
    if v.dtype != _TORCH_OF_TAG[int(tag)]:
        raise ArgumentError(f"{name} must be {_TORCH_OF_TAG[int(tag)]} for this output dtype, not {v.dtype}")
    if v.numel() < 8 * nv or not v.is_contiguous():
        raise ArgumentError(f"{name} too small or not contiguous (needs {8 * nv} elements)")
    return v


def _u32(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == torch.uint32:
        return t.contiguous()
    return t.to(torch.int32).contiguous()


@dataclass
class CsrMatrix:
    """ref matrix.hpp:20-49 on the device (u32 indices as int32/uint32 tensors)."""
    rows: int
    cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    values: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    def _c(self):
        for name in ("row_ptr", "col_idx", "values"):
            _dev(getattr(self, name), name)
        self.row_ptr, self.col_idx = _u32(self.row_ptr), _u32(self.col_idx)
        self.values = self.values.to(torch.float32).contiguous()
        return _abi.tcs_csr(self.rows, self.cols, self.nnz, self.row_ptr.data_ptr(), self.col_idx.data_ptr(),
                            self.values.data_ptr())


class MeBcrsMatrix:
    """Device ME-BCRS (ref mebcrs.hpp:23-78) owned by the C library."""

    def __init__(self, handle: _abi.tcs_mebcrs, keepalive=()):
        self._h = handle
        self._keep = list(keepalive)

    # reference accessors
    rows = property(lambda self: self._h.rows)
    cols = property(lambda self: self._h.cols)
    k = property(lambda self: self._h.k)
    vector_height = property(lambda self: self._h.vector_height)
    precision = property(lambda self: Precision(self._h.precision))
    num_windows = property(lambda self: self._h.num_windows)
    num_vectors = property(lambda self: self._h.num_vectors)
    num_blocks = property(lambda self: self._h.num_blocks)
    max_window_vectors = property(lambda self: self._h.max_window_vectors)
    value_dtype = property(lambda self: self._h.value_dtype)

    def to_host(self):
        """(row_pointers, column_indices, values[f32]) as numpy arrays."""
        import numpy as np

        rp = np.empty(self.num_windows + 1, np.uint32)
        ci = np.empty(max(1, self.num_vectors), np.uint32)
        v = np.empty(max(1, self.vector_height * self.num_vectors), np.float32)
        _check(_abi.load().tcs_mebcrs_download(C.byref(self._h), rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                               _stream()))
        return rp, ci[: self.num_vectors], v[: self.vector_height * self.num_vectors]

    def validate(self):
        _check(_abi.load().tcs_mebcrs_validate(C.byref(self._h), _stream()))

    def decode(self):
        """ref decode_mebcrs (mebcrs.hpp:116-138) on the GPU: the stored
        values != 0 as CSR, returned as host numpy arrays (row_ptr, col_idx,
        values) -- the reference's test-side round trip."""
        return _decode_to_host(lambda h: _abi.load().tcs_mebcrs_decode(C.byref(self._h), C.byref(h), _stream()))

    def free(self):
        if getattr(self, "_h", None) is not None and (self._h.flags or self._h.plan):
            _abi.load().tcs_mebcrs_free(C.byref(self._h), _stream())
        self._keep = []

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @staticmethod
    def from_host(rows, cols, precision, row_pointers, column_indices, values) -> "MeBcrsMatrix":
        import numpy as np

        rp = np.ascontiguousarray(row_pointers, np.uint32)
        ci = np.ascontiguousarray(column_indices, np.uint32)
        v = np.ascontiguousarray(values, np.float32)
        h = _abi.tcs_mebcrs()
        _check(_abi.load().tcs_mebcrs_upload(rows, cols, int(precision), rp.ctypes.data, ci.ctypes.data,
                                             v.ctypes.data, C.byref(h), _stream()))
        return MeBcrsMatrix(h)


def _decode_to_host(run):
    """Runs a tcs_*_decode call into a device CSR and returns it as host
    numpy arrays (row_ptr, col_idx, values); the device CSR is freed."""
    import numpy as np

    lib = _abi.load()
    h = _abi.tcs_csr()
    _check(run(h))
    try:
        rows, nnz = int(h.rows), int(h.nnz)
        rp = np.empty(rows + 1, np.uint32)
        ci = np.empty(max(1, nnz), np.uint32)
        v = np.empty(max(1, nnz), np.float32)
        _check(lib.tcs_csr_download(C.byref(h), rp.ctypes.data, ci.ctypes.data, v.ctypes.data, _stream()))
    finally:
        lib.tcs_csr_free(C.byref(h), _stream())
    return rp, ci[:nnz], v[:nnz]


def encode_mebcrs(csr: CsrMatrix, precision: Precision, value_dtype: int | None = None,
                  vector_height: int = 8) -> MeBcrsMatrix:
    """ref mebcrs.hpp:80.  value_dtype: TCS_DTYPE_F16 (default for fp16) or TCS_DTYPE_F32.
    vector_height 16 builds the 16-row-window layout of the 16x1 baseline
    (ref partition.hpp:40-66 with vector_height 16; for spmm_baseline16)."""
    if value_dtype is None:
        value_dtype = _abi.TCS_DTYPE_F16 if int(precision) == 0 else _abi.TCS_DTYPE_F32
    c = csr._c()
    h = _abi.tcs_mebcrs()
    lib = _abi.load()
    if vector_height == 8:
        _check(lib.tcs_mebcrs_encode(C.byref(c), int(precision), int(value_dtype), C.byref(h), _stream()))
    else:
        _check(lib.tcs_mebcrs_encode_v(C.byref(c), int(precision), int(value_dtype), int(vector_height), C.byref(h),
                                       _stream()))
    return MeBcrsMatrix(h)


@dataclass
class SpmmResult:
    output: torch.Tensor
    counters: KernelCounters = field(default_factory=KernelCounters)


def _dtype_tag(t: torch.Tensor) -> int:
    if t.dtype == torch.float16:
        return _abi.TCS_DTYPE_F16
    if t.dtype == torch.float32:
        return _abi.TCS_DTYPE_F32
    raise ArgumentError(f"unsupported dense dtype {t.dtype}")


def spmm(sparse: MeBcrsMatrix, dense: torch.Tensor, cfg: KernelConfig = KernelConfig(),
         out: torch.Tensor | None = None) -> SpmmResult:
    """ref spmm.hpp:173.  dense: [K, N] f16 (FP16) or f32 CUDA tensor, row-major
    (any row stride).  Returns C [M, N] f32.  An SrBcrsMatrix runs the
    reference's spmm(SrBcrsMatrix) overload (spmm.hpp:181)."""
    if isinstance(sparse, SrBcrsMatrix):
        return spmm_srbcrs(sparse, dense, cfg, out)
    _dev(dense, "dense")
    if dense.dim() != 2 or dense.stride(1) != 1:
        dense = dense.contiguous()
    m, n = sparse.rows, dense.shape[1]
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=dense.device)
    _out_rows(out, m, n)
    cnt = _abi.tcs_counters()
    _check(_abi.load().tcs_spmm(C.byref(sparse._h), dense.data_ptr(), _dtype_tag(dense), dense.stride(0),
                                dense.shape[0], n, out.data_ptr(), out.stride(0), C.byref(cfg._c()), C.byref(cnt),
                                _stream()))
    return SpmmResult(out, KernelCounters._from(cnt))


def spmm_baseline16(sparse: MeBcrsMatrix, dense: torch.Tensor, cfg: KernelConfig | None = None,
                    out: torch.Tensor | None = None) -> SpmmResult:
    """ref spmm.hpp:187-257 (the non-swapped 16x1 ablation).  ``sparse`` is a
    vector_height-16 encoding (encode_mebcrs(..., vector_height=16)); cfg
    defaults to the matrix precision with vector_height 16."""
    if cfg is None:
        cfg = KernelConfig(sparse.precision, vector_height=16)
    _dev(dense, "dense")
    if dense.dim() != 2 or dense.stride(1) != 1:
        dense = dense.contiguous()
    m, n = sparse.rows, dense.shape[1]
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=dense.device)
    _out_rows(out, m, n)
    cnt = _abi.tcs_counters()
    _check(_abi.load().tcs_spmm_baseline16(C.byref(sparse._h), dense.data_ptr(), _dtype_tag(dense), dense.stride(0),
                                           dense.shape[0], n, out.data_ptr(), out.stride(0), C.byref(cfg._c()),
                                           C.byref(cnt), _stream()))
    return SpmmResult(out, KernelCounters._from(cnt))


class SrBcrsMatrix:
    """Device SR-BCRS (ref srbcrs.hpp:11-38), the zero-vector padded baseline
    format, owned by the C library."""

    def __init__(self, handle: _abi.tcs_srbcrs):
        self._h = handle

    rows = property(lambda self: self._h.rows)
    cols = property(lambda self: self._h.cols)
    k = property(lambda self: self._h.k)
    vector_height = property(lambda self: self._h.vector_height)
    precision = property(lambda self: Precision(self._h.precision))
    num_windows = property(lambda self: self._h.num_windows)
    num_padded = property(lambda self: self._h.num_padded)

    def to_host(self):
        """(row_pointer_pairs, column_indices, values[f32]) as numpy arrays."""
        import numpy as np

        rpp = np.empty(max(1, 2 * self.num_windows), np.uint32)
        ci = np.empty(max(1, self.num_padded), np.uint32)
        v = np.empty(max(1, 8 * self.num_padded), np.float32)
        _check(_abi.load().tcs_srbcrs_download(C.byref(self._h), rpp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                               _stream()))
        return rpp[: 2 * self.num_windows], ci[: self.num_padded], v[: 8 * self.num_padded]

    def decode(self):
        """ref decode_srbcrs (srbcrs.hpp:74-90) on the GPU: host numpy
        (row_ptr, col_idx, values) of the stored values != 0."""
        return _decode_to_host(lambda h: _abi.load().tcs_srbcrs_decode(C.byref(self._h), C.byref(h), _stream()))

    def free(self):
        if getattr(self, "_h", None) is not None and self._h.impl:
            _abi.load().tcs_srbcrs_free(C.byref(self._h), _stream())

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @staticmethod
    def from_host(rows, cols, precision, row_pointer_pairs, column_indices, values) -> "SrBcrsMatrix":
        import numpy as np

        rpp = np.ascontiguousarray(row_pointer_pairs, np.uint32)
        ci = np.ascontiguousarray(column_indices, np.uint32)
        v = np.ascontiguousarray(values, np.float32)
        h = _abi.tcs_srbcrs()
        _check(_abi.load().tcs_srbcrs_upload(rows, cols, int(precision), rpp.ctypes.data, ci.ctypes.data,
                                             v.ctypes.data, C.byref(h), _stream()))
        return SrBcrsMatrix(h)


def encode_srbcrs(csr: CsrMatrix | MeBcrsMatrix, precision: Precision | None = None,
                  value_dtype: int | None = None) -> SrBcrsMatrix:
    """ref encode_srbcrs (srbcrs.hpp:40-72) on the GPU, from a CSR (encoded
    to ME-BCRS first) or directly from a device ME-BCRS."""
    h = _abi.tcs_srbcrs()
    lib = _abi.load()
    if isinstance(csr, MeBcrsMatrix):
        _check(lib.tcs_srbcrs_from_mebcrs(C.byref(csr._h), C.byref(h), _stream()))
    else:
        if value_dtype is None:
            value_dtype = _abi.TCS_DTYPE_F16 if int(precision) == 0 else _abi.TCS_DTYPE_F32
        c = csr._c()
        _check(lib.tcs_srbcrs_encode(C.byref(c), int(precision), int(value_dtype), C.byref(h), _stream()))
    return SrBcrsMatrix(h)


def spmm_srbcrs(sparse: SrBcrsMatrix, dense: torch.Tensor, cfg: KernelConfig = KernelConfig(),
                out: torch.Tensor | None = None) -> SpmmResult:
    """ref spmm(const SrBcrsMatrix&, ...) (spmm.hpp:181-185): same kernel and
    result as spmm() on the compact format."""
    _dev(dense, "dense")
    if dense.dim() != 2 or dense.stride(1) != 1:
        dense = dense.contiguous()
    m, n = sparse.rows, dense.shape[1]
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=dense.device)
    _out_rows(out, m, n)
    cnt = _abi.tcs_counters()
    _check(_abi.load().tcs_spmm_srbcrs(C.byref(sparse._h), dense.data_ptr(), _dtype_tag(dense), dense.stride(0),
                                       dense.shape[0], n, out.data_ptr(), out.stride(0), C.byref(cfg._c()),
                                       C.byref(cnt), _stream()))
    return SpmmResult(out, KernelCounters._from(cnt))


@dataclass
class SddmmOperands:
    """ref sddmm.hpp:16-20: mask (ME-BCRS), a [M, F], b_t [N, F]."""
    mask: MeBcrsMatrix
    a: torch.Tensor
    b_t: torch.Tensor


@dataclass
class SddmmResult:
    output: MeBcrsMatrix
    counters: KernelCounters = field(default_factory=KernelCounters)


def sddmm(ops: SddmmOperands, cfg: KernelConfig = KernelConfig(), out_dtype: int = _abi.TCS_DTYPE_F32,
          out_values: torch.Tensor | None = None) -> SddmmResult:
    """ref sddmm.hpp:84.  The output shares the mask's structure (kept alive).
    ``out_values`` (optional): caller-owned device tensor of 8 * nv elements
    of out_dtype receiving the values (else the library allocates them)."""
    a = _dev(ops.a, "a") if ops.a.stride(-1) == 1 else _dev(ops.a, "a").contiguous()
    b = _dev(ops.b_t, "b_t") if ops.b_t.stride(-1) == 1 else _dev(ops.b_t, "b_t").contiguous()
    h = _abi.tcs_mebcrs()
    keep = [ops.mask]
    if out_values is not None:
        h.values = _out_values(out_values, ops.mask.num_vectors, out_dtype).data_ptr()
        keep.append(out_values)
    cnt = _abi.tcs_counters()
    _check(_abi.load().tcs_sddmm(C.byref(ops.mask._h), a.data_ptr(), _dtype_tag(a), a.stride(0), a.shape[0],
                                 a.shape[1], b.data_ptr(), _dtype_tag(b), b.stride(0), b.shape[0], b.shape[1],
                                 C.byref(h), int(out_dtype), C.byref(cfg._c()), C.byref(cnt), _stream()))
    return SddmmResult(MeBcrsMatrix(h, keepalive=keep), KernelCounters._from(cnt))


def row_softmax(scores: MeBcrsMatrix, mask: MeBcrsMatrix, scale: float = 1.0,
                out_dtype: int = _abi.TCS_DTYPE_F16, out_values: torch.Tensor | None = None) -> MeBcrsMatrix:
    """Row-wise softmax over the pattern (tcs_mebcrs_row_softmax): the AGNN
    attention normalisation between SDDMM and SpMM."""
    h = _abi.tcs_mebcrs()
    keep = [scores, mask]
    if out_values is not None:
        h.values = _out_values(out_values, scores.num_vectors, out_dtype).data_ptr()
        keep.append(out_values)
    _check(_abi.load().tcs_mebcrs_row_softmax(C.byref(scores._h), C.byref(mask._h), float(scale), C.byref(h),
                                              int(out_dtype), _stream()))
    return MeBcrsMatrix(h, keepalive=keep)


def sddmm_row_softmax(ops: SddmmOperands, scale: float = 1.0, cfg: KernelConfig = KernelConfig(),
                      score_dtype: int = _abi.TCS_DTYPE_F32, out_dtype: int = _abi.TCS_DTYPE_F16,
                      out_values: torch.Tensor | None = None) -> MeBcrsMatrix:
    """Fused ``row_softmax(sddmm(ops).output, ops.mask, scale)``
    (tcs_sddmm_row_softmax): the scores (stored as score_dtype) carry the
    per-row softmax partials out of the SDDMM kernel and are normalised in
    one pass."""
    a = _dev(ops.a, "a") if ops.a.stride(-1) == 1 else _dev(ops.a, "a").contiguous()
    b = _dev(ops.b_t, "b_t") if ops.b_t.stride(-1) == 1 else _dev(ops.b_t, "b_t").contiguous()
    h = _abi.tcs_mebcrs()
    keep = [ops.mask]
    if out_values is not None:
        h.values = _out_values(out_values, ops.mask.num_vectors, out_dtype).data_ptr()
        keep.append(out_values)
    _check(_abi.load().tcs_sddmm_row_softmax(C.byref(ops.mask._h), a.data_ptr(), _dtype_tag(a), a.stride(0),
                                             a.shape[0], a.shape[1], b.data_ptr(), _dtype_tag(b), b.stride(0),
                                             b.shape[0], b.shape[1], float(scale), int(score_dtype), C.byref(h),
                                             int(out_dtype), C.byref(cfg._c()), _stream()))
    return MeBcrsMatrix(h, keepalive=keep)


def agnn_aggregate(mask: MeBcrsMatrix, hn: torch.Tensor, hc: torch.Tensor, scale: float = 1.0,
                   cfg: KernelConfig | None = None, out: torch.Tensor | None = None, row0: int = 0) -> torch.Tensor:
    """C = row_softmax(scale * (hn[row0 + i] . hn[j]) at the mask's live
    slots) @ hc (tcs_agnn_aggregate): == spmm(sddmm_row_softmax(..., binary16
    scores and P), hc) bit for bit, with the softmax applied inside the SpMM.
    hn, hc hold every node; the mask holds the adjacency rows
    [row0, row0 + mask.rows) (a row shard, or the whole graph)."""
    if cfg is None:
        cfg = KernelConfig(mask.precision)
    hn = _dev(hn, "hn") if hn.stride(-1) == 1 else _dev(hn, "hn").contiguous()
    hc = _dev(hc, "hc") if hc.stride(-1) == 1 else _dev(hc, "hc").contiguous()
    rows, n = mask.rows, hc.shape[1]
    # the kernels read feature rows of every node (mask.cols of them) and
    # the score rows [row0, row0 + rows)
    if hn.dim() != 2 or hc.dim() != 2 or hn.shape[0] < max(mask.cols, row0 + rows) or hc.shape[0] < mask.cols:
        raise ShapeError(f"hn / hc must hold every node's row ({mask.cols}; row0 + rows = {row0 + rows})")
    if out is None:
        out = torch.empty((rows, n), dtype=torch.float32, device=hc.device)
    _out_rows(out, rows, n)
    _check(_abi.load().tcs_agnn_aggregate(C.byref(mask._h), hn.data_ptr(), _dtype_tag(hn), hn.stride(0), int(row0),
                                          rows, hn.shape[1], float(scale), hc.data_ptr(), _dtype_tag(hc),
                                          hc.stride(0), n, out.data_ptr(), out.stride(0), C.byref(cfg._c()),
                                          _stream()))
    return out


def agnn_attend(mask: MeBcrsMatrix, h: torch.Tensor, scale: float = 1.0, cfg: KernelConfig | None = None,
                out: torch.Tensor | None = None, row0: int = 0, eps: float = 1e-12) -> torch.Tensor:
    """C[i] = sum_j softmax_j(scale * cos(h[row0 + i], h[j])) h[j] over the
    mask's live slots, fused in one pass (tcs_agnn_attend): h is the f16
    feature matrix of every node (F = 32 or 64), gathered once per stored
    vector for both the scores and the aggregation."""
    if cfg is None:
        cfg = KernelConfig(mask.precision)
    if h.dtype != torch.float16 or h.dim() != 2:
        raise ArgumentError("h must be a 2-D float16 tensor")
    h = _dev(h, "h") if h.stride(-1) == 1 else _dev(h, "h").contiguous()
    rows, f = mask.rows, h.shape[1]
    if h.shape[0] < max(mask.cols, row0 + rows):  # every node's row (agnn.cu reads mask.cols rows)
        raise ShapeError(f"h must hold every node's row ({mask.cols}; row0 + rows = {row0 + rows})")
    if out is None:
        out = torch.empty((rows, f), dtype=torch.float32, device=h.device)
    _out_rows(out, rows, f)
    _check(_abi.load().tcs_agnn_attend(C.byref(mask._h), h.data_ptr(), _abi.TCS_DTYPE_F16, h.stride(0), int(row0),
                                       f, float(scale), float(eps), out.data_ptr(), out.stride(0),
                                       C.byref(cfg._c()), _stream()))
    return out


def rows_normalize(h: torch.Tensor, dtype: torch.dtype = torch.float16, eps: float = 1e-12,
                   normalized: bool = True, copy: bool = True):
    """(h / max(||h_i||, eps), h) in `dtype` from one pass over the f32 rows
    (tcs_rows_normalize; the AGNN layer's SDDMM / SpMM operands)."""
    if h.dtype != torch.float32 or h.dim() != 2 or h.stride(-1) != 1:
        raise ArgumentError("h must be a 2-D f32 tensor with unit column stride")
    _dev(h, "h")
    rows, f = h.shape
    hn = torch.empty(rows, f, dtype=dtype, device=h.device) if normalized else None
    hc = torch.empty(rows, f, dtype=dtype, device=h.device) if copy else None
    tag = _abi.TCS_DTYPE_F16 if dtype == torch.float16 else _abi.TCS_DTYPE_F32
    _check(_abi.load().tcs_rows_normalize(h.data_ptr(), rows, f, h.stride(0),
                                          hn.data_ptr() if hn is not None else None,
                                          hc.data_ptr() if hc is not None else None, f, tag, float(eps), _stream()))
    return hn, hc


def round_values(x: torch.Tensor, precision: Precision) -> torch.Tensor:
    """Device operand rounding used by the kernels (diagnostics)."""
    x = _dev(x, "x").to(torch.float32).contiguous()
    out = torch.empty_like(x)
    _check(_abi.load().tcs_round_values(int(precision), x.data_ptr(), out.data_ptr(), x.numel(), _stream()))
    return out


# ------------------------------------------------------ ingest / containers
def _host_csr_to_device(h: _abi.tcs_csr) -> CsrMatrix:
    import numpy as np

    try:
        rows, cols, nnz = int(h.rows), int(h.cols), int(h.nnz)
        rp = np.ctypeslib.as_array(C.cast(h.row_ptr, C.POINTER(C.c_uint32)), shape=(rows + 1,)).copy()
        ci = np.ctypeslib.as_array(C.cast(h.col_idx, C.POINTER(C.c_uint32)), shape=(max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(C.cast(h.values, C.POINTER(C.c_float)), shape=(max(nnz, 1),))[:nnz].copy()
    finally:
        _abi.load().tcs_csr_free_host(C.byref(h))
    dev = torch.device("cuda", torch.cuda.current_device())
    return CsrMatrix(rows, cols, torch.from_numpy(rp.view(np.int32)).to(dev), torch.from_numpy(ci.view(np.int32)).to(dev),
                     torch.from_numpy(v).to(dev))


def parse_matrix_market(text: str | bytes) -> CsrMatrix:
    """ref parse_matrix_market (matrix_market.hpp:28-94); CSR assembled on the GPU."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = _abi.tcs_csr()
    _check(_abi.load().tcs_matrix_market_parse(b, len(b), C.byref(h), _stream()))
    return _host_csr_to_device(h)


def read_matrix_market(path: str) -> CsrMatrix:
    h = _abi.tcs_csr()
    _check(_abi.load().tcs_matrix_market_read(str(path).encode(), C.byref(h), _stream()))
    return _host_csr_to_device(h)


def write_matrix_market(path: str, csr: CsrMatrix) -> None:
    """ref write_matrix_market (matrix_market.hpp:97-104)."""
    import numpy as np

    rp = csr.row_ptr.cpu().numpy().astype(np.uint32)
    ci = csr.col_idx.cpu().numpy().astype(np.uint32)
    v = csr.values.cpu().numpy().astype(np.float32)
    h = _abi.tcs_csr(csr.rows, csr.cols, ci.size, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    _check(_abi.load().tcs_matrix_market_write(str(path).encode(), C.byref(h)))


def write_mebcrs(path: str, m: MeBcrsMatrix) -> None:
    """ref write_mebcrs (container_io.hpp:56-68), MEBC v1."""
    _check(_abi.load().tcs_mebcrs_write(str(path).encode(), C.byref(m._h), _stream()))


def read_mebcrs(path: str) -> MeBcrsMatrix:
    """ref read_mebcrs (container_io.hpp:70-91): validated, F32 values on the device."""
    h = _abi.tcs_mebcrs()
    _check(_abi.load().tcs_mebcrs_read(str(path).encode(), C.byref(h), _stream()))
    return MeBcrsMatrix(h)


def mebcrs_cost(m: MeBcrsMatrix, nnz: int, n_cols: int,
                mapping: ThreadMapping = ThreadMapping.coalesced) -> dict:
    """ref analysis.hpp:34-131 / footprint.hpp (tcs_mebcrs_cost): swap8 for a
    vector-height-8 matrix, the 16x1 baseline for a vector-height-16 one."""
    c = _abi.tcs_cost()
    _check(_abi.load().tcs_mebcrs_cost(C.byref(m._h), int(nnz), int(n_cols), int(mapping), C.byref(c), _stream()))
    return {name: int(getattr(c, name)) for name, _ in _abi.tcs_cost._fields_}


def launch_count() -> int:
    return int(_abi.load().tcs_launch_count())


def version() -> str:
    return _abi.load().tcs_version().decode()
