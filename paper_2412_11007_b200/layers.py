"""GNN layers on the B200 FlashSparse kernels -- the callers that BASELINE.json
configs[3] and configs[4] name ("end-to-end GNN"):

* ``GCNLayer``: H' = Â (H W) with Â = D^-1/2 (A + I) D^-1/2 (Kipf & Welling).
  The dense transform H W is a plain library GEMM (cuBLAS through torch);
  the aggregation Â · (HW) is tcs_spmm over the ME-BCRS encoding of Â.
* ``AGNNLayer``: H' = softmax_row(beta * cos(h_i, h_j) on the edges) · H.
  FP16 with F = 32 or 64: tcs_agnn_attend, one kernel (scores, online
  softmax and aggregation from a single gather of each neighbour row).
  Otherwise cos via tcs_sddmm over the row-normalised features, the row
  softmax and the aggregation via tcs_agnn_aggregate (FP16) or
  tcs_sddmm_row_softmax + tcs_spmm (TF32) -- no re-encoding between stages
  (the pipeline closure of ref tests/test_kernels.cpp:313-327).

Inputs are torch CUDA tensors; the graph is given once as CSR and encoded
once on the GPU.
"""
from __future__ import annotations

import torch

from . import _abi
from . import tcsparse as T


def normalized_adjacency(rows: int, row_ptr: torch.Tensor, col_idx: torch.Tensor, add_self_loops: bool = True):
    """CSR of D^-1/2 (A + I) D^-1/2 (values f32) from a pattern CSR (int32)."""
    dev = row_ptr.device
    rp = row_ptr.to(torch.int64)
    ci = col_idx.to(torch.int64)
    r = torch.repeat_interleave(torch.arange(rows, device=dev), rp[1:] - rp[:-1])
    if add_self_loops:
        keys = torch.unique(torch.cat([r * rows + ci, torch.arange(rows, device=dev) * (rows + 1)]))
        r, ci = keys // rows, keys % rows
    deg = torch.bincount(r, minlength=rows).to(torch.float32)
    dinv = deg.clamp(min=1).rsqrt()
    vals = dinv[r] * dinv[ci]
    new_rp = torch.zeros(rows + 1, dtype=torch.int64, device=dev)
    new_rp[1:] = torch.cumsum(torch.bincount(r, minlength=rows), 0)
    return new_rp.to(torch.int32), ci.to(torch.int32), vals


class GCNLayer:
    def __init__(self, rows: int, row_ptr: torch.Tensor, col_idx: torch.Tensor, weight: torch.Tensor,
                 precision: T.Precision = T.Precision.fp16):
        rp, ci, v = normalized_adjacency(rows, row_ptr, col_idx)
        self.rows = rows
        self.adj = T.encode_mebcrs(T.CsrMatrix(rows, rows, rp, ci, v), precision)
        self.weight = weight
        self.cfg = T.KernelConfig(precision)
        self.dtype = torch.float16 if precision == T.Precision.fp16 else torch.float32

    def __call__(self, H: torch.Tensor) -> torch.Tensor:
        HW = (H.to(self.weight.dtype) @ self.weight).to(self.dtype)  # cuBLAS GEMM
        return T.spmm(self.adj, HW, self.cfg).output


class AGNNLayer:
    def __init__(self, rows: int, row_ptr: torch.Tensor, col_idx: torch.Tensor, beta: float = 1.0,
                 precision: T.Precision = T.Precision.fp16):
        ones = torch.ones(col_idx.numel(), dtype=torch.float32, device=col_idx.device)
        self.rows = rows
        self.mask = T.encode_mebcrs(T.CsrMatrix(rows, rows, row_ptr, col_idx, ones), precision)
        self.beta = float(beta)
        self.cfg = T.KernelConfig(precision)
        # the adjacency mask never changes: its sampling rule is read from
        # cached liveness bytes (TCS_CFG_STATIC_MASK)
        self.mask_cfg = T.KernelConfig(precision, static_mask=True)
        self.precision = precision
        self.dtype = torch.float16 if precision == T.Precision.fp16 else torch.float32

    def attention(self, H: torch.Tensor, fused: bool = True, Hn: torch.Tensor | None = None) -> T.MeBcrsMatrix:
        """P = row_softmax(beta * cos(h_i, h_j)) over the edges.  fused: one
        SDDMM kernel writes the scores with -inf at non-edges, then the
        softmax passes need no mask (tcs_sddmm_row_softmax; FP16 keeps the
        scores in f16, normalised in place); else SDDMM ->
        tcs_mebcrs_row_softmax."""
        if Hn is None:
            Hn, _ = T.rows_normalize(H.float().contiguous(), self.dtype, copy=False)
        ops = T.SddmmOperands(self.mask, Hn, Hn)
        pdt = _abi.TCS_DTYPE_F16 if self.precision == T.Precision.fp16 else _abi.TCS_DTYPE_F32
        if fused:
            return T.sddmm_row_softmax(ops, self.beta, self.mask_cfg, score_dtype=pdt, out_dtype=pdt)
        scores = T.sddmm(ops, self.mask_cfg).output  # cos(h_i, h_j) at the edges
        return T.row_softmax(scores, self.mask, self.beta, pdt)

    def __call__(self, H: torch.Tensor, one_pass: bool = True) -> torch.Tensor:
        if one_pass and self.precision == T.Precision.fp16 and H.shape[1] in (32, 64):
            # tcs_agnn_attend: scores, online softmax and aggregation in one
            # kernel, each neighbour row gathered once
            _, Hc = T.rows_normalize(H.float().contiguous(), torch.float16, normalized=False)
            return T.agnn_attend(self.mask, Hc, self.beta, self.mask_cfg)
        # one pass over H: the normalised rows (SDDMM operand) and H itself
        # in the kernels' dtype (SpMM operand)
        Hn, Hc = T.rows_normalize(H.float().contiguous(), self.dtype)
        if self.precision == T.Precision.fp16:
            # SDDMM -> softmax -> SpMM without materialising P (tcs_agnn_aggregate)
            return T.agnn_aggregate(self.mask, Hn, Hc, self.beta, self.mask_cfg)
        P = self.attention(H, Hn=Hn)
        return T.spmm(P, Hc, self.cfg).output
