"""Row-window sharding of the FlashSparse path over the GPUs of one box
(one process per GPU, torch.distributed with NCCL; gloo works for the host
logic and is what the CPU tests use).

The unit of work is the 8-row window: windows own disjoint output rows
(ref SPEC.md:364), so SpMM/SDDMM shard with no data-path collective.

* ``shard_windows``: contiguous window ranges, cut at nnz quantiles (the
  north star's balance criterion) -- or at nv quantiles if the ME-BCRS row
  pointers are given (gather bytes scale with nv).
* ``local_rows``: the CSR rows of one shard (row_ptr rebased; global column
  indices kept, so every shard gathers from the full dense operand).
* ``broadcast_dense``: dense B from one rank to all (NCCL broadcast over
  NVLink/NVSwitch), done once per operand, outside the timed SpMM loop.
* ``gather_rows``: optional all-gather of the per-shard outputs when layers
  chain (GCN / AGNN): shards are padded to the largest one, all-gathered in
  one collective, and trimmed.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class Shard:
    rank: int
    world: int
    w0: int  # first window
    w1: int  # one past the last window
    r0: int  # first row
    r1: int  # one past the last row

    @property
    def rows(self) -> int:
        return self.r1 - self.r0


def shard_windows(row_ptr: torch.Tensor, rows: int, world: int, weights: str = "nnz",
                  mebcrs_row_pointers: torch.Tensor | None = None) -> list[int]:
    """Window cut points [0 = c_0 <= c_1 <= ... <= c_world = W] such that
    shard r = windows [c_r, c_{r+1}) carries ~1/world of the weight.
    weights = "nnz" uses CSR row_ptr at window starts; "nv" uses the
    ME-BCRS row pointers (stored 8x1 vectors per window)."""
    W = (rows + 7) // 8
    if weights == "nv":
        if mebcrs_row_pointers is None:
            raise ValueError("weights='nv' needs the ME-BCRS row pointers")
        prefix = mebcrs_row_pointers.to(torch.int64).cpu()
    else:
        idx = torch.clamp(torch.arange(W + 1, dtype=torch.int64) * 8, max=rows)
        prefix = row_ptr.to(torch.int64).cpu()[idx]
    total = int(prefix[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(torch.searchsorted(prefix, total * r // world)))
    cuts.append(W)
    for i in range(1, len(cuts)):  # monotone even for degenerate inputs
        cuts[i] = max(cuts[i], cuts[i - 1])
    return cuts


def shard_of(cuts: list[int], rank: int, rows: int) -> Shard:
    w0, w1 = cuts[rank], cuts[rank + 1]
    return Shard(rank, len(cuts) - 1, w0, w1, min(8 * w0, rows), min(8 * w1, rows))


def local_rows(row_ptr: torch.Tensor, col_idx: torch.Tensor, values: torch.Tensor, shard: Shard):
    """CSR of rows [r0, r1) with row_ptr rebased to 0."""
    b, e = int(row_ptr[shard.r0]), int(row_ptr[shard.r1])
    return (row_ptr[shard.r0:shard.r1 + 1] - b).contiguous(), col_idx[b:e].contiguous(), values[b:e].contiguous()


_DISTS: dict = {}


def tcs_dist(group=None):
    """The library's tcs_dist (include/tcs/tcs_dist.h) bound to torch's own
    NCCL communicator of `group` (ProcessGroupNCCL._comm_ptr), or None when
    the process group is not NCCL (gloo: the CPU tests).  Cached per group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_backend(group) != "nccl":
        return None
    key = id(group)
    if key not in _DISTS:
        import ctypes as C

        from . import _abi

        pg = group if group is not None else dist.distributed_c10d._get_default_group()
        ptr = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))._comm_ptr()
        d = _abi.tcs_dist()
        rc = _abi.load().tcs_dist_init(C.byref(d), C.c_void_p(ptr), 0)
        if rc != 0:
            raise RuntimeError(f"tcs_dist_init: {_abi.load().tcs_last_error().decode()}")
        _DISTS[key] = d
    return _DISTS[key]


def broadcast_dense(B: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast of the dense operand.  NCCL process groups: the
    library's tcs_dist_broadcast on torch's communicator (one NCCL broadcast
    over NVLink/NVSwitch, stream-ordered on the current stream); other
    backends: torch.distributed.broadcast."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return B
    d = tcs_dist(group) if B.is_cuda else None
    if d is None:
        dist.broadcast(B, src=src, group=group)
        return B
    import ctypes as C

    from . import _abi

    root = dist.get_group_rank(group, src) if group is not None else src
    lib = _abi.load()
    rc = lib.tcs_dist_broadcast(C.byref(d), C.c_void_p(B.data_ptr()), B.numel() * B.element_size(), root,
                                C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"tcs_dist_broadcast: {lib.tcs_last_error().decode()}")
    return B


def gather_rows(C_local: torch.Tensor, shard_rows: list[int], group=None) -> torch.Tensor:
    """All-gather row shards of different heights into the full matrix
    (every rank receives it).  shard_rows[r] = rows owned by rank r."""
    world = len(shard_rows)
    if world == 1:
        return C_local
    hmax = max(shard_rows)
    pad = torch.zeros((hmax,) + tuple(C_local.shape[1:]), dtype=C_local.dtype, device=C_local.device)
    pad[: C_local.shape[0]] = C_local
    out = torch.empty((world * hmax,) + tuple(C_local.shape[1:]), dtype=C_local.dtype, device=C_local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * hmax: r * hmax + shard_rows[r]] for r in range(world)], dim=0)


class ShardedSpmm:
    """SpMM of one graph over all ranks: each rank converts and multiplies
    its own window shard (tcs_mebcrs_encode + tcs_spmm on its GPU)."""

    def __init__(self, rows, cols, row_ptr, col_idx, values, precision, group=None):
        from . import tcsparse as T

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cuts = shard_windows(row_ptr, rows, self.world)
        self.shard = shard_of(self.cuts, self.rank, rows)
        self.shard_rows = [shard_of(self.cuts, r, rows).rows for r in range(self.world)]
        lrp, lci, lv = local_rows(row_ptr, col_idx, values, self.shard)
        self.csr = T.CsrMatrix(self.shard.rows, cols, lrp, lci, lv)
        self.me = T.encode_mebcrs(self.csr, precision)
        self.cfg = T.KernelConfig(precision)
        self._T = T

    def __call__(self, B: torch.Tensor, gather: bool = False) -> torch.Tensor:
        C = self._T.spmm(self.me, B, self.cfg).output
        return gather_rows(C, self.shard_rows, self.group) if gather else C


def local_input(H: torch.Tensor, shard: Shard, rows: int) -> torch.Tensor:
    """The rows of H this rank owns: H is either the full matrix (every
    node) or already the shard's rows (a previous layer's local output)."""
    if H.shape[0] == shard.rows:
        return H
    if H.shape[0] != rows:
        raise ValueError(f"expected {rows} (all) or {shard.rows} (this shard's) rows, got {H.shape[0]}")
    return H[shard.r0:shard.r1]


class ShardedGCNLayer:
    """GCN layer H' = Â (H W) over all ranks (BASELINE configs[3]).  Each
    rank transforms only its own rows (cuBLAS GEMM), all-gathers the
    transformed rows in the SpMM's operand dtype (f16: half the bytes of
    gathering the f32 output, and no replicated GEMM), and aggregates its
    window shard of Â.  Input: all rows or this shard's rows; output: this
    shard's rows (``gather=False``, what the next layer takes) or all rows."""

    def __init__(self, rows, row_ptr, col_idx, weight, precision=None, group=None):
        from . import layers as L
        from . import tcsparse as T

        precision = T.Precision.fp16 if precision is None else precision
        rp, ci, v = L.normalized_adjacency(rows, row_ptr, col_idx)
        self.spmm = ShardedSpmm(rows, rows, rp, ci, v, precision, group)
        self.weight = weight
        self.rows = rows
        self.dtype = torch.float16 if precision == T.Precision.fp16 else torch.float32

    def __call__(self, H: torch.Tensor, gather: bool = True) -> torch.Tensor:
        sp = self.spmm
        Hl = local_input(H, sp.shard, self.rows)
        HW_local = (Hl.to(self.weight.dtype) @ self.weight).to(self.dtype)  # cuBLAS GEMM, own rows
        HW = gather_rows(HW_local.contiguous(), sp.shard_rows, sp.group)  # every node's row, f16
        return sp(HW, gather=gather)


class ShardedAGNNLayer:
    """AGNN layer (BASELINE configs[4]) over all ranks: the attention rows of
    a window shard need that shard's rows against every node's.  Each rank
    converts its own rows to the f16 gather operand, all-gathers that (half
    the bytes of gathering the f32 output) and computes its rows with
    tcs_agnn_attend (row offset = its first row).  Input: all rows or this
    shard's rows; output: this shard's rows (``gather=False``) or all rows."""

    def __init__(self, rows, row_ptr, col_idx, beta=1.0, group=None):
        from . import tcsparse as T

        self.rows = rows
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cuts = shard_windows(row_ptr, rows, world)
        self.shard = shard_of(self.cuts, rank, rows)
        self.shard_rows = [shard_of(self.cuts, r, rows).rows for r in range(world)]
        ones = torch.ones(col_idx.numel(), dtype=torch.float32, device=col_idx.device)
        lrp, lci, lv = local_rows(row_ptr, col_idx, ones, self.shard)
        self.mask = T.encode_mebcrs(T.CsrMatrix(self.shard.rows, rows, lrp, lci, lv), T.Precision.fp16)
        self.beta = float(beta)
        self.cfg = T.KernelConfig(T.Precision.fp16, static_mask=True)
        self._T = T

    def __call__(self, H: torch.Tensor, gather: bool = True, one_pass: bool = True) -> torch.Tensor:
        T = self._T
        if one_pass and H.shape[1] in (32, 64):  # as AGNNLayer: tcs_agnn_attend
            Hl = local_input(H, self.shard, self.rows)
            _, Hc_local = T.rows_normalize(Hl.float().contiguous(), torch.float16, normalized=False)
            Hc = gather_rows(Hc_local, self.shard_rows, self.group)  # every node's row, f16
            C = T.agnn_attend(self.mask, Hc, self.beta, self.cfg, row0=self.shard.r0)
        else:
            if H.shape[0] != self.rows:
                raise ValueError("the three-pass path needs every node's rows")
            Hn, Hc = T.rows_normalize(H.float().contiguous(), torch.float16)
            C = T.agnn_aggregate(self.mask, Hn, Hc, self.beta, self.cfg, row0=self.shard.r0)
        return gather_rows(C, self.shard_rows, self.group) if gather else C
