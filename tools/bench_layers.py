"""BASELINE configs[3] / configs[4] on one B200: GCN layer on the
ogbn-products-shaped graph and AGNN layer on R-MAT scale 23 (timing aid;
prints one JSON object).  CUDA events, L2 flushed before each timed call."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.layers as L  # noqa: E402
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


out = {}
which = sys.argv[1:] or ["c4", "c5"]
if "c4" in which:
    t = time.time()
    rows, cols, rp, ci, v = G.power_law_csr(G.C4_PRODUCTS, values="real")
    gen_s = time.time() - t
    F = 128
    W = torch.randn(F, F, device="cuda").half() / F ** 0.5
    H = torch.randn(rows, F, device="cuda").half()
    t = time.time()
    layer = L.GCNLayer(rows, rp, ci, W)
    torch.cuda.synchronize()
    build_s = time.time() - t
    nnz = layer.adj.num_vectors  # placeholder, replaced below
    nnz = int(ci.numel()) + rows  # A + I
    HW = (H @ W)
    spmm_ms = timed(lambda: T.spmm(layer.adj, HW, layer.cfg))
    layer_ms = timed(lambda: layer(H))
    gemm_ms = timed(lambda: H @ W)
    out["c4_gcn"] = {"nodes": rows, "nnz_with_self_loops": nnz, "F": F, "max_window_vectors": layer.adj.max_window_vectors,
                     "spmm_ms": round(spmm_ms, 3), "gemm_ms": round(gemm_ms, 3), "layer_ms": round(layer_ms, 3),
                     "spmm_gflops": round(2 * nnz * F / spmm_ms / 1e6, 1), "gen_s": round(gen_s, 1),
                     "build_s": round(build_s, 2)}
    del layer, H, HW, rp, ci, v
    torch.cuda.empty_cache()
if "c5" in which:
    t = time.time()
    rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
    gen_s = time.time() - t
    F = 32
    H = torch.randn(rows, F, device="cuda")
    t = time.time()
    layer = L.AGNNLayer(rows, rp, ci, beta=1.0)
    torch.cuda.synchronize()
    build_s = time.time() - t
    nnz = int(ci.numel())
    Hn = torch.nn.functional.normalize(H, dim=1).half()
    sddmm_ms = timed(lambda: T.sddmm(T.SddmmOperands(layer.mask, Hn, Hn), layer.cfg))
    scores = T.sddmm(T.SddmmOperands(layer.mask, Hn, Hn), layer.cfg).output
    softmax_ms = timed(lambda: T.row_softmax(scores, layer.mask, 1.0))
    P = T.row_softmax(scores, layer.mask, 1.0)
    spmm_ms = timed(lambda: T.spmm(P, H.half(), layer.cfg))
    fused_ms = timed(lambda: T.sddmm_row_softmax(T.SddmmOperands(layer.mask, Hn, Hn), 1.0, layer.cfg,
                                                 score_dtype=0, out_dtype=0))
    fused_static_ms = timed(lambda: T.sddmm_row_softmax(T.SddmmOperands(layer.mask, Hn, Hn), 1.0, layer.mask_cfg,
                                                        score_dtype=0, out_dtype=0))
    Hc = H.half()
    agg_ms = timed(lambda: T.agnn_aggregate(layer.mask, Hn, Hc, 1.0, layer.mask_cfg))
    attend_ms = timed(lambda: T.agnn_attend(layer.mask, Hc, 1.0, layer.mask_cfg))
    layer3_ms = timed(lambda: layer(H, one_pass=False))
    layer_ms = timed(lambda: layer(H))
    out["c5_agnn"] = {"agnn_attend_ms": round(attend_ms, 3), "layer_three_pass_ms": round(layer3_ms, 3),
                      "agnn_aggregate_ms": round(agg_ms, 3),"fused_sddmm_softmax_static_mask_ms": round(fused_static_ms, 3),"nodes": rows, "nnz": nnz, "nv": layer.mask.num_vectors, "F": F,
                      "max_window_vectors": layer.mask.max_window_vectors,
                      "sddmm_ms": round(sddmm_ms, 3), "softmax_ms": round(softmax_ms, 3),
                      "fused_sddmm_softmax_ms": round(fused_ms, 3), "spmm_ms": round(spmm_ms, 3),
                      "layer_ms": round(layer_ms, 3), "sddmm_gflops": round(2 * nnz * F / sddmm_ms / 1e6, 1),
                      "spmm_gflops": round(2 * nnz * F / spmm_ms / 1e6, 1), "gen_s": round(gen_s, 1),
                      "build_s": round(build_s, 2)}
print(json.dumps(out))
