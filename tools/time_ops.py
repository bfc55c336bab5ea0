"""Timing aid for A/B builds (TCS_LIB_PATH): SpMM on C3 (FP16 / TF32,
N=128), C4 (FP16, N=128), C5 (FP16, N=32) and SDDMM on C3 and C5 (FP16, F=32).
CUDA events, L2 flushed before every timed call; prints one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=10):
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
    return round(sorted(ts)[len(ts) // 2], 4)


which = sys.argv[1:] or ["c3", "c4", "c5"]
out = {}
if "c3" in which:
    rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
    csr = T.CsrMatrix(rows, cols, rp, ci, v)
    for prec, dt in ((T.Precision.fp16, torch.float16), (T.Precision.tf32, torch.float32)):
        me = T.encode_mebcrs(csr, prec)
        B = G.dense(cols, 128, 2, dtype=dt)
        C = torch.empty(rows, 128, device="cuda")
        out[f"c3_spmm_{prec.name}_n128"] = timed(lambda: T.spmm(me, B, T.KernelConfig(prec), out=C))
        if prec == T.Precision.fp16:
            B1 = G.dense(cols, 64, 2, dtype=dt)
            C1 = torch.empty(rows, 64, device="cuda")
            out["c3_spmm_fp16_n64"] = timed(lambda: T.spmm(me, B1, T.KernelConfig(prec), out=C1))
            del B1, C1
            B2 = G.dense(cols, 256, 2, dtype=dt)
            C2 = torch.empty(rows, 256, device="cuda")
            out["c3_spmm_fp16_n256"] = timed(lambda: T.spmm(me, B2, T.KernelConfig(prec), out=C2))
            del B2, C2
        if prec == T.Precision.fp16:
            A = G.dense(rows, 32, 4)
            Bt = G.dense(cols, 32, 5)
            ov = torch.empty(8 * me.num_vectors, device="cuda")
            out["c3_sddmm_fp16_f32"] = timed(lambda: T.sddmm(T.SddmmOperands(me, A, Bt), T.KernelConfig(), out_values=ov))
            sm = T.KernelConfig(static_mask=True)
            out["c3_sddmm_fp16_f32_static"] = timed(lambda: T.sddmm(T.SddmmOperands(me, A, Bt), sm, out_values=ov))
            del A, Bt, ov
        me.free()
        del B, C
    del csr, rp, ci, v
    torch.cuda.empty_cache()
if "c4" in which:
    rows, cols, rp, ci, v = G.power_law_csr(G.C4_PRODUCTS, values="real")
    me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, v), T.Precision.fp16)
    B = G.dense(cols, 128, 2)
    C = torch.empty(rows, 128, device="cuda")
    out["c4_spmm_fp16_n128"] = timed(lambda: T.spmm(me, B, T.KernelConfig(), out=C))
    me.free()
    del B, C, rp, ci, v
    torch.cuda.empty_cache()
if "c5" in which:
    rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
    me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, v), T.Precision.fp16)
    B = G.dense(cols, 32, 2)
    C = torch.empty(rows, 32, device="cuda")
    out["c5_spmm_fp16_n32"] = timed(lambda: T.spmm(me, B, T.KernelConfig(), out=C))
    del B, C
    A = G.dense(rows, 32, 4)
    Bt = G.dense(cols, 32, 5)
    ov = torch.empty(8 * me.num_vectors, device="cuda")
    out["c5_sddmm_fp16_f32"] = timed(lambda: T.sddmm(T.SddmmOperands(me, A, Bt), T.KernelConfig(), out_values=ov))
    del A, Bt, ov
    me.free()
print(json.dumps(out))
