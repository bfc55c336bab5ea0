"""Timing aid: C3 TF32 SpMM at N = 64 / 128 / 256, packed dense operand vs
the f32-gather ablation (TCS_CFG_TF32_F32_GATHER).  CUDA events, L2 flushed
before every call, median of 10; prints one JSON object (ms)."""
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


rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, v), T.Precision.tf32)
out = {}
for n in (64, 128, 256):
    B = G.dense(cols, n, 3, values="real", dtype=torch.float32)
    C = torch.empty(rows, n, device="cuda")
    out[f"n{n}_packed"] = timed(lambda: T.spmm(me, B, T.KernelConfig(T.Precision.tf32), out=C))
    out[f"n{n}_f32"] = timed(lambda: T.spmm(me, B, T.KernelConfig(T.Precision.tf32, tf32_f32_gather=True), out=C))
    del B, C
print(json.dumps(out))
