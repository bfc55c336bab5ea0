"""Timing aid (TCS_LIB_PATH A/B builds): tcs_agnn_attend on C5 (R-MAT
scale 23, F=32, static mask), CUDA events, L2 flushed, median of 10."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.layers as L  # noqa: E402
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


rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
layer = L.AGNNLayer(rows, rp, ci, beta=1.0)
out = {}
for f in (32, 64):
    H = torch.randn(rows, f, device="cuda").half()
    C = torch.empty(rows, f, device="cuda")
    out[f"c5_attend_f{f}"] = timed(lambda: T.agnn_attend(layer.mask, H, 1.0, layer.mask_cfg, out=C))
print(json.dumps(out))
