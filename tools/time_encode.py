"""Timing aid: CSR -> ME-BCRS on C3 (FP16 values) and C5, median of 5 (CUDA
events around the whole call, host syncs included).  TCS_LIB_PATH picks
the build."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

out = {}
for name, gen in [x for x in (("c3", lambda: G.power_law_csr(G.C3_REDDIT, values="real")), ("c5", lambda: G.rmat_csr(G.C5_RMAT, values="real"))) if x[0] in (sys.argv[1:] or ["c3", "c5"])]:
    rows, cols, rp, ci, v = gen()
    csr = T.CsrMatrix(rows, cols, rp, ci, v)
    ts = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        me = T.encode_mebcrs(csr, T.Precision.fp16)
        b.record()
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
        me.free()
    out[name] = round(sorted(ts)[len(ts) // 2], 3)
    del csr, rp, ci, v
    torch.cuda.empty_cache()
print(os.environ.get("TCS_LIB_PATH", "default"), out)
