"""Fused SDDMM -> row softmax on the C5 R-MAT pattern, F=32 (profiling aid:
run under `ncu --metrics gpu__time_duration.sum` for the per-kernel split)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

g = G.C5_RMAT if os.environ.get("GRAPH", "c5") == "c5" else G.C3_REDDIT
rows, cols, rp, ci, v = (G.rmat_csr if g is G.C5_RMAT else G.power_law_csr)(g, values="real")
me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, torch.ones_like(v)), T.Precision.fp16)
H = torch.nn.functional.normalize(torch.randn(rows, 32, device="cuda"), dim=1).half()
ops = T.SddmmOperands(me, H, H)
for _ in range(int(os.environ.get("REPS", "2"))):
    P = T.sddmm_row_softmax(ops, 1.0, T.KernelConfig(), score_dtype=0, out_dtype=0)
    S = T.sddmm(ops, T.KernelConfig(), out_dtype=0).output
    P2 = T.row_softmax(S, me, 1.0, 0)
    torch.cuda.synchronize()
    del P, S, P2
print("ok")
