"""SDDMM on the C3 pattern, F=32 (profiling aid: run under ncu -k regex:sddmm)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, v), T.Precision.fp16)
F = int(os.environ.get("F", "32"))
A = G.dense(rows, F, 4)
Bt = G.dense(cols, F, 5)
out = torch.empty(8 * me.num_vectors, device="cuda")
ops = T.SddmmOperands(me, A, Bt)
for _ in range(3):
    T.sddmm(ops, T.KernelConfig(), out_values=out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    T.sddmm(ops, T.KernelConfig(), out_values=out)
e1.record()
torch.cuda.synchronize()
print(f"sddmm F={F}: {e0.elapsed_time(e1) / 5:.3f} ms")
