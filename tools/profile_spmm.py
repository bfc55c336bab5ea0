"""SpMM variants for ncu (profiling aid): `c3tf32` = C3 TF32 N=128,
`c3tc05` = C3 FP16 N=128 on the tcgen05 path, `c4` = C4
products-shaped FP16 N=128 (the GCN aggregation), `c5` = C5
R-MAT FP16 N=32.  Three rounds; profile the last with --launch-skip."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

which = sys.argv[1]
path = "auto"
if which == "c3tc05":
    rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
    prec, N, dt, path = T.Precision.fp16, 128, torch.float16, "tcgen05"
elif which == "c3tf32":
    rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
    prec, N, dt = T.Precision.tf32, 128, torch.float32
elif which == "c4":
    rows, cols, rp, ci, v = G.power_law_csr(G.C4_PRODUCTS, values="real")
    prec, N, dt = T.Precision.fp16, 128, torch.float16
else:
    rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
    prec, N, dt = T.Precision.fp16, 32, torch.float16
csr = T.CsrMatrix(rows, cols, rp, ci, v)
me = T.encode_mebcrs(csr, prec)
B = G.dense(cols, N, 2, dtype=dt)
C = torch.empty(rows, N, device="cuda")
for _ in range(3):
    T.spmm(me, B, T.KernelConfig(prec, path=path), out=C)
    torch.cuda.synchronize()
print("ok")
