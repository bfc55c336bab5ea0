"""C5 AGNN layer, three calls (profiling aid: ncu launch list of the last)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.layers as L  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
H = torch.randn(rows, 32, device="cuda")
layer = L.AGNNLayer(rows, rp, ci, beta=1.0)
for _ in range(3):
    layer(H)
    torch.cuda.synchronize()
print("ok")
