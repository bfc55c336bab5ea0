"""Diagnostic: C5 (R-MAT scale 23) window-size classes as the encoder sees
them (entries per 8-row window: small <= 2048, medium <= 12288, huge)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_11007_b200 import graphs as G  # noqa: E402

rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
rp = rp.long()
W = (rows + 7) // 8
idx = torch.arange(W + 1, device=rp.device) * 8
n = rp[idx.clamp(max=rows)][1:] - rp[idx.clamp(max=rows)][:-1]
for name, lo, hi in (("small", 0, 2048), ("medium", 2049, 12288), ("huge", 12289, 1 << 40)):
    m = (n >= lo) & (n <= hi)
    print(f"{name:6s} windows {int(m.sum()):9d}  entries {int(n[m].sum()):11d}")
top = torch.topk(n, 20).values.tolist()
print("largest windows (entries):", top)
print("entries in windows > 100k:", int(n[n > 100000].sum()), "count", int((n > 100000).sum()))
