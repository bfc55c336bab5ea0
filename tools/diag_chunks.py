"""Diagnostic: encode + SpMM times of the 8 window-range chunks the host
pipeline (tcs_spmm_csr_host) cuts C3 into, each timed alone with CUDA
events -- to see the per-chunk fixed costs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
nnz = ci.numel()
B = G.dense(cols, 128, 3, dtype=torch.float16)
nch = int(sys.argv[1]) if len(sys.argv) > 1 else 8
W = (rows + 7) // 8
rp_h = rp.cpu()
cuts = [0]
for i in range(1, nch):
    target = nnz * i // nch
    w = int(torch.searchsorted(rp_h[0::8].contiguous(), torch.tensor([target]), right=False)[0])
    cuts.append(max(cuts[-1], min(W, w)))
cuts.append(W)


def ev():
    return torch.cuda.Event(enable_timing=True)


for i in range(nch):
    r0, r1 = min(rows, 8 * cuts[i]), min(rows, 8 * cuts[i + 1])
    lrp, lci, lv = G.row_slice(rp, ci, v, r0, r1)
    csr = T.CsrMatrix(r1 - r0, cols, lrp, lci, lv)
    for rep in range(2):
        a, b, c = ev(), ev(), ev()
        a.record()
        me = T.encode_mebcrs(csr, T.Precision.fp16)
        b.record()
        out = T.spmm(me, B, T.KernelConfig()).output
        c.record()
        torch.cuda.synchronize()
        if rep:
            print(f"chunk {i}: rows {r1 - r0} nnz {lci.numel()} encode {a.elapsed_time(b):.3f} ms "
                  f"spmm {b.elapsed_time(c):.3f} ms nv {me.num_vectors}")
        me.free()
