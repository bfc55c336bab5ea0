"""One call of a hot-path operator inside cudaProfilerStart/Stop (profiling
aid: run under `ncu --profile-from-start off ...`, so only that call's
kernels are captured; a warm-up call precedes it so the memory pool and the
plan are settled).

  python tools/profile_ops.py CONFIG OP [PRECISION] [N_OR_F]
    CONFIG: c1 | c3 | c4 | c5      OP: spmm | sddmm | sddmm_static | encode | attend (AGNN, F = N_OR_F)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

cfg_name, op = sys.argv[1], sys.argv[2]
prec = T.Precision.fp16 if (sys.argv[3] if len(sys.argv) > 3 else "fp16") == "fp16" else T.Precision.tf32
width = int(sys.argv[4]) if len(sys.argv) > 4 else (32 if op.startswith("sddmm") else 128)
dt = torch.float16 if prec == T.Precision.fp16 else torch.float32
if cfg_name == "c1":  # the reference's own C1 inputs (generate.hpp restated)
    rows = cols = 4096
    rp, ci, v = (torch.from_numpy(x.view("int32") if x.dtype.kind == "u" else x).cuda()
                 for x in G.reference_random_csr(rows, cols, 16.0 / 4096, 1, "real"))
elif cfg_name == "c3":
    rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
elif cfg_name == "c4":
    rows, cols, rp, ci, v = G.power_law_csr(G.C4_PRODUCTS, values="real")
else:
    rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="real")
csr = T.CsrMatrix(rows, cols, rp, ci, v)
me = T.encode_mebcrs(csr, prec)
if op == "spmm":
    B = G.dense(cols, width, 2, dtype=dt)
    C = torch.empty(rows, width, device="cuda")
    call = lambda: T.spmm(me, B, T.KernelConfig(prec), out=C)  # noqa: E731
elif op.startswith("sddmm"):
    A = G.dense(rows, width, 4, dtype=dt)
    Bt = G.dense(cols, width, 5, dtype=dt)
    ov = torch.empty(8 * me.num_vectors, device="cuda")
    kc = T.KernelConfig(prec, static_mask=(op == "sddmm_static"))
    call = lambda: T.sddmm(T.SddmmOperands(me, A, Bt), kc, out_values=ov)  # noqa: E731
elif op == "attend":  # one-pass AGNN attention on the layer's static mask (tools/time_attend.py)
    import paper_2412_11007_b200.layers as L  # noqa: E402

    layer = L.AGNNLayer(rows, rp, ci, beta=1.0)
    H = torch.randn(rows, width, device="cuda").half()
    C = torch.empty(rows, width, device="cuda")
    call = lambda: T.agnn_attend(layer.mask, H, 1.0, layer.mask_cfg, out=C)  # noqa: E731
else:
    call = lambda: T.encode_mebcrs(csr, prec)  # noqa: E731
for _ in range(2):
    call()
torch.cuda.synchronize()
torch.cuda.profiler.start()
call()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
