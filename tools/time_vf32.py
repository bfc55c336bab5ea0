"""Timing aid (TCS_LIB_PATH A/B builds): C3 FP16 SpMM at N = 64 / 128 / 256
on ME-BCRS handles with f32-stored values (the bit-exact variant the C++
drop-in adapter uses) and with binary16 values.  CUDA events, L2 flushed
before every call, median of 10; prints one JSON object (ms)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200._abi as abi  # noqa: E402
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
csr = T.CsrMatrix(rows, cols, rp, ci, v)
out = {}
for name, vdt in (("f32v", abi.TCS_DTYPE_F32), ("f16v", abi.TCS_DTYPE_F16)):
    me = T.encode_mebcrs(csr, T.Precision.fp16, value_dtype=vdt)
    for n in (64, 128, 256):
        B = G.dense(cols, n, 3, values="real", dtype=torch.float16)
        C = torch.empty(rows, n, device="cuda")
        out[f"{name}_n{n}"] = timed(lambda: T.spmm(me, B, T.KernelConfig(T.Precision.fp16), out=C))
    me.free()
print(json.dumps(out))
