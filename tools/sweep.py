"""BASELINE configs[2] grid on one B200 (timing aid; prints one JSON object):
SpMM FP16/TF32 at N = 64/128/256 and SDDMM FP16/TF32 at F = 32/64/128 on
the Reddit-shaped power-law graph, each with its SURVEY §8(d) algorithmic
bytes and the fraction of the measured HBM peak.  CUDA events on the
launching stream, L2 flushed (256 MB write) before every timed call.

  python tools/sweep.py [--n 64 128 256] [--f 32 64 128] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import _abi  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="*", default=[64, 128, 256])
ap.add_argument("--f", type=int, nargs="*", default=[32, 64, 128])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--precisions", nargs="*", default=["fp16", "tf32"])
args = ap.parse_args()

with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
    PEAK = float(json.load(f)["hbm_gbs"])

flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
nnz = int(ci.numel())
csr = T.CsrMatrix(rows, cols, rp, ci, v)
out = {"workload": "C3 Reddit-shaped power law", "nodes": rows, "nnz": nnz, "peak_gbs": PEAK,
       "l2": "flushed before every timed call", "spmm": [], "sddmm": []}
for pname in args.precisions:
    prec = T.Precision.fp16 if pname == "fp16" else T.Precision.tf32
    dt = torch.float16 if pname == "fp16" else torch.float32
    me = T.encode_mebcrs(csr, prec)
    W, nv = me.num_windows, me.num_vectors
    vA = 2 if me.value_dtype == _abi.TCS_DTYPE_F16 else 4
    vB = 2 if dt == torch.float16 else 4
    cfg = T.KernelConfig(prec)
    for N in args.n:
        B = G.dense(cols, N, 2, dtype=dt)
        C = torch.empty(rows, N, device="cuda")
        ms = timed(lambda: T.spmm(me, B, cfg, out=C))
        balg = 4 * (W + 1) + 4 * nv + 8 * nv * vA + nv * N * vB + 4 * rows * N
        bmin = 4 * (W + 1) + 4 * nv + 8 * nv * vA + cols * N * vB + 4 * rows * N
        out["spmm"].append({"precision": pname, "N": N, "ms": round(ms, 4),
                            "gflops": round(2 * nnz * N / ms / 1e6, 1),
                            "bytes_alg": balg, "alg_gbs": round(balg / ms / 1e6, 1),
                            "frac_alg": round(balg / ms / 1e6 / PEAK, 4),
                            "frac_min": round(bmin / ms / 1e6 / PEAK, 4)})
        del B, C
    for F in args.f:
        A = G.dense(rows, F, 4, dtype=dt)
        Bt = G.dense(cols, F, 5, dtype=dt)
        ov = torch.empty(8 * nv, device="cuda")
        ops = T.SddmmOperands(me, A, Bt)
        ms = timed(lambda: T.sddmm(ops, cfg, out_values=ov))
        balg = 4 * (W + 1) + 4 * nv + 8 * nv * vA + rows * F * vB + nv * F * vB + 8 * nv * 4
        out["sddmm"].append({"precision": pname, "F": F, "ms": round(ms, 4),
                             "gflops": round(2 * nnz * F / ms / 1e6, 1),
                             "bytes_alg": balg, "alg_gbs": round(balg / ms / 1e6, 1),
                             "frac_alg": round(balg / ms / 1e6 / PEAK, 4)})
        del A, Bt, ov
    me.free()
    torch.cuda.empty_cache()
print(json.dumps(out))
