"""Paper ablations on B200, C3 Reddit-shaped
graph: the 8x1 swap-and-transpose SpMM with the memory-efficient (coalesced)
vs the direct thread mapping, against the non-swapped 16x1 baseline
(ref spmm.hpp:187-257), FP16 and TF32.  Prints one JSON object (timing aid).
CUDA events, L2 flushed before every timed call.

  python tools/ablation.py [--n 128] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import graphs as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()

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
N = args.n
out = {"workload": "C3 Reddit-shaped power law", "nodes": rows, "nnz": nnz, "N": N, "runs": []}
for pname in ("fp16", "tf32"):
    prec = T.Precision.fp16 if pname == "fp16" else T.Precision.tf32
    dt = torch.float16 if pname == "fp16" else torch.float32
    B = G.dense(cols, N, 2, dtype=dt)
    C = torch.empty(rows, N, device="cuda")
    me = T.encode_mebcrs(csr, prec)
    enc8 = timed(lambda: T.encode_mebcrs(csr, prec).free())
    maps = [("coalesced", T.ThreadMapping.coalesced)] + ([("direct", T.ThreadMapping.direct)] if pname == "fp16" else [])
    for mname, mp in maps:
        cfg = T.KernelConfig(prec, mapping=mp)
        ms = timed(lambda: T.spmm(me, B, cfg, out=C))
        ref_c = C.clone() if mname == "coalesced" else None
        if mname == "coalesced":
            base_out = ref_c
        else:
            assert torch.equal(C, base_out), "direct mapping changed the result"
        out["runs"].append({"kernel": f"swap8/{mname}", "precision": pname, "ms": round(ms, 4),
                            "gflops": round(2 * nnz * N / ms / 1e6, 1), "nv": me.num_vectors,
                            "mma": me.num_blocks * ((N + 15) // 16), "encode_ms": round(enc8, 3)})
    # SR-BCRS: the zero-vector padded format (ref srbcrs.hpp) on the same kernel
    sr = T.encode_srbcrs(me)
    enc_sr = timed(lambda: T.encode_srbcrs(me).free())
    ms = timed(lambda: T.spmm(sr, B, T.KernelConfig(prec), out=C))
    # long windows may be split at other points than on the compact format
    # (the work-list segment size follows the vector count), so real-valued
    # sums can associate differently: compare in rel-L2
    rel_sr = float((C - base_out).norm() / base_out.norm())
    assert rel_sr < 1e-5, rel_sr
    vb = 2 if pname == "fp16" else 4
    W = me.num_windows
    out["runs"].append({"kernel": "swap8/srbcrs", "precision": pname, "ms": round(ms, 4),
                        "gflops": round(2 * nnz * N / ms / 1e6, 1), "nv_padded": sr.num_padded,
                        "footprint_me_bytes": 4 * (W + 1) + me.num_vectors * (4 + 8 * vb),
                        "footprint_sr_bytes": 8 * W + sr.num_padded * (4 + 8 * vb),
                        "pad_ms": round(enc_sr, 3), "rel_l2_vs_swap8": rel_sr})
    sr.free()
    me.free()
    m16 = T.encode_mebcrs(csr, prec, vector_height=16)
    enc16 = timed(lambda: T.encode_mebcrs(csr, prec, vector_height=16).free())
    ms = timed(lambda: T.spmm_baseline16(m16, B, out=C))
    rel = float((C - base_out).norm() / base_out.norm())
    out["runs"].append({"kernel": "baseline16", "precision": pname, "ms": round(ms, 4),
                        "gflops": round(2 * nnz * N / ms / 1e6, 1), "nv": m16.num_vectors,
                        "mma": m16.num_blocks * ((N + 7) // 8), "encode_ms": round(enc16, 3),
                        "rel_l2_vs_swap8": rel})
    m16.free()
    del B, C
    torch.cuda.empty_cache()
print(json.dumps(out))
