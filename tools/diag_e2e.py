"""Stage timings of the host-buffer pipeline (profiling aid, not a bench)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11007_b200.tcsparse as T  # noqa: E402
from paper_2412_11007_b200 import _abi, graphs as G  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = ev(), ev()
        w0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
        wall = (time.perf_counter() - w0) * 1e3
    print(f"{label:40s} {best:9.3f} ms (events)  {wall:9.3f} ms (wall, last)")


rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
N = 128
csr = T.CsrMatrix(rows, cols, rp, ci, v)
B = G.dense(cols, N, 3, dtype=torch.float32)
rp_h, ci_h, v_h = rp.cpu().pin_memory(), ci.cpu().pin_memory(), v.cpu().pin_memory()
B_h = B.cpu().pin_memory()
C_h = torch.empty(rows, N).pin_memory()
rp_d, ci_d, v_d = torch.empty_like(rp), torch.empty_like(ci), torch.empty_like(v)
B_d = torch.empty_like(B)
C_d = torch.empty(rows, N, device="cuda")

timed("H2D CSR (torch, pinned)", lambda: (rp_d.copy_(rp_h, non_blocking=True), ci_d.copy_(ci_h, non_blocking=True),
                                         v_d.copy_(v_h, non_blocking=True)))
timed("H2D B f32", lambda: B_d.copy_(B_h, non_blocking=True))
timed("D2H C f32", lambda: C_h.copy_(C_d, non_blocking=True))
me_holder = {}


def enc():
    if "me" in me_holder:
        me_holder["me"].free()
    me_holder["me"] = T.encode_mebcrs(csr, T.Precision.fp16)


timed("encode (device CSR)", enc)
timed("spmm f32 B (convert+kernel)", lambda: T.spmm(me_holder["me"], B, T.KernelConfig(), out=C_d))
Bh16 = B.half()
timed("spmm f16 B (kernel)", lambda: T.spmm(me_holder["me"], Bh16, T.KernelConfig(), out=C_d))
lib = _abi.load()
c = _abi.tcs_csr(rows, cols, ci.numel(), rp_h.data_ptr(), ci_h.data_ptr(), v_h.data_ptr())
cfg = _abi.tcs_kernel_config(0, 8, 1, 0)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def host_encode():
    h = _abi.tcs_mebcrs()
    assert lib.tcs_mebcrs_encode_host(C.byref(c), 0, 0, C.byref(h), s) == 0
    lib.tcs_mebcrs_free(C.byref(h), s)


timed("tcs_mebcrs_encode_host", host_encode)
timed("tcs_spmm_csr_host", lambda: lib.tcs_spmm_csr_host(C.byref(c), 0, B_h.data_ptr(), N, C_h.data_ptr(),
                                                          C.byref(cfg), None, s))
