"""Timing aid: tcs_spmm_csr_host on C3 FP16 N=128 from pinned host buffers
(the bench's e2e call), median of 7 after one warm-up.  TCS_LIB_PATH picks
the build."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_11007_b200 import _abi, graphs as G  # noqa: E402

rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="real")
N = 128
B = G.dense(cols, N, 3, dtype=torch.float32)
rp_h, ci_h, v_h = rp.cpu().pin_memory(), ci.cpu().pin_memory(), v.cpu().pin_memory()
B_h = B.cpu().pin_memory()
C_h = torch.empty(rows, N).pin_memory()
lib = _abi.load()
csr = _abi.tcs_csr(rows, cols, ci.numel(), rp_h.data_ptr(), ci_h.data_ptr(), v_h.data_ptr())
cfg = _abi.tcs_kernel_config(0, 8, 1, 0)
st = torch.cuda.current_stream()
ts = []
for i in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    rc = lib.tcs_spmm_csr_host(C.byref(csr), 0, B_h.data_ptr(), N, C_h.data_ptr(), C.byref(cfg), None,
                               C.c_void_p(st.cuda_stream))
    b.record(st)
    torch.cuda.synchronize()
    assert rc == 0, lib.tcs_last_error()
    if i:
        ts.append(a.elapsed_time(b))
print(os.environ.get("TCS_LIB_PATH", "default"), "e2e ms median", sorted(ts)[len(ts) // 2], "min", min(ts))
