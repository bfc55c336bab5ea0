"""One tcs_spmm_csr_host call on C3 FP16 N=128 (after a warm-up call)
inside cudaProfilerStart/Stop, for `ncu --profile-from-start off` launch
lists of the pipelined chunk encode + SpMM."""
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
for i in range(2):
    if i:
        torch.cuda.profiler.start()
    rc = lib.tcs_spmm_csr_host(C.byref(csr), 0, B_h.data_ptr(), N, C_h.data_ptr(), C.byref(cfg), None,
                               C.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0, lib.tcs_last_error()
torch.cuda.profiler.stop()
print("ok")
