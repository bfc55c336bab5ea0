"""The multi-GPU C-ABI on torch's own NCCL communicator (the path bench.py
and the sharded layers take under an NCCL process group): a world-1 NCCL
group on cuda:0 (NCCL refuses two ranks on one device, and the test box has
one GPU).  tcs_dist_init on ProcessGroupNCCL._comm_ptr(), a broadcast, and
tcs_spmm_sharded with B broadcast + C exchange == tcs_spmm bit for bit."""
import ctypes as C
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import ctypes as C, os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
import paper_2412_11007_b200.tcsparse as T
from paper_2412_11007_b200 import _abi, distributed as D, graphs as G
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
d = D.tcs_dist()
assert d is not None and d.world == 1 and d.rank == 0
lib = _abi.load()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
x = torch.arange(1000, dtype=torch.float32, device="cuda")
assert lib.tcs_dist_broadcast(C.byref(d), C.c_void_p(x.data_ptr()), 4000, 0, s) == 0, lib.tcs_last_error()
assert lib.tcs_dist_wait(C.byref(d), s, 10000) == 0
assert torch.equal(x, torch.arange(1000, dtype=torch.float32, device="cuda"))
rows, cols, rp, ci, v = G.uniform_csr(3001, 2003, 0.02, seed=5, values="int", device="cuda")
csr = T.CsrMatrix(rows, cols, rp, ci, v)
hc = _abi.tcs_csr(rows, cols, ci.numel(), rp.data_ptr(), ci.data_ptr(), v.data_ptr())
cuts = (C.c_uint64 * 2)()
assert lib.tcs_shard_windows(C.byref(hc), 1, cuts, s) == 0
me = _abi.tcs_mebcrs()
assert lib.tcs_mebcrs_encode_shard(C.byref(hc), cuts[0], cuts[1], 0, 0, C.byref(me), s) == 0
B = G.dense(cols, 128, 3, dtype=torch.float16, device="cuda")
want = T.spmm(T.encode_mebcrs(csr, T.Precision.fp16), B, T.KernelConfig()).output
got = torch.full((rows, 128), float("nan"), device="cuda")
cfg = _abi.tcs_kernel_config(0, 8, 1, 0)
rc = lib.tcs_spmm_sharded(C.byref(d), cuts, rows, C.byref(me), C.c_void_p(B.data_ptr()), 0, 128, cols, 128, 0,
                          _abi.TCS_DIST_BROADCAST_B | _abi.TCS_DIST_ALLGATHER_C, C.c_void_p(got.data_ptr()), 128,
                          C.byref(cfg), None, s)
assert rc == 0, lib.tcs_last_error()
assert lib.tcs_dist_wait(C.byref(d), s, 10000) == 0
assert torch.equal(got, want)
lib.tcs_mebcrs_free(C.byref(me), s)
dist.destroy_process_group()
print("ok")
"""


def test_tcs_dist_on_torch_nccl_communicator():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT="29561", RANK="0", WORLD_SIZE="1")
    r = subprocess.run([sys.executable, "-c", WORKER], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
