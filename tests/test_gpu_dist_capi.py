"""The multi-GPU C-ABI (include/tcs/tcs_dist.h) from C++ with a real NCCL
communicator: oracle/_ref/dist_gpu (built here against the reference
headers, shipped prebuilt) checks tcsparse::gpu::spmm_sharded against the
reference spmm bit for bit, the nnz cut rule, shard encodes as slices of the
whole encode, tcs_spmm_sharded == tcs_spmm, and the NCCL error / timeout
taxonomy (ncclCommAbort on timeout)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dist_gpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="dist_gpu not built (needs the reference headers)")
def test_multi_gpu_capi_from_cpp():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "all multi-GPU C-ABI checks passed" in p.stdout
