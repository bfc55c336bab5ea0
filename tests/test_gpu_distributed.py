"""Chained GNN layers sharded over ranks (the §8(e) all-gather chaining),
run through torchrun with 2 ranks on gloo -- both ranks on the one visible
GPU, so this checks the sharding and chaining logic on the real kernels,
not NVLink performance.  Each rank's rows must match the single-process
layers: AGNN bit for bit (a row's softmax and aggregation do not depend on
the shard), GCN to fp32 rounding (split windows can associate their
partial sums differently when the shard's work list cuts them elsewhere)."""
import os
import re
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sharded_gcn_and_agnn_chain_match_single_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", "tests/_dist_layers_worker.py"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = re.findall(r"RANK(\d) gcn_rel_l2=(\S+) agnn_exact=(\S+) agnn_rel_l2=(\S+)", r.stdout)
    assert len(lines) == 2, r.stdout
    for _, gcn, exact, _agnn in lines:
        assert float(gcn) < 1e-5
        assert exact == "True"
