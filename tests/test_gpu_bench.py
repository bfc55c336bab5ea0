"""bench.py contract on the GPU: one JSON line with the driver's keys, at
world size 1 and -- through torchrun with the gloo backend, both ranks on
the one visible GPU -- at world size 2 (the sharded multi-rank path:
nnz-balanced window shards, B broadcast, max-over-ranks timing).  Small
workload (C1); the timings themselves are not checked."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"}


def _run(cmd, env=None):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ, **(env or {}))
    r = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    line = _run([sys.executable, "bench.py", "--workload", "c1", "--quick", "--steps", "3", "--warmup", "3"])
    assert KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] >= 3
    assert line["roofline"]["bound"] == "hbm" and line["roofline"]["achieved"] > 0


def test_bench_two_ranks_sharded():
    one = _run([sys.executable, "bench.py", "--workload", "c1", "--quick", "--steps", "3", "--warmup", "3"])
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--workload",
                "c1", "--quick", "--steps", "3", "--warmup", "3"], env={"TCS_DIST_BACKEND": "gloo"})
    assert two["n_gpus"] == 2 and len(two["shards"]) == 2
    assert sum(s["nnz"] for s in two["shards"]) == one["config"]["nnz"]
    # windows never straddle shards, so the vector count is the same
    assert two["config"]["nv_8x1"] == one["config"]["nv_8x1"]


def test_bench_gpus_flag_launches_ranks_itself():
    """`bench.py --gpus 2` with no torchrun: bench.py starts the ranks itself
    (gloo when the box has fewer GPUs than ranks, NCCL otherwise)."""
    one = _run([sys.executable, "bench.py", "--workload", "c1", "--quick", "--steps", "3", "--warmup", "3"])
    two = _run([sys.executable, "bench.py", "--gpus", "2", "--workload", "c1", "--quick", "--steps", "3",
                "--warmup", "3"])
    assert two["n_gpus"] == 2 and len(two["shards"]) == 2
    assert two["config"]["backend"] in ("nccl", "gloo")
    if torch.cuda.device_count() >= 2:
        assert two["config"]["backend"] == "nccl"
    assert sum(s["nnz"] for s in two["shards"]) == one["config"]["nnz"]
    ref = _run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--workload", "c1", "--steps", "3",
                "--warmup", "3"])
    assert ref["impl"] == "reference" and ref["n_gpus"] == 2 and ref["value"] > 0
