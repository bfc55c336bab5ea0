"""The drop-in proof: reference acceptance criteria 2, 3, 6, 7 re-run with
tcsparse::gpu:: substituted for the reference functions
(oracle/acceptance_gpu.cpp, built here against the reference headers and
shipped prebuilt; links libtcsparse_b200.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="acceptance_gpu not built (needs the reference headers)")
def test_reference_acceptance_with_gpu_dropin():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "all drop-in criteria passed" in p.stdout
