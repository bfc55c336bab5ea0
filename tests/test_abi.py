"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads
without a GPU, exports every symbol include/tcs/tcs.h declares, and fails
loudly (TCS_ERR_CUDA, never a silent CPU fallback) when no device exists."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", "tcs", h) for h in ("tcs.h", "tcs_dist.h")]


def declared_functions():
    names = set()
    for header in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(header).read(), flags=re.S)
        names |= set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tcs_\w+)\s*\(", src, flags=re.M))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    from paper_2412_11007_b200 import _abi

    if not os.path.exists(_abi.LIB_PATH):
        subprocess.run(["make", "-s", "-C", ROOT, "lib"], check=True)
    return _abi.load()


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for required in ("tcs_mebcrs_encode", "tcs_spmm", "tcs_sddmm", "tcs_mebcrs_free", "tcs_last_error",
                     "tcs_spmm_host", "tcs_sddmm_host", "tcs_mebcrs_download"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2412_11007_b200 import _abi

    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _abi.EXPORTS, f"{name} missing from the ctypes table"


def test_struct_layouts_match_header(lib):
    from paper_2412_11007_b200 import _abi

    assert C.sizeof(_abi.tcs_csr) == 48
    assert C.sizeof(_abi.tcs_mebcrs) == 104
    assert C.sizeof(_abi.tcs_kernel_config) == 16
    assert C.sizeof(_abi.tcs_counters) == 32
    assert C.sizeof(_abi.tcs_dist) == 24


def test_version_and_no_silent_fallback(lib):
    import torch

    assert b"sm_100a" in lib.tcs_version()
    if torch.cuda.is_available():
        pytest.skip("GPU present: the no-device path is not reachable")
    from paper_2412_11007_b200 import _abi

    h = _abi.tcs_mebcrs()
    import numpy as np

    rp = np.zeros(2, np.uint32)
    rc = lib.tcs_mebcrs_upload(8, 8, 0, rp.ctypes.data, None, None, C.byref(h), None)
    assert rc == _abi.TCS_ERR_CUDA, rc
    assert lib.tcs_last_error()  # a message, not silence


def test_argument_errors_precede_device_work(lib):
    from paper_2412_11007_b200 import _abi

    cfg = _abi.tcs_kernel_config(0, 16, 1, 0)
    rc = lib.tcs_spmm_host(8, 8, 0, None, None, None, None, 8, 16, None, C.byref(cfg), None, None)
    assert rc == _abi.TCS_ERR_ARGUMENT  # vector height 16 (ref spmm.hpp:106)
    cfg = _abi.tcs_kernel_config(1, 8, 1, 0)
    rc = lib.tcs_spmm_host(8, 8, 0, None, None, None, None, 8, 16, None, C.byref(cfg), None, None)
    assert rc == _abi.TCS_ERR_ARGUMENT  # precision mismatch (ref spmm.hpp:107)
    cfg = _abi.tcs_kernel_config(0, 8, 1, 0)
    rc = lib.tcs_spmm_host(8, 8, 0, None, None, None, None, 9, 16, None, C.byref(cfg), None, None)
    assert rc == _abi.TCS_ERR_SHAPE  # sparse cols != dense rows (ref spmm.hpp:109)


def test_dist_argument_errors_without_device(lib):
    """tcs_dist_* reject bad arguments before touching NCCL or the device."""
    from paper_2412_11007_b200 import _abi

    d = _abi.tcs_dist()
    assert lib.tcs_dist_init(C.byref(d), None, 0) == _abi.TCS_ERR_ARGUMENT
    assert lib.tcs_dist_broadcast(C.byref(d), None, 0, 0, None) == _abi.TCS_ERR_NCCL  # never bound
    assert b"communicator" in lib.tcs_last_error()
    assert lib.tcs_shard_windows(None, 2, None, None) == _abi.TCS_ERR_ARGUMENT
