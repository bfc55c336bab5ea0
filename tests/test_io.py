"""Ingest / container host logic against the reference (no GPU needed):
every malformed MatrixMarket input and every malformed MEBC container is
rejected by the C-ABI before any device work, with the reference's error
class and message (ref matrix_market.hpp:28-94, errors.hpp:11-22,
container_io.hpp:70-91, mebcrs.hpp:58-77)."""
import ctypes as C
import struct

import numpy as np
import pytest

import oracle as O
from paper_2412_11007_b200 import _abi

BANNER = "%%MatrixMarket matrix coordinate real general\n"

BAD_MTX = [
    "",
    "hello\n",
    "%%MatrixMarket vector coordinate real general\n",
    "%%MatrixMarket matrix array real general\n1 1\n",
    "%%MatrixMarket matrix coordinate complex general\n3 3 1\n",
    "%%MatrixMarket matrix coordinate real hermitian\n3 3 1\n",
    "%%matrixmarket matrix coordinate real general\n3 3 1\n",
    "%%MatrixMarket MATRIX Coordinate REAL General\n",
    BANNER,
    BANNER + "% c\n\n  \t\n3 x 3\n",
    BANNER + "3 3 -1\n",
    BANNER + "3 3 3\n1 1 1.0\n2 x 1\n",
    BANNER + "3 3 2\n1 1\n",
    BANNER + "3 3 2\n4 1 1.0\n",
    BANNER + "3 3 2\n0 1 1.0\n",
    BANNER + "3 3 2\n-1 2 3\n",
    BANNER + "3 3 2\n1.5 2 3\n",
    BANNER + "3 3 3\n1 1 1.0\n2 2 2.0\n",
    BANNER + "3 3 1\n1 1 1e\n",
    BANNER + "3 3 1\n1 1 inf\n",
    BANNER + "3 3 1\n1 1 nan\n",
    BANNER + "3 3 1\n1 1 1e400\n",
    BANNER + "3 3 1\n1 1 .\n",
    BANNER + "3 3 1\n 1 1 1.0\n%x\n",  # leading blank: fine; then EOF? no: 1 entry declared -> valid
    "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n1 2\n",
    BANNER + "3 3 2\r\n1 1 1.0\r\n",
]


def _ours(text: str):
    b = text.encode()
    h = _abi.tcs_csr()
    rc = _abi.load().tcs_matrix_market_parse(b, len(b), C.byref(h), None)
    msg = _abi.load().tcs_last_error().decode()
    if rc == _abi.TCS_OK:
        _abi.load().tcs_csr_free_host(C.byref(h))
    return rc, msg


def _ref(text: str):
    try:
        O.Ref.parse_matrix_market(text)
        return None
    except ValueError as e:
        return str(e)


pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


@pytest.mark.parametrize("i", range(len(BAD_MTX)))
def test_matrix_market_errors_match_reference(i):
    text = BAD_MTX[i]
    want = _ref(text)
    rc, msg = _ours(text)
    if want is None:  # valid input: the host parse passes and the GPU assembly is reached
        assert rc != _abi.TCS_ERR_PARSE, msg
    else:
        assert rc == _abi.TCS_ERR_PARSE, (rc, msg)
        assert msg == want


def _big_body(n_lines, bad_at=None, declared=None, extra_bad_after=False):
    rng = np.random.default_rng(3)
    r = rng.integers(1, 5001, n_lines)
    c = rng.integers(1, 5001, n_lines)
    lines = [f"{a} {b} {0.5 * (k % 7)}" for k, (a, b) in enumerate(zip(r, c))]
    if bad_at is not None:
        lines[bad_at] = "1 1 oops"
    if extra_bad_after:
        lines.append("garbage line")
    d = n_lines if declared is None else declared
    return BANNER + "% generated\n" + f"5000 5000 {d}\n" + "\n".join(lines) + "\n"


@pytest.mark.parametrize("bad_at", [0, 7, 150_000, 299_999])
def test_matrix_market_error_line_across_chunks(bad_at):
    """The body is tokenised in parallel chunks; the reported line number is
    the file's (banner + comment + size line + entry index)."""
    text = _big_body(300_000, bad_at=bad_at)
    rc, msg = _ours(text)
    assert rc == _abi.TCS_ERR_PARSE
    assert msg == f"line {bad_at + 4}: entry value missing" == _ref(text)


def test_matrix_market_short_file_across_chunks():
    text = _big_body(300_000, declared=300_001)
    rc, msg = _ours(text)
    assert rc == _abi.TCS_ERR_PARSE and msg == _ref(text)


def test_matrix_market_missing_file():
    h = _abi.tcs_csr()
    rc = _abi.load().tcs_matrix_market_read(b"/nonexistent/x.mtx", C.byref(h), None)
    assert rc == _abi.TCS_ERR_PARSE
    assert _abi.load().tcs_last_error().decode() == "cannot open '/nonexistent/x.mtx'"


# ---------------------------------------------------------------- MEBC
def _container(rows=16, cols=16, vh=8, k=8, prec=0, rp=(0, 1, 2), ci=(3, 4), vals=None, magic=b"MEBC", version=1):
    vals = [1.0] * (vh * len(ci)) if vals is None else vals
    b = magic + struct.pack("<IQQIIB", version, rows, cols, vh, k, prec)
    for arr, fmt in ((rp, "I"), (ci, "I"), (vals, "f")):
        b += struct.pack("<I", len(arr)) + struct.pack(f"<{len(arr)}{fmt}", *arr)
    return b


BAD_MEBC = [
    b"",
    b"MEB",
    b"XEBC" + b"\0" * 64,
    _container(version=2),
    _container()[:20],
    _container()[:-3],
    _container(prec=2),
    _container(rp=(0, 1)),                 # wrong length
    _container(rp=(1, 1, 2)),              # must start at 0
    _container(rp=(0, 2, 1)),              # nondecreasing
    _container(rp=(0, 1, 3)),              # end != nv
    _container(vals=[1.0] * 3),            # values length
    _container(ci=(3, 16)),                # column out of range
    _container(rp=(0, 2, 2), ci=(5, 5)),   # ascending within a window
]


@pytest.mark.parametrize("i", range(len(BAD_MEBC)))
def test_container_errors_match_reference(tmp_path, i):
    path = tmp_path / "x.mebc"
    path.write_bytes(BAD_MEBC[i])
    with pytest.raises(ValueError) as ex:
        O.Ref.read_mebcrs(path)
    h = _abi.tcs_mebcrs()
    rc = _abi.load().tcs_mebcrs_read(str(path).encode(), C.byref(h), None)
    assert rc == _abi.TCS_ERR_FORMAT
    assert _abi.load().tcs_last_error().decode() == str(ex.value)


def test_container_missing_file():
    h = _abi.tcs_mebcrs()
    assert _abi.load().tcs_mebcrs_read(b"/nonexistent/x.mebc", C.byref(h), None) == _abi.TCS_ERR_IO
