"""Ingest, containers, cost model and the CLI on the GPU path against the
reference itself:

* MatrixMarket text -> CSR (host tokeniser + GPU assembly) equals the
  reference's parse_matrix_market bit for bit, on the reference's grammar
  (general/symmetric, real/integer/pattern, comments, CRLF, duplicates,
  lines past the declared count) and on a multi-chunk file;
* MEBC containers written from the GPU encoding are byte-identical to the
  reference CLI's `convert --output`, and read back to the same arrays;
* tcsparse-b200 (the reference CLI on the B200 library) prints what the
  reference CLI prints -- convert, spmm (8x1 coalesced/direct, 16x1
  baseline), sddmm, stats (CSV/JSON, i.e. the GPU cost model == ref
  analyze_matrix), bench -- with the same exit codes.
"""
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2412_11007_b200", "tcsparse-b200")
T = None


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    global T
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not O.ref_available():
        pytest.skip("oracle/_ref missing")
    import paper_2412_11007_b200.tcsparse as tcs

    T = tcs


BANNER = "%%MatrixMarket matrix coordinate real general\n"
GOOD_MTX = [
    BANNER + "3 4 3\n1 1 1.5\n3 4 -2\n2 2 0\n",
    "%%MatrixMarket matrix coordinate integer general\n% c\n\n4 4 2\n4 4 7\n1 3 -3\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n5 5 4\n1 1\n2 1\n5 3\n4 4\n",
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 0.25\n3 3 1e-3\n3 1 -0.0\n",
    BANNER + "3 3 4\n1 1 1.0\n1 1 2.5\n% mid comment\n\n2 3 4\n2 3 -4\n",  # duplicates summed
    BANNER + "2 2 1\r\n1 2 3.25\r\n",
    BANNER + "2 2 1\n1 2 3\nthis line is never read\n",
    BANNER + "0 0 0\n",
    BANNER + "6 6 0\n",
    BANNER + "2 2 2\n1 1 +1.5e+1\n2 2 -.5\n",
    "%%MatrixMarket matrix coordinate real general extra tokens\n2 2 1 9\n1 1 1 7\n",
]


def _csr_equal(dev: "T.CsrMatrix", ref: O.Csr):
    assert (dev.rows, dev.cols) == (ref.rows, ref.cols)
    assert np.array_equal(dev.row_ptr.cpu().numpy().view(np.uint32), ref.row_ptr)
    assert np.array_equal(dev.col_idx.cpu().numpy().view(np.uint32), ref.col_idx)
    assert np.array_equal(dev.values.cpu().numpy().view(np.uint32), ref.values.view(np.uint32))


@pytest.mark.parametrize("i", range(len(GOOD_MTX)))
def test_matrix_market_parse_matches_reference(i):
    _csr_equal(T.parse_matrix_market(GOOD_MTX[i]), O.Ref.parse_matrix_market(GOOD_MTX[i]))


def test_matrix_market_large_multichunk():
    rng = np.random.default_rng(12)
    n = 400_000
    r, c = rng.integers(1, 20001, n), rng.integers(1, 30001, n)
    r[::97] = r[1::97][: len(r[::97])]  # some duplicate coordinates (pairs)
    c[::97] = c[1::97][: len(c[::97])]
    v = rng.integers(-8, 9, n) / 4.0
    text = BANNER + "% big\n" + f"20000 30000 {n}\n" + "".join(f"{a} {b} {x}\n" for a, b, x in zip(r, c, v))
    _csr_equal(T.parse_matrix_market(text), O.Ref.parse_matrix_market(text))


def test_matrix_market_write_roundtrip(tmp_path):
    m = O.generate_random_sparse(70, 50, 0.1, 5, real=True)
    dev = T.CsrMatrix(m.rows, m.cols, torch.from_numpy(m.row_ptr.view(np.int32)).cuda(),
                      torch.from_numpy(m.col_idx.view(np.int32)).cuda(), torch.from_numpy(m.values).cuda())
    path = tmp_path / "m.mtx"
    T.write_matrix_market(path, dev)
    back = O.Ref.parse_matrix_market(path.read_text())  # ref: parse maps it back to the identical CSR
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.col_idx, m.col_idx)
    assert np.array_equal(back.values.view(np.uint32), m.values.view(np.uint32))


def test_coo_to_csr_device_matches_reference():
    rng = np.random.default_rng(4)
    rows, cols, n = 300, 200, 5000
    r = rng.integers(0, rows, n).astype(np.uint32)
    c = rng.integers(0, cols, n).astype(np.uint32)
    v = (rng.integers(-5, 6, n) / 2.0).astype(np.float32)
    text = BANNER + f"{rows} {cols} {n}\n" + "".join(f"{a + 1} {b + 1} {x}\n" for a, b, x in zip(r, c, v))
    want = O.Ref.parse_matrix_market(text)
    import ctypes as C
    from paper_2412_11007_b200 import _abi

    dr, dc, dv = (torch.from_numpy(x.view(np.int32) if x.dtype == np.uint32 else x).cuda() for x in (r, c, v))
    h = _abi.tcs_csr()
    assert _abi.load().tcs_coo_to_csr(rows, cols, n, dr.data_ptr(), dc.data_ptr(), dv.data_ptr(), C.byref(h),
                                      None) == 0
    torch.cuda.synchronize()
    nnz = int(h.nnz)
    rp = torch.empty(rows + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
    vv = torch.empty(nnz, dtype=torch.float32, device="cuda")
    import glob

    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                  "libcudart.so*"))
    rt = C.CDLL(libs[0] if libs else "libcudart.so")
    for dst, src, nb in ((rp, h.row_ptr, 4 * (rows + 1)), (ci, h.col_idx, 4 * nnz), (vv, h.values, 4 * nnz)):
        assert rt.cudaMemcpy(C.c_void_p(dst.data_ptr()), C.c_void_p(src), C.c_size_t(nb), 3) == 0
    _abi.load().tcs_csr_free(C.byref(h), None)
    _csr_equal(T.CsrMatrix(rows, cols, rp, ci, vv), want)


# ------------------------------------------------------------- containers
def _write_mtx(path, m: O.Csr, pattern=False):
    lines = [f"%%MatrixMarket matrix coordinate {'pattern' if pattern else 'real'} general",
             f"{m.rows} {m.cols} {m.nnz}"]
    for r in range(m.rows):
        for p in range(m.row_ptr[r], m.row_ptr[r + 1]):
            lines.append(f"{r + 1} {m.col_idx[p] + 1}" + ("" if pattern else f" {repr(float(m.values[p]))}"))
    path.write_text("\n".join(lines) + "\n")


@pytest.fixture(scope="module")
def mtx_dir(tmp_path_factory):
    d = tmp_path_factory.mktemp("mtx")
    R = O.Ref
    _write_mtx(d / "a_uniform.mtx", R.generate_random_sparse(90, 70, 0.08, 1))
    _write_mtx(d / "b_dense_rows.mtx", R.generate_random_sparse(33, 300, 0.4, 2))
    _write_mtx(d / "c_tiny.mtx", R.generate_random_sparse(5, 9, 0.5, 3))
    _write_mtx(d / "d_pattern.mtx", R.generate_random_sparse(40, 40, 0.1, 4), pattern=True)
    (d / "e_empty.mtx").write_text(BANNER + "17 12 0\n")
    (d / "f_sym.mtx").write_text("%%MatrixMarket matrix coordinate integer symmetric\n12 12 5\n1 1 2\n7 3 -1\n"
                                 "12 11 3\n9 9 1\n5 2 4\n")
    return d


@pytest.fixture(scope="module")
def real_mtx(tmp_path_factory):
    d = tmp_path_factory.mktemp("real")
    _write_mtx(d / "r.mtx", O.Ref.generate_random_sparse(64, 48, 0.1, 7, real=True))
    return d / "r.mtx"


def _ours(*args):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


@pytest.mark.parametrize("prec", [0, 1])
def test_convert_container_byte_identical(mtx_dir, tmp_path, prec):
    for f in sorted(mtx_dir.glob("*.mtx")):
        ours, ref = tmp_path / f"o_{f.stem}.mebc", tmp_path / f"r_{f.stem}.mebc"
        got = _ours("convert", "--input", f, "--output", ours, "--precision", ["fp16", "tf32"][prec])
        want = O.Ref.cli("convert", input=f, output=ref, precision=prec)
        assert got == want, f
        assert ours.read_bytes() == ref.read_bytes(), f
        me = T.read_mebcrs(ours)
        r = O.Ref.read_mebcrs(ref)
        rp, ci, v = me.to_host()
        assert np.array_equal(rp, r.row_pointers) and np.array_equal(ci, r.column_indices)
        assert np.array_equal(v.view(np.uint32), r.values.view(np.uint32))


def test_convert_errors(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text(BANNER + "3 3 2\n1 1 1\n")
    assert _ours("convert", "--input", bad) == O.Ref.cli("convert", input=bad)
    assert _ours("convert", "--input", tmp_path / "none.mtx") == O.Ref.cli("convert", input=tmp_path / "none.mtx")


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("vh,mapping", [(8, 1), (8, 0), (16, 1)])
@pytest.mark.parametrize("n", [128, 40])
def test_spmm_cli_matches_reference(mtx_dir, prec, vh, mapping, n):
    for f in sorted(mtx_dir.glob("*.mtx")):
        got = _ours("spmm", "--input", f, "--n", n, "--vector", vh, "--precision", ["fp16", "tf32"][prec],
                    "--mapping", ["direct", "coalesced"][mapping], "--seed", 3, "--verify")
        want = O.Ref.cli("spmm", input=f, n=[n], vector_height=vh, precision=prec, mapping=mapping, seed=3,
                         verify=True)
        assert got == want, (f, got, want)


TOL_LINE = re.compile(r"max_abs_diff=([0-9.e+-]+)")


def _same_up_to_diff(got, want, tol):
    """Real-valued runs: identical text and verdict except the max_abs_diff
    figure (the tensor core sums in another order).  That figure is the
    error against the CLI's double-precision check of the UNROUNDED inputs,
    dominated by operand rounding, so it must track the reference's own
    figure; the reference itself exceeds the per-element TF32 threshold on
    some inputs (SURVEY §8(c) caveat, ref cli.hpp:67), and so must we then."""
    assert got[0] == want[0]
    assert TOL_LINE.sub("X", got[1]) == TOL_LINE.sub("X", want[1])
    assert TOL_LINE.sub("X", got[2]) == TOL_LINE.sub("X", want[2])
    mine = [float(x) for x in TOL_LINE.findall(got[1] + got[2])]
    theirs = [float(x) for x in TOL_LINE.findall(want[1] + want[2])]
    assert len(mine) == len(theirs)
    for x, y in zip(mine, theirs):
        assert abs(x - y) <= 0.05 * y + 0.05 * tol, (x, y)


@pytest.mark.parametrize("prec", [0, 1])
def test_spmm_cli_real_mode(real_mtx, prec):
    for vh in (8, 16):
        got = _ours("spmm", "--input", real_mtx, "--vector", vh, "--precision", ["fp16", "tf32"][prec], "--real",
                    "--verify")
        want = O.Ref.cli("spmm", input=real_mtx, vector_height=vh, precision=prec, real=True, verify=True)
        _same_up_to_diff(got, want, [1e-2, 1e-3][prec])


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("n", [32, 20])
def test_sddmm_cli_matches_reference(mtx_dir, tmp_path, prec, n):
    for f in sorted(mtx_dir.glob("*.mtx")):
        ours, ref = tmp_path / "o.mebc", tmp_path / "r.mebc"
        got = _ours("sddmm", "--input", f, "--n", n, "--precision", ["fp16", "tf32"][prec], "--seed", 5,
                    "--verify", "--output", ours)
        want = O.Ref.cli("sddmm", input=f, n=[n], precision=prec, seed=5, verify=True, output=ref)
        assert got == want, (f, got, want)
        assert ours.read_bytes() == ref.read_bytes(), f


@pytest.mark.parametrize("prec", [0, 1])
def test_sddmm_cli_real_mode(real_mtx, prec):
    got = _ours("sddmm", "--input", real_mtx, "--precision", ["fp16", "tf32"][prec], "--real", "--verify")
    want = O.Ref.cli("sddmm", input=real_mtx, precision=prec, real=True, verify=True)
    _same_up_to_diff(got, want, [1e-2, 1e-3][prec])


@pytest.mark.parametrize("fmt", ["csv", "json"])
@pytest.mark.parametrize("mapping", [1, 0])
def test_stats_cli_matches_reference(mtx_dir, tmp_path, fmt, mapping):
    """The GPU cost model (tcs_mebcrs_cost) == ref analyze_matrix, incl. the
    transaction model, for both vector heights, precisions and several N."""
    bad = tmp_path / "zz_bad.mtx"
    bad.write_text(BANNER + "3 3 1\n9 9 1\n")
    for f in sorted(mtx_dir.glob("*.mtx")):
        (tmp_path / f.name).write_text(f.read_text())
    args = ["--n", 16, "--n", 40, "--n", 128, "--n", 8, "--mapping", ["direct", "coalesced"][mapping],
            "--format", fmt]
    got = _ours("stats", "--dir", mtx_dir, *args)
    want = O.Ref.cli("stats", dir=mtx_dir, n=[16, 40, 128, 8], mapping=mapping, json=fmt == "json")
    assert got == want
    got = _ours("stats", "--dir", tmp_path, *args)  # includes the malformed file: skipped, exit 1
    want = O.Ref.cli("stats", dir=tmp_path, n=[16, 40, 128, 8], mapping=mapping, json=fmt == "json")
    assert got == want and got[0] == 1


def test_bench_cli_matches_reference(mtx_dir):
    for n in (64, 24):
        got = _ours("bench", "--dir", mtx_dir, "--n", n, "--seed", 2)
        want = O.Ref.cli("bench", dir=mtx_dir, n=[n], seed=2)
        assert got == want


@pytest.mark.parametrize("p", [0, 1])
@pytest.mark.parametrize("vh", [8, 16])
def test_cost_model_at_scale_consistent(p, vh):
    """Size-independent properties of the GPU cost model on a 3 M-nnz power-law
    graph: mma_count == blocks x tiles, zero fill == vh*nv - nnz, and the
    SpMM counters (all tiles) equal the extrapolated model when no segment
    merges happen (N >= 32)."""
    import paper_2412_11007_b200.graphs as G

    spec = G.GraphSpec("mid", 60_000, 3_000_000, alpha=1.2, cap=60.0, seed=5)
    rows, cols, rp, ci, v = G.power_law_csr(spec, values="int")
    csr = T.CsrMatrix(rows, cols, rp, ci, v)
    me = T.encode_mebcrs(csr, T.Precision(p), vector_height=vh)
    for n in (32, 128):
        c = T.mebcrs_cost(me, csr.nnz, n)
        tw = 16 if vh == 8 else 8
        assert c["mma_count"] == me.num_blocks * ((n + tw - 1) // tw)
        assert c["zero_fill"] == vh * me.num_vectors - csr.nnz
        assert c["padded_vectors"] == me.num_blocks * me.k
        assert c["transactions"] == c["exec_transactions"]
