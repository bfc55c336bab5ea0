"""Pins the CPU oracle (oracle/oracle.cpp) against the reference.

(a) golden.json -- hashes of the reference's own outputs (tests/golden/
    make_golden.py ran the unmodified reference headers via oracle/_ref);
(b) the reference's known-answer tests, restated with their literal values;
(c) when oracle/_ref is present, a live differential check on random inputs.
"""
import math
import struct

import numpy as np
import pytest

import cases
import oracle as O


def _f(bits):
    return struct.unpack("<f", struct.pack("<I", bits))[0]


# tests/test_tcu_emu.cpp:68-98
@pytest.mark.parametrize("x,p,want", [
    (1.0, 0, 1.0), (1.0, 1, 1.0), (-3.0, 0, -3.0), (0.0, 0, 0.0),
    (2049.0, 0, 2048.0), (2051.0, 0, 2052.0),
    (1.0 + 2**-11, 1, 1.0), (1.0 + 2**-10, 1, 1.0 + 2**-10), (1.0 + 2**-11 + 2**-23, 1, 1.0 + 2**-10),
    (65504.0, 0, 65504.0), (65519.0, 0, 65504.0), (65520.0, 0, math.inf), (-70000.0, 0, -math.inf),
    (math.inf, 0, math.inf), (2**-24, 0, 2**-24), (2**-25, 0, 0.0), (1.5 * 2**-25, 0, 2**-24),
])
def test_rounding_known_answers(x, p, want):
    got = O.round_fp16(x) if p == 0 else O.round_tf32(x)
    assert got == want


def test_rounding_nan_passthrough():
    assert math.isnan(O.round_fp16(math.nan)) and math.isnan(O.round_tf32(math.nan))


def test_rounding_random_bits_match_golden(golden):
    g = golden["rounding"]
    rng = np.random.default_rng(g["seed"])
    xs = rng.integers(0, 2**32, size=g["n"], dtype=np.uint64).astype(np.uint32).view(np.float32)
    f16 = np.array([O.round_fp16(float(x)) for x in xs], np.float32)
    t32 = np.array([O.round_tf32(float(x)) for x in xs], np.float32)
    assert cases.sha(f16) == g["fp16_sha"]
    assert cases.sha(t32) == g["tf32_sha"]


def check_case(case, rec):
    m = case.csr
    assert cases.sha(m.row_ptr, m.col_idx, m.values) == rec["csr"], "generator restatement drifted"
    for key in ("B", "A", "Bt", "D"):
        arr = getattr(case, key)
        if arr is not None:
            assert cases.sha(arr) == rec[key]["sha"], key
    for p in case.precisions:
        tag = "fp16" if p == 0 else "tf32"
        me = O.encode_mebcrs(m, p)
        assert me.nv == rec[f"me_{tag}"]["nv"]
        assert cases.sha(me.row_pointers, me.column_indices, me.values) == rec[f"me_{tag}"]["sha"]
        if case.B is not None:
            assert cases.sha(O.spmm(me, case.B)) == rec[f"spmm_{tag}"]["sha"]
            assert O.count_mma_spmm(me, case.B.shape[1]) == rec[f"spmm_{tag}"]["mma"]
            m16 = O.encode_mebcrs(m, p, vector_height=16)
            assert m16.nv == rec[f"b16_{tag}"]["nv"]
            assert cases.sha(m16.row_pointers, m16.column_indices) == rec[f"b16_{tag}"]["part_sha"]
            assert cases.sha(O.spmm(m16, case.B)) == rec[f"b16_{tag}"]["sha"]
            blocks = int(sum((int(m16.row_pointers[w + 1] - m16.row_pointers[w]) + m16.k - 1) // m16.k
                             for w in range(m16.num_windows)))
            assert blocks * ((case.B.shape[1] + 7) // 8) == rec[f"b16_{tag}"]["mma"]
        sr = O.encode_srbcrs(me)
        r_sr = rec[f"sr_{tag}"]
        assert sr.column_indices.shape[0] == r_sr["np"]
        assert cases.sha(sr.row_pointer_pairs, sr.column_indices, sr.values) == r_sr["sha"]
        if case.B is not None:  # ref spmm(SrBcrs) == spmm(MeBcrs) bit for bit (spmm.hpp:179-180)
            assert r_sr["spmm_sha"] == rec[f"spmm_{tag}"]["sha"] and r_sr["mma"] == rec[f"spmm_{tag}"]["mma"]
        if case.A is not None:
            out = O.sddmm(me, case.A, case.Bt)
            assert cases.sha(out) == rec[f"sddmm_{tag}"]["sha"]
            assert O.count_mma_sddmm(me, case.A.shape[1]) == rec[f"sddmm_{tag}"]["mma"]
            if case.D is not None:
                chained = O.MeBcrs(me.rows, me.cols, p, me.row_pointers, me.column_indices, out)
                assert cases.sha(O.spmm(chained, case.D)) == rec[f"chain_{tag}"]["sha"]


def test_kat_cases_match_golden(golden):
    for case in cases.kat_cases():
        check_case(case, golden["cases"][case.name])


def test_acceptance2_replay_matches_golden(golden):
    params = cases.acceptance2_params()
    for i in range(200):
        check_case(cases.acceptance2_case(i, params), golden["cases"][f"acc2_{i:03d}"])


def test_acceptance6_replay_matches_golden(golden):
    params = cases.acceptance6_params()
    for i in range(100):
        check_case(cases.acceptance6_case(i, params), golden["cases"][f"acc6_{i:03d}"])


@pytest.mark.parametrize("real", [False, True])
def test_config1_matches_golden(golden, real):
    c = cases.c1_case(real)
    check_case(c, golden["cases"][c.name])
    assert c.csr.nnz == 64899  # SURVEY §8 table (C1 nnz)


def test_me_layout_known_answers():
    # tests/test_formats.cpp:81-86: empty 32x32 -> row pointers {0,0,0,0,0}
    e = O.encode_mebcrs(O.Csr(32, 32, np.zeros(33, np.uint32), [], []), 0)
    assert list(e.row_pointers) == [0] * 5 and e.nv == 0
    # :88-98 identity layout: 64 values, diagonal ones
    ident = O.encode_mebcrs(O.Csr.from_coords(8, 8, [(i, i, 1.0) for i in range(8)]), 0)
    assert ident.values.shape == (64,)
    assert np.array_equal(ident.values.reshape(8, 8), np.eye(8, dtype=np.float32))
    # :116-124 residue block widths 8 then 1 (window of 9 vectors)
    coords = [(c % 8, c, float(c + 1)) for c in range(9)] + [(8 + c, c, 2.0) for c in range(3)]
    me = O.encode_mebcrs(O.Csr.from_coords(16, 16, coords), 0)
    assert list(me.row_pointers) == [0, 9, 12]
    # block 1 of window 0 has width 1: its 8 values are rows 0..7 of vector 8
    assert list(me.values[64:72]) == [9.0, 0, 0, 0, 0, 0, 0, 0]


def test_sddmm_skips_explicit_zero_mask():
    # entries (0,1)=1, (2,3)=0.0, (4,5)=-0.0; all-ones, F=4
    mz = O.Csr(8, 8, [0, 1, 1, 2, 2, 3, 3, 3, 3], [1, 3, 5], np.array([1.0, 0.0, -0.0], np.float32))
    for p in (0, 1):
        me = O.encode_mebcrs(mz, p)
        assert me.nv == 3
        out = O.sddmm(me, np.ones((8, 4), np.float32), np.ones((8, 4), np.float32))
        d = O.mebcrs_to_dense(O.MeBcrs(8, 8, p, me.row_pointers, me.column_indices, out))
        assert d[0, 1] == 4.0 and d[2, 3] == 0.0 and d[4, 5] == 0.0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_live_differential_against_reference():
    rng = np.random.default_rng(5)
    for t in range(6):
        rows, cols = int(rng.integers(1, 90)), int(rng.integers(1, 90))
        m = O.generate_random_sparse(rows, cols, float(rng.uniform(0.01, 0.5)), 100 + t, real=bool(t % 2))
        B = O.generate_random_dense(cols, int(rng.integers(1, 40)), 200 + t, real=bool(t % 2))
        for p in (0, 1):
            a, b = O.encode_mebcrs(m, p), O.Ref.encode_mebcrs(m, p)
            assert np.array_equal(a.values.view(np.uint32), b.values.view(np.uint32))
            assert np.array_equal(O.spmm(a, B).view(np.uint32), O.Ref.spmm(b, B)[0].view(np.uint32))


def _csr_form_matches(case, rec):
    m = case.csr
    for p in case.precisions:
        tag = "fp16" if p == 0 else "tf32"
        if case.B is not None:
            assert cases.sha(O.spmm_csr_rows(m, case.B, p)) == rec[f"spmm_{tag}"]["sha"], (case.name, p)
            rows = np.arange(m.rows)[::3]
            assert np.array_equal(O.spmm_csr_rows(m, case.B, p, rows).view(np.uint32),
                                  O.spmm_csr_rows(m, case.B, p)[rows].view(np.uint32))
        if case.A is not None:
            me = O.encode_mebcrs(m, p)
            dot, pos = O.sddmm_csr_rows(m, p, me.row_pointers, me.column_indices, case.A, case.Bt)
            assert not np.any(pos == np.iinfo(np.uint64).max)
            out = np.zeros(8 * me.nv, np.float32)
            out[pos.astype(np.int64)] = dot
            assert cases.sha(out) == rec[f"sddmm_{tag}"]["sha"], (case.name, p)


def test_csr_form_oracle_matches_golden(golden):
    """The CSR-form restatements used for the full-size (C3-C5) parity gates
    (orc_spmm_csr_rows / orc_sddmm_csr_rows) give the reference's bits on
    every golden case: KATs, the acceptance replays and C1 in both value
    modes."""
    todo = list(cases.kat_cases())
    p2, p6 = cases.acceptance2_params(), cases.acceptance6_params()
    todo += [cases.acceptance2_case(i, p2) for i in range(0, 200, 2)]
    todo += [cases.acceptance6_case(i, p6) for i in range(0, 100, 2)]
    todo += [cases.c1_case(False), cases.c1_case(True)]
    for case in todo:
        _csr_form_matches(case, golden["cases"][case.name])
