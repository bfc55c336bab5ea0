"""GPU parity: the sm_100a kernels (through the C-ABI) against the
reference's own outputs (golden hashes from oracle/_ref) and the pinned CPU
oracle.  Bar: bit-exact for the ME-BCRS arrays and for small-integer inputs
(ref generate.hpp:13-18 makes every product and sum exact); rel-L2 <= 1e-2
(FP16) / 1e-3 (TF32) for real-valued inputs (BASELINE.json north star).
"""
import numpy as np
import pytest
import torch

import cases
import oracle as O

pytestmark = pytest.mark.gpu

T = None  # paper_2412_11007_b200.tcsparse, imported lazily (needs the built .so)
F16, F32 = 0, 1
REL_TOL = {0: 1e-2, 1: 1e-3}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    global T
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_11007_b200.tcsparse as tcs

    T = tcs


def dev_csr(m: O.Csr):
    return T.CsrMatrix(m.rows, m.cols, torch.from_numpy(m.row_ptr.view(np.int32)).cuda(),
                       torch.from_numpy(m.col_idx.view(np.int32)).cuda(), torch.from_numpy(m.values).cuda())


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den else 1.0)


def check_case(case, rec, value_dtype, path="auto", mapping=None):
    for p in case.precisions:
        if p == 1 and value_dtype == F16:
            continue
        tag = "fp16" if p == 0 else "tf32"
        me = T.encode_mebcrs(dev_csr(case.csr), T.Precision(p), value_dtype)
        rp, ci, v = me.to_host()
        assert cases.sha(rp) == rec[f"me_{tag}"]["rp_sha"], case.name
        assert cases.sha(ci) == rec[f"me_{tag}"]["ci_sha"], case.name
        ref_me = O.encode_mebcrs(case.csr, p)  # pinned == reference (test_oracle.py)
        if value_dtype == F32:
            assert cases.sha(rp, ci, v) == rec[f"me_{tag}"]["sha"], case.name
        else:  # binary16 storage == the reference's round_to_fp16 of its values
            assert np.array_equal(v.view(np.uint32), O.round_array(ref_me.values, 0).view(np.uint32)), case.name
        cfg = T.KernelConfig(T.Precision(p))
        scfg = T.KernelConfig(T.Precision(p), path=path if (p == 0 and value_dtype == F16) else "auto")
        if mapping is not None:
            scfg.mapping = mapping
        if case.B is not None:
            for dense in ([torch.from_numpy(case.B).cuda()] +
                          ([torch.from_numpy(case.B).cuda().half()] if p == 0 else [])):
                res = T.spmm(me, dense, scfg)
                got = res.output.cpu().numpy()
                assert cases.sha(got) == rec[f"spmm_{tag}"]["sha"], (case.name, dense.dtype)
                assert res.counters.mma_invocations == rec[f"spmm_{tag}"]["mma"]
        if case.A is not None:
            ops = T.SddmmOperands(me, torch.from_numpy(case.A).cuda(), torch.from_numpy(case.Bt).cuda())
            res = T.sddmm(ops, cfg)
            out = res.output.to_host()[2]
            assert cases.sha(out) == rec[f"sddmm_{tag}"]["sha"], case.name
            assert res.counters.mma_invocations == rec[f"sddmm_{tag}"]["mma"]
            if case.D is not None:  # pipeline closure: SDDMM output drives SpMM (ref tests/test_kernels.cpp:313)
                chained = T.spmm(res.output, torch.from_numpy(case.D).cuda(), cfg).output.cpu().numpy()
                assert cases.sha(chained) == rec[f"chain_{tag}"]["sha"], case.name
        me.free()


@pytest.mark.parametrize("value_dtype", [F32, F16])
def test_known_answer_cases(golden, value_dtype):
    for case in cases.kat_cases():
        check_case(case, golden["cases"][case.name], value_dtype)


@pytest.mark.parametrize("value_dtype", [F32, F16])
def test_acceptance2_replay(golden, value_dtype):
    """tests/acceptance.cpp criterion 2: 200 seeded matrices, both precisions, bit-exact."""
    params = cases.acceptance2_params()
    for i in range(200):
        check_case(cases.acceptance2_case(i, params), golden["cases"][f"acc2_{i:03d}"], value_dtype)


@pytest.mark.parametrize("path", ["mma_sync", "tcgen05"])
def test_spmm_instruction_paths_bit_exact(golden, path):
    """Both SpMM instruction paths (warp mma.sync vs TMA-gather + tcgen05) on
    the replayed acceptance matrices and C1, FP16 with binary16 values."""
    params = cases.acceptance2_params()
    for i in range(0, 200, 3):
        check_case(cases.acceptance2_case(i, params), golden["cases"][f"acc2_{i:03d}"], F16, path)
    for case in cases.kat_cases():
        check_case(case, golden["cases"][case.name], F16, path)
    check_case(cases.c1_case(False), golden["cases"]["c1"], F16, path)


@pytest.mark.parametrize("value_dtype", [F32, F16])
def test_direct_mapping_replay(golden, value_dtype):
    """ThreadMapping::direct runs the direct-mapping ablation kernel (FP16);
    results must equal the reference's, exactly as for coalesced
    (ref tests/acceptance.cpp:103-104)."""
    params = cases.acceptance2_params()
    for i in range(1, 200, 3):
        check_case(cases.acceptance2_case(i, params), golden["cases"][f"acc2_{i:03d}"], value_dtype,
                   mapping=T.ThreadMapping.direct)
    check_case(cases.c1_case(False), golden["cases"]["c1"], value_dtype, mapping=T.ThreadMapping.direct)


def test_acceptance6_replay(golden):
    """tests/acceptance.cpp criterion 6: 100 SDDMM triples + chained SpMM."""
    params = cases.acceptance6_params()
    for i in range(100):
        check_case(cases.acceptance6_case(i, params), golden["cases"][f"acc6_{i:03d}"], F32)


@pytest.mark.parametrize("value_dtype", [F32, F16])
def test_config1_small_int_bit_exact(golden, value_dtype):
    c = cases.c1_case(False)
    check_case(c, golden["cases"]["c1"], value_dtype)


@pytest.mark.parametrize("p", [0, 1])
def test_config1_real_mode_tolerance(golden, p):
    """C1/C2 with uniform [-1,1) values: rel-L2 vs the reference's fp32 result."""
    c = cases.c1_case(True)
    me_ref = O.encode_mebcrs(c.csr, p)
    me = T.encode_mebcrs(dev_csr(c.csr), T.Precision(p))
    cfg = T.KernelConfig(T.Precision(p))
    got = T.spmm(me, torch.from_numpy(c.B).cuda(), cfg).output.cpu().numpy()
    want = O.spmm(me_ref, c.B)
    assert cases.sha(want) == golden["cases"]["c1_real"][f"spmm_{'fp16' if p == 0 else 'tf32'}"]["sha"]
    err = rel_l2(got, want)
    assert err <= REL_TOL[p], err
    assert err < 1e-5  # only summation order differs from the reference
    out = T.sddmm(T.SddmmOperands(me, torch.from_numpy(c.A).cuda(), torch.from_numpy(c.Bt).cuda()), cfg)
    err2 = rel_l2(out.output.to_host()[2], O.sddmm(me_ref, c.A, c.Bt))
    assert err2 <= REL_TOL[p] and err2 < 1e-5, err2


@pytest.mark.parametrize("p", [0, 1])
def test_rounding_exhaustive_on_device(p):
    """Every binary32 bit pattern: device RNE (__float2half_rn / cvt.rn.tf32)
    == the reference's round_to_fp16 / round_to_tf32.
    The reference formula is restated with torch integer ops on the GPU and
    pinned to the oracle on a random sample first."""

    def ref_round(bits: torch.Tensor) -> torch.Tensor:  # int64 bit patterns -> int64 result bits
        sign = bits & 0x80000000
        mag = bits & 0x7FFFFFFF
        rne = lambda b: (b + 0xFFF + ((b >> 13) & 1)) & ~0x1FFF  # noqa: E731
        if p == 1:
            return torch.where((bits & 0x7F800000) == 0x7F800000, bits, rne(bits) & 0xFFFFFFFF)
        x = (bits & 0xFFFFFFFF).to(torch.int32).view(torch.float32)
        sub = (torch.round(x.double() * 2.0**24) / 2.0**24).float().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        out = torch.where(mag >= 0x38800000, sign | rne(mag), sub)
        out = torch.where(mag >= 0x477FF000, sign | 0x7F800000, out)
        return torch.where(mag >= 0x7F800000, bits, out)

    rng = np.random.default_rng(7)
    sample = rng.integers(0, 2**32, 100000, dtype=np.uint64).astype(np.uint32)
    want = O.round_array(sample.view(np.float32), p).view(np.uint32)
    got = ref_round(torch.from_numpy(sample.astype(np.int64)).cuda()).cpu().numpy().astype(np.uint32)
    nan = np.isnan(sample.view(np.float32))
    assert np.array_equal(got[~nan], want[~nan])
    chunk = 1 << 28
    for start in range(0, 1 << 32, chunk):
        bits = torch.arange(start, start + chunk, dtype=torch.int64, device="cuda")
        x = (bits & 0xFFFFFFFF).to(torch.int32).view(torch.float32)
        dev = T.round_values(x, T.Precision(p)).view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        ref = ref_round(bits)
        isnan = torch.isnan(x)
        bad = (dev != ref) & ~isnan
        assert int(bad.sum()) == 0, f"mismatch at {int(bits[bad][0]):#x}"
        assert bool(torch.isnan(dev.to(torch.int32).view(torch.float32))[isnan].all())


def test_reference_error_taxonomy():
    """ref tests/test_kernels.cpp:127-137, 303-312."""
    ident = O.Csr.from_coords(8, 8, [(i, i, 1.0) for i in range(8)])
    me = T.encode_mebcrs(dev_csr(ident), T.Precision.fp16)
    dense = torch.ones(8, 16, device="cuda")
    with pytest.raises(T.ArgumentError):
        T.spmm(me, dense, T.KernelConfig(T.Precision.fp16, 16))
    with pytest.raises(T.ArgumentError):
        T.spmm(me, dense, T.KernelConfig(T.Precision.tf32, 8))
    with pytest.raises(T.ShapeError):
        T.spmm(me, torch.ones(9, 16, device="cuda"), T.KernelConfig())
    mask = T.encode_mebcrs(dev_csr(O.generate_random_sparse(16, 16, 0.2, 81)), T.Precision.fp16)
    a, b = torch.ones(16, 8, device="cuda"), torch.ones(16, 8, device="cuda")
    with pytest.raises(T.ArgumentError):
        T.sddmm(T.SddmmOperands(mask, a, b), T.KernelConfig(T.Precision.tf32))
    with pytest.raises(T.ShapeError):
        T.sddmm(T.SddmmOperands(mask, torch.ones(15, 8, device="cuda"), b))
    with pytest.raises(T.ShapeError):
        T.sddmm(T.SddmmOperands(mask, torch.ones(16, 9, device="cuda"), b))
    # malformed CSR -> FormatError (ref matrix.hpp:31-48)
    bad = T.CsrMatrix(2, 4, torch.tensor([0, 2, 2], dtype=torch.int32, device="cuda"),
                      torch.tensor([3, 1], dtype=torch.int32, device="cuda"), torch.ones(2, device="cuda"))
    with pytest.raises(T.FormatError):
        T.encode_mebcrs(bad, T.Precision.fp16)


def check_baseline16(case, rec, value_dtype):
    """16x1 non-swapped ablation (ref spmm.hpp:187-257) on the 16-row-window
    layout: partition bit-exact with ref partition_windows(m, 16, k), values
    laid out like the 8-row format, output and counters == the reference's
    spmm_baseline16 (golden hashes)."""
    for p in case.precisions:
        if p == 1 and value_dtype == F16:
            continue
        tag = "fp16" if p == 0 else "tf32"
        r16 = rec[f"b16_{tag}"]
        m16 = T.encode_mebcrs(dev_csr(case.csr), T.Precision(p), value_dtype, vector_height=16)
        rp, ci, v = m16.to_host()
        assert cases.sha(rp, ci) == r16["part_sha"], case.name
        ref16 = O.encode_mebcrs(case.csr, p, vector_height=16)  # pinned by test_oracle.py
        want_v = ref16.values if value_dtype == F32 else O.round_array(ref16.values, 0)
        assert np.array_equal(v.view(np.uint32), want_v.view(np.uint32)), case.name
        for dense in ([torch.from_numpy(case.B).cuda()] + ([torch.from_numpy(case.B).cuda().half()] if p == 0 else [])):
            res = T.spmm_baseline16(m16, dense)
            assert cases.sha(res.output.cpu().numpy()) == r16["sha"], (case.name, dense.dtype)
            assert res.counters.mma_invocations == r16["mma"]
        m16.free()


@pytest.mark.parametrize("value_dtype", [F32, F16])
def test_baseline16_matches_reference(golden, value_dtype):
    params = cases.acceptance2_params()
    todo = [c for c in cases.kat_cases() if c.B is not None]
    todo += [cases.acceptance2_case(i, params) for i in range(0, 200, 2)]
    todo += [cases.c1_case(False)]
    for c in todo:
        check_baseline16(c, golden["cases"][c.name], value_dtype)


def test_baseline16_errors():
    """ref spmm.hpp:190-191: the baseline needs vector height 16."""
    m = O.generate_random_sparse(40, 24, 0.2, 3)
    m16 = T.encode_mebcrs(dev_csr(m), T.Precision.fp16, vector_height=16)
    m8 = T.encode_mebcrs(dev_csr(m), T.Precision.fp16)
    B = torch.ones(24, 16, device="cuda")
    with pytest.raises(T.ArgumentError):
        T.spmm_baseline16(m16, B, T.KernelConfig(T.Precision.fp16, vector_height=8))
    with pytest.raises(T.ArgumentError):
        T.spmm_baseline16(m8, B, T.KernelConfig(T.Precision.fp16, vector_height=16))
    with pytest.raises(T.ArgumentError):  # a 16-high handle is not a swap8 operand
        T.spmm(m16, B, T.KernelConfig(T.Precision.fp16))
    with pytest.raises(T.ShapeError):
        T.spmm_baseline16(m16, torch.ones(23, 16, device="cuda"))
    with pytest.raises(T.ArgumentError):
        T.encode_mebcrs(dev_csr(m), T.Precision.fp16, vector_height=4)


def check_srbcrs(case, rec, value_dtype):
    """SR-BCRS padded ablation format (ref srbcrs.hpp:40-72): arrays
    bit-exact with ref encode_srbcrs, and spmm over it (ref spmm.hpp:181)
    == the compact-format result == the reference's (golden hashes)."""
    for p in case.precisions:
        if p == 1 and value_dtype == F16:
            continue
        tag = "fp16" if p == 0 else "tf32"
        r_sr = rec[f"sr_{tag}"]
        me = T.encode_mebcrs(dev_csr(case.csr), T.Precision(p), value_dtype)
        for sr in (T.encode_srbcrs(dev_csr(case.csr), T.Precision(p), value_dtype), T.encode_srbcrs(me)):
            assert sr.num_padded == r_sr["np"], case.name
            pairs, ci, v = sr.to_host()
            want = O.encode_srbcrs(O.encode_mebcrs(case.csr, p))  # pinned by test_oracle.py
            assert np.array_equal(pairs, want.row_pointer_pairs) and np.array_equal(ci, want.column_indices)
            want_v = want.values if value_dtype == F32 else O.round_array(want.values, 0)
            assert np.array_equal(v.view(np.uint32), want_v.view(np.uint32)), case.name
            if value_dtype == F32:
                assert cases.sha(pairs, ci, v) == r_sr["sha"], case.name
            # ref decode_srbcrs (srbcrs.hpp:74-90) == decode of the compact format
            drp, dci, dv = sr.decode()
            want_rp, want_ci, want_v = me.decode()
            assert np.array_equal(drp, want_rp) and np.array_equal(dci, want_ci), case.name
            assert np.array_equal(dv.view(np.uint32), want_v.view(np.uint32)), case.name
            if case.B is not None:
                res = T.spmm(sr, torch.from_numpy(case.B).cuda(), T.KernelConfig(T.Precision(p)))
                assert cases.sha(res.output.cpu().numpy()) == r_sr["spmm_sha"], case.name
                assert res.counters.mma_invocations == r_sr["mma"]
            sr.free()
        me.free()


@pytest.mark.parametrize("value_dtype", [F32, F16])
def test_srbcrs_matches_reference(golden, value_dtype):
    params = cases.acceptance2_params()
    todo = list(cases.kat_cases())
    todo += [cases.acceptance2_case(i, params) for i in range(0, 200, 3)]
    todo += [cases.c1_case(False)]
    for c in todo:
        check_srbcrs(c, golden["cases"][c.name], value_dtype)


def test_srbcrs_padding_inert_and_upload():
    """Padded vectors gather the reference's absent (zero) row: non-finite B
    rows cannot leak into the result; host upload of the reference's own
    arrays runs the same kernel; malformed pairs -> FormatError."""
    m = O.generate_random_sparse(300, 200, 0.03, 11, real=True)
    B = O.generate_random_dense(200, 48, 12, real=True)
    B[0, :] = np.nan  # column 0 may be gathered by real vectors only
    for p in (0, 1):
        me = T.encode_mebcrs(dev_csr(m), T.Precision(p), F32)
        cfg = T.KernelConfig(T.Precision(p))
        want = T.spmm(me, torch.from_numpy(B).cuda(), cfg).output.cpu().numpy()
        ref = O.Ref.encode_srbcrs(m, p)
        sr = T.SrBcrsMatrix.from_host(m.rows, m.cols, p, ref.row_pointer_pairs, ref.column_indices, ref.values)
        got = T.spmm(sr, torch.from_numpy(B).cuda(), cfg).output.cpu().numpy()
        assert np.array_equal(got, want, equal_nan=True)
        ref_c, _ = O.Ref.spmm_srbcrs(ref, np.nan_to_num(B, nan=0.0))
        got0 = T.spmm(sr, torch.from_numpy(np.nan_to_num(B, nan=0.0)).cuda(), cfg).output.cpu().numpy()
        assert rel_l2(got0, ref_c) < 1e-5
        bad = ref.row_pointer_pairs.copy()
        bad[1] += 1  # window 0 no longer a multiple of k
        with pytest.raises(T.FormatError):
            T.SrBcrsMatrix.from_host(m.rows, m.cols, p, bad, ref.column_indices, ref.values)
        with pytest.raises(T.ShapeError):
            T.spmm(sr, torch.ones(199, 16, device="cuda"), cfg)
        with pytest.raises(T.ArgumentError):
            T.spmm(sr, torch.ones(200, 16, device="cuda"), T.KernelConfig(T.Precision(1 - p)))


def test_sddmm_static_mask_matches_reference(golden):
    """TCS_CFG_STATIC_MASK (liveness bytes cached in the work list) gives the
    reference's SDDMM bit for bit, incl. explicit 0.0 / -0.0 mask entries
    (kat_zero_mask) and both value storages; the cache follows the values
    (an SDDMM output used as the next mask gets its own liveness)."""
    params = cases.acceptance6_params()
    todo = [c for c in cases.kat_cases() if c.A is not None]
    todo += [cases.acceptance6_case(i, params) for i in range(0, 100, 4)]
    for case in todo:
        rec = golden["cases"][case.name]
        for p in case.precisions:
            tag = "fp16" if p == 0 else "tf32"
            for vdt in ((F32, F16) if p == 0 else (F32,)):
                me = T.encode_mebcrs(dev_csr(case.csr), T.Precision(p), vdt)
                ops = T.SddmmOperands(me, torch.from_numpy(case.A).cuda(), torch.from_numpy(case.Bt).cuda())
                cfg = T.KernelConfig(T.Precision(p), static_mask=True)
                for _ in range(2):
                    res = T.sddmm(ops, cfg)
                    assert cases.sha(res.output.to_host()[2]) == rec[f"sddmm_{tag}"]["sha"], (case.name, vdt)
                # the output (same structure and work list, other values) as the next mask
                ops2 = T.SddmmOperands(res.output, ops.a, ops.b_t)
                want = T.sddmm(ops2, T.KernelConfig(T.Precision(p))).output.to_host()[2]
                got = T.sddmm(ops2, cfg).output.to_host()[2]
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), case.name
                again = T.sddmm(ops, cfg).output.to_host()[2]
                assert cases.sha(again) == rec[f"sddmm_{tag}"]["sha"], case.name
                me.free()


def test_decode_matches_reference(golden):
    """GPU decode_mebcrs (ref mebcrs.hpp:116-138) == the reference's decode
    of the same ME-BCRS: stored zeros (fill, explicit 0.0 / -0.0 entries)
    dropped, rows sorted; binary16 storage decodes its rounded values."""
    params = cases.acceptance2_params()
    todo = list(cases.kat_cases()) + [cases.acceptance2_case(i, params) for i in range(0, 200, 5)]
    for case in todo:
        for p in case.precisions:
            for vdt in ((F32, F16) if p == 0 else (F32,)):
                me = T.encode_mebcrs(dev_csr(case.csr), T.Precision(p), vdt)
                rp, ci, v = me.decode()
                ref_me = O.encode_mebcrs(case.csr, p)  # pinned == reference
                if vdt == F16:
                    ref_me = O.MeBcrs(ref_me.rows, ref_me.cols, p, ref_me.row_pointers, ref_me.column_indices,
                                      O.round_array(ref_me.values, 0))
                want = O.Ref.decode_mebcrs(ref_me)
                assert np.array_equal(rp, want.row_ptr) and np.array_equal(ci, want.col_idx), (case.name, p, vdt)
                assert np.array_equal(v.view(np.uint32), want.values.view(np.uint32)), (case.name, p, vdt)
                me.free()


@pytest.mark.parametrize("p", [0, 1])
def test_shapes_strides_and_alignment(p):
    """Dense widths across the slab boundaries (N = 1 .. 300: 32/64/128-
    feature slabs, 3 slabs past 256), strided and misaligned dense operands
    (the padding/conversion path), strided outputs, and SDDMM inner
    dimensions across the pass boundaries (F = 1 .. 100) -- all bit-exact
    against the oracle on small-integer inputs."""
    m = O.generate_random_sparse(203, 157, 0.06, 41)
    ref = O.encode_mebcrs(m, p)
    for vdt in ((F32, F16) if p == 0 else (F32,)):
        me = T.encode_mebcrs(dev_csr(m), T.Precision(p), vdt)
        cfg = T.KernelConfig(T.Precision(p))
        for n in (1, 7, 33, 64, 100, 130, 256, 300):
            B = O.generate_random_dense(m.cols, n, 40 + n)
            want = O.spmm(ref, B)
            Bd = torch.from_numpy(B).cuda()
            variants = [Bd]
            wide = torch.zeros(m.cols, n + 5, device="cuda")
            wide[:, :n] = Bd
            variants.append(wide[:, :n])  # row stride n + 5
            flat = torch.zeros(m.cols * n + 1, device="cuda")
            flat[1:] = Bd.flatten()
            variants.append(flat[1:].view(m.cols, n))  # misaligned by 4 bytes
            if p == 0:
                variants.append(Bd.half())
            for dense in variants:
                out = torch.full((m.rows, n + 3), 7.0, device="cuda")
                got = T.spmm(me, dense, cfg, out=out[:, :n]).output
                assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32)), (n, dense.stride())
                assert torch.all(out[:, n:] == 7.0), "wrote past the output columns"
        for f in (1, 8, 13, 33, 64, 65, 100):
            A = O.generate_random_dense(m.rows, f, 70 + f)
            Bt = O.generate_random_dense(m.cols, f, 80 + f)
            got = T.sddmm(T.SddmmOperands(me, torch.from_numpy(A).cuda(), torch.from_numpy(Bt).cuda()),
                          cfg).output.to_host()[2]
            assert np.array_equal(got.view(np.uint32), O.sddmm(ref, A, Bt).view(np.uint32)), f
        me.free()


def test_tiny_mask_values_sampled_with_binary16_storage(golden):
    """Mask values that are nonzero in f32 but round to a binary16 zero
    (1e-10, -3e-9, 2^-25, -1e-12) are sampled by the reference SDDMM, which
    tests the f32 value (ref sddmm.hpp:131).  With binary16 value storage the
    encoder keeps exact liveness bytes for them: the SDDMM (default and
    static-mask), the fused SDDMM -> row softmax and a re-prepared handle
    all sample them; an SDDMM output used as the next mask does not inherit
    them (its own values decide)."""
    case = next(c for c in cases.kat_cases() if c.name == "kat_tiny_mask")
    rec = golden["cases"][case.name]
    me = T.encode_mebcrs(dev_csr(case.csr), T.Precision.fp16, F16)
    ops = T.SddmmOperands(me, torch.from_numpy(case.A).cuda(), torch.from_numpy(case.Bt).cuda())
    for static in (False, True, False):
        out = T.sddmm(ops, T.KernelConfig(T.Precision.fp16, static_mask=static)).output.to_host()[2]
        assert cases.sha(out) == rec["sddmm_fp16"]["sha"], static
    # 6 live slots (the explicit 0.0 is stored but not sampled)
    assert int(np.count_nonzero(out)) == 6
    sm = T.sddmm_row_softmax(ops, 1.0, T.KernelConfig(T.Precision.fp16)).to_host()[2]
    assert int(np.count_nonzero(sm)) == 6 and np.all(np.isfinite(sm))
    import ctypes
    from paper_2412_11007_b200 import _abi
    assert _abi.load().tcs_mebcrs_prepare(ctypes.byref(me._h),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    out = T.sddmm(ops, T.KernelConfig(T.Precision.fp16)).output.to_host()[2]
    assert cases.sha(out) == rec["sddmm_fp16"]["sha"]
    me.free()


@pytest.mark.parametrize("n", [64, 96, 128, 200, 256])
def test_tf32_packed_operand_equals_f32_gather(n):
    """TF32 SpMM on the 2.5-byte repacked dense operand (hi 16 bits + a
    nibble of the next mantissa bits) == the f32-gather kernel bit for bit,
    on real values with full 10-bit TF32 mantissas, signed zeros, subnormals,
    inf and large magnitudes; both within the north-star tolerance of the
    oracle (the reference's sequential binary32 sums)."""
    rng = np.random.default_rng(n)
    m = O.generate_random_sparse(1203, 997, 0.05, 90 + n, real=True)
    B = rng.standard_normal((m.cols, n)).astype(np.float32) * np.float32(3.7)
    B[::97, ::5] = np.float32(1e-39)   # subnormal
    B[::89, 1::7] = -0.0
    B[::83, 2::11] = np.float32(3e30)
    me = T.encode_mebcrs(dev_csr(m), T.Precision.tf32)
    Bd = torch.from_numpy(B).cuda()
    packed = T.spmm(me, Bd, T.KernelConfig(T.Precision.tf32)).output.cpu().numpy()
    plain = T.spmm(me, Bd, T.KernelConfig(T.Precision.tf32, tf32_f32_gather=True)).output.cpu().numpy()
    assert np.array_equal(packed.view(np.uint32), plain.view(np.uint32))
    want = O.spmm_csr_rows(m, B, 1)
    assert rel_l2(packed, want) < 1e-3
    Bd[5, 3] = float("inf")
    packed = T.spmm(me, Bd, T.KernelConfig(T.Precision.tf32)).output.cpu().numpy()
    plain = T.spmm(me, Bd, T.KernelConfig(T.Precision.tf32, tf32_f32_gather=True)).output.cpu().numpy()
    assert np.array_equal(packed.view(np.uint32), plain.view(np.uint32))
    me.free()
