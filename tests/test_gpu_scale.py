"""GPU parity beyond the reference's desk-scale cases.

* mid-size power-law graphs and hub-heavy windows (split windows, the
  512-thread and global-scratch merge paths) against the pinned oracle,
  bit-exact with small-integer values;
* BASELINE config 3 at full size (Reddit-shaped, ~115 M nnz) through
  size-independent properties: ME-BCRS row pointers equal an independent
  torch count of distinct (window, column) pairs; integer-valued SpMM equals
  an independent exact fp32 product (every partial sum is an integer below
  2^24, so any summation order gives the same bits); SDDMM equals direct
  dot products at sampled positions;
* the host-buffer entry points (value semantics of the reference API).
"""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
T = None
G = None


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    global T, G
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_11007_b200.graphs as graphs
    import paper_2412_11007_b200.tcsparse as tcs

    T, G = tcs, graphs


def to_oracle(rows, cols, rp, ci, v):
    return O.Csr(rows, cols, rp.cpu().numpy().view(np.uint32), ci.cpu().numpy().view(np.uint32), v.cpu().numpy())


def dev(m: O.Csr):
    return T.CsrMatrix(m.rows, m.cols, torch.from_numpy(m.row_ptr.view(np.int32)).cuda(),
                       torch.from_numpy(m.col_idx.view(np.int32)).cuda(), torch.from_numpy(m.values).cuda())


def hub_matrix(cols=40000):
    """Windows of every size class: tiny, > 2048 entries (512-thread merge),
    > 12288 entries (hub), plus windows longer than the SpMM segment (split +
    deterministic reduction) and empty windows.  cols > 819,200 takes the
    wide-column-space paths (window_sort_big: shared-memory merges, hub
    windows on a global-memory bitmap) instead of the shared-memory bitmap."""
    rng = np.random.default_rng(11)
    rows = 96
    per_row = [3] * 8 + [400] * 8 + [0] * 8 + [2500] * 8 + [12] * 8 + [6000] * 8 + [1] * 8 + [0] * 8 + \
              [900] * 8 + [30000] * 8 + [5] * 8 + [2] * 8
    rp = np.zeros(rows + 1, np.uint32)
    ci_list = []
    for r, d in enumerate(per_row):
        c = np.sort(rng.choice(cols, size=d, replace=False)).astype(np.uint32)
        ci_list.append(c)
        rp[r + 1] = rp[r] + d
    ci = np.concatenate(ci_list)
    vals = rng.integers(1, 5, ci.size).astype(np.float32) * rng.choice([-1, 1], ci.size).astype(np.float32)
    return O.Csr(rows, cols, rp, ci, vals)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [0, 1])
def test_hub_windows_wide_column_space_bit_exact(p):
    """R-MAT-like column space (> the shared-memory bitmap): the medium
    windows merge in shared memory, the hub windows (> 12288 entries) are
    ranked on a CTA-private global-memory bitmap."""
    m = hub_matrix(cols=1_000_003)
    ref = O.encode_mebcrs(m, p)
    for vd in (1, 0) if p == 0 else (1,):
        me = T.encode_mebcrs(dev(m), T.Precision(p), vd)
        rp, ci, v = me.to_host()
        assert np.array_equal(rp, ref.row_pointers) and np.array_equal(ci, ref.column_indices)
        if vd == 1:
            assert np.array_equal(v.view(np.uint32), ref.values.view(np.uint32))
    B = O.generate_random_dense(m.cols, 64, 5)
    want = O.spmm(ref, B)
    me = T.encode_mebcrs(dev(m), T.Precision(p), 1)
    got = T.spmm(me, torch.from_numpy(B).cuda(), T.KernelConfig(T.Precision(p))).output.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("p", [0, 1])
@pytest.mark.parametrize("n", [128, 64, 32, 256, 40, 200])
def test_hub_windows_bit_exact(p, n):
    m = hub_matrix()
    ref = O.encode_mebcrs(m, p)
    me = T.encode_mebcrs(dev(m), T.Precision(p), 1)
    rp, ci, v = me.to_host()
    assert np.array_equal(rp, ref.row_pointers) and np.array_equal(ci, ref.column_indices)
    assert np.array_equal(v.view(np.uint32), ref.values.view(np.uint32))
    B = O.generate_random_dense(m.cols, n, 5)
    want = O.spmm(ref, B)
    got = T.spmm(me, torch.from_numpy(B).cuda(), T.KernelConfig(T.Precision(p))).output.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if p == 0:  # binary16 storage: both instruction paths, f16 and f32 dense operands
        me16 = T.encode_mebcrs(dev(m), T.Precision(p), 0)
        for path in ("mma_sync", "tcgen05"):
            for dense in (torch.from_numpy(B).cuda(), torch.from_numpy(B).cuda().half()):
                got = T.spmm(me16, dense, T.KernelConfig(T.Precision(p), path=path)).output.cpu().numpy()
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (path, dense.dtype)
    A = O.generate_random_dense(m.rows, 32, 6)
    Bt = O.generate_random_dense(m.cols, 32, 7)
    want_s = O.sddmm(ref, A, Bt)
    ops = T.SddmmOperands(me, torch.from_numpy(A).cuda(), torch.from_numpy(Bt).cuda())
    out = T.sddmm(ops, T.KernelConfig(T.Precision(p))).output.to_host()[2]
    assert np.array_equal(out.view(np.uint32), want_s.view(np.uint32))
    # TCS_CFG_STATIC_MASK: liveness bytes built on the first call, cached after
    for _ in range(2):
        out = T.sddmm(ops, T.KernelConfig(T.Precision(p), static_mask=True)).output.to_host()[2]
        assert np.array_equal(out.view(np.uint32), want_s.view(np.uint32))


@pytest.mark.parametrize("p", [0, 1])
def test_power_law_midsize_bit_exact(p):
    spec = G.GraphSpec("mid", 60_000, 3_000_000, alpha=1.2, cap=60.0, seed=5)
    rows, cols, rp, ci, v = G.power_law_csr(spec, values="int")
    m = to_oracle(rows, cols, rp, ci, v)
    ref = O.encode_mebcrs(m, p)
    me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, v), T.Precision(p))
    h_rp, h_ci, h_v = me.to_host()
    assert np.array_equal(h_rp, ref.row_pointers) and np.array_equal(h_ci, ref.column_indices)
    B = O.generate_random_dense(cols, 128, 9)
    Bd = torch.from_numpy(B).cuda()
    got = T.spmm(me, Bd.half() if p == 0 else Bd, T.KernelConfig(T.Precision(p))).output.cpu().numpy()
    want = O.spmm(ref, B)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # the pipelined host-buffer call (3 window-range chunks at 3 M nnz)
    import paper_2412_11007_b200._abi as abi

    csr = abi.tcs_csr(rows, cols, m.nnz, m.row_ptr.ctypes.data, m.col_idx.ctypes.data, m.values.ctypes.data)
    cfg = abi.tcs_kernel_config(p, 8, 1, 0)
    cnt = abi.tcs_counters()
    Ch = np.empty((rows, 128), np.float32)
    rc = abi.load().tcs_spmm_csr_host(C.byref(csr), p, B.ctypes.data, 128, Ch.ctypes.data, C.byref(cfg),
                                      C.byref(cnt), None)
    assert rc == 0, abi.load().tcs_last_error()
    assert np.array_equal(Ch.view(np.uint32), want.view(np.uint32))
    assert cnt.mma_invocations == O.count_mma_spmm(ref, 128)


def test_config3_full_size_properties():
    rows, cols, rp, ci, v = G.power_law_csr(G.C3_REDDIT, values="int")
    nnz = ci.numel()
    assert 100e6 < nnz < 130e6
    me = T.encode_mebcrs(T.CsrMatrix(rows, cols, rp, ci, v), T.Precision.fp16)
    # (1) row pointers == independent count of distinct (window, column) pairs
    r_of = torch.repeat_interleave(torch.arange(rows, device="cuda"), (rp[1:] - rp[:-1]).long())
    keys = torch.unique((r_of // 8) * cols + ci.long())
    counts = torch.bincount(keys // cols, minlength=me.num_windows)
    del keys
    import paper_2412_11007_b200._abi as abi

    nv = me.num_vectors
    rp_host = np.empty(me.num_windows + 1, np.uint32)
    ci_host = np.empty(nv, np.uint32)
    assert abi.load().tcs_mebcrs_download(C.byref(me._h), rp_host.ctypes.data, ci_host.ctypes.data, None,
                                          C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    want_rp = np.concatenate([[0], np.cumsum(counts.cpu().numpy())]).astype(np.uint32)
    assert np.array_equal(rp_host, want_rp)
    # (1b) decode(encode(A)) == A (no value is 0, so nothing is dropped)
    drp, dci, dv = me.decode()
    assert np.array_equal(drp, rp.cpu().numpy().view(np.uint32))
    assert np.array_equal(dci, ci.cpu().numpy().view(np.uint32))
    assert np.array_equal(dv, v.cpu().numpy())
    del drp, dci, dv
    # (2) integer SpMM == exact independent product
    B = G.dense(cols, 128, 3, values="int", dtype=torch.float32)
    got = T.spmm(me, B.half(), T.KernelConfig()).output
    A = torch.sparse_csr_tensor(rp.long(), ci.long(), v, size=(rows, cols))
    assert torch.equal(got, A @ B)
    del got, A, B
    # (3) SDDMM at 20k sampled vectors == direct dot products where the
    # pattern has an entry, 0 elsewhere (ref sddmm.hpp:131)
    Af = G.dense(rows, 32, 4, values="int", dtype=torch.float32)
    Bt = G.dense(cols, 32, 5, values="int", dtype=torch.float32)
    out_vals = torch.empty(8 * nv, dtype=torch.float32, device="cuda")
    T.sddmm(T.SddmmOperands(me, Af, Bt), T.KernelConfig(), out_values=out_vals)
    vid = np.sort(np.random.default_rng(3).choice(nv, 20000, replace=False))
    check_sddmm_samples(rows, cols, rp, ci, rp_host, ci_host, Af, Bt, out_vals, vid, k=8)
    me.free()


def check_sddmm_samples(rows, cols, rp, ci, rp_host, ci_host, Af, Bt, out_vals, vid, k):
    """SDDMM output at the stored vectors `vid` == direct dot products of
    A's rows and Bt's rows where the CSR has an entry, 0 elsewhere."""
    r_of = torch.repeat_interleave(torch.arange(rows, device="cuda"), (rp[1:] - rp[:-1]).long())
    entry_keys = r_of * cols + ci.long()  # CSR order == sorted
    del r_of
    w = np.searchsorted(rp_host, vid, side="right") - 1
    vl = vid - rp_host[w]
    nvw = rp_host[w + 1] - rp_host[w]
    b, j = vl // k, vl % k
    width = np.minimum(k, nvw - k * b)
    col = ci_host[vid].astype(np.int64)
    for r in range(8):
        row = 8 * w.astype(np.int64) + r
        ok = row < rows
        pos = 8 * (rp_host[w].astype(np.int64) + k * b) + r * width + j
        got_r = out_vals[torch.from_numpy(pos).cuda()].cpu().numpy()
        q = torch.from_numpy(np.where(ok, row, 0) * cols + col).cuda()
        idx = torch.searchsorted(entry_keys, q).clamp(max=entry_keys.numel() - 1)
        present = ((entry_keys[idx] == q).cpu().numpy()) & ok
        dots = (Af[torch.from_numpy(np.where(ok, row, 0)).cuda()] * Bt[torch.from_numpy(col).cuda()]).sum(1)
        want_r = np.where(present, dots.cpu().numpy(), 0.0).astype(np.float32)
        assert np.array_equal(got_r, want_r), r


def test_config5_full_size_64bit_offsets():
    """BASELINE config 5 at full size (R-MAT scale 23, ~250 M nnz): the
    FP16 value array holds 1.9e9 elements (3.9 GB, byte offsets past 2^31)
    and the TF32 one 7.8 GB (past 2^32).  Integer-valued SpMM (both
    precisions, N = 32) == an independent exact fp32 product; SDDMM at
    vectors sampled from the top end of the value array == direct dots."""
    rows, cols, rp, ci, v = G.rmat_csr(G.C5_RMAT, values="int")
    nnz = ci.numel()
    assert 230e6 < nnz < 280e6
    csr = T.CsrMatrix(rows, cols, rp, ci, v)
    A = torch.sparse_csr_tensor(rp.long(), ci.long(), v, size=(rows, cols))
    B = G.dense(cols, 32, 3, values="int", dtype=torch.float32)
    want = A @ B
    del A
    import paper_2412_11007_b200._abi as abi

    for p in (T.Precision.fp16, T.Precision.tf32):
        me = T.encode_mebcrs(csr, p)
        # FP16: 3.9 GB of values (byte offsets past 2^31); TF32: 7.8 GB (past 2^32)
        assert 8 * me.num_vectors * (2 if p == T.Precision.fp16 else 4) > (1 << (31 if p == T.Precision.fp16 else 32))
        got = T.spmm(me, B.half() if p == T.Precision.fp16 else B, T.KernelConfig(p)).output
        assert torch.equal(got, want), p
        del got
        if p == T.Precision.tf32:
            nv = me.num_vectors
            rp_host = np.empty(me.num_windows + 1, np.uint32)
            ci_host = np.empty(nv, np.uint32)
            assert abi.load().tcs_mebcrs_download(C.byref(me._h), rp_host.ctypes.data, ci_host.ctypes.data, None,
                                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
            Af = G.dense(rows, 32, 4, values="int", dtype=torch.float32)
            Bt = G.dense(cols, 32, 5, values="int", dtype=torch.float32)
            out_vals = torch.empty(8 * nv, dtype=torch.float32, device="cuda")
            T.sddmm(T.SddmmOperands(me, Af, Bt), T.KernelConfig(p), out_values=out_vals)
            rng = np.random.default_rng(5)
            vid = np.sort(rng.choice(np.arange(nv - nv // 10, nv), 20000, replace=False))
            check_sddmm_samples(rows, cols, rp, ci, rp_host, ci_host, Af, Bt, out_vals, vid, k=4)
            del out_vals, Af, Bt
        me.free()
        torch.cuda.empty_cache()


def test_host_entry_points_match_device_path():
    m = O.generate_random_sparse(300, 200, 0.05, 3)
    B = O.generate_random_dense(200, 48, 4)
    lib = __import__("paper_2412_11007_b200._abi", fromlist=["x"]).load()
    cfg = __import__("paper_2412_11007_b200._abi", fromlist=["x"]).tcs_kernel_config(0, 8, 1, 0)
    for p in (0, 1):
        cfg.precision = p
        ref = O.encode_mebcrs(m, p)
        want = O.spmm(ref, B)
        Cm = np.empty((300, 48), np.float32)
        rc = lib.tcs_spmm_host(300, 200, p, ref.row_pointers.ctypes.data, ref.column_indices.ctypes.data,
                               ref.values.ctypes.data, B.ctypes.data, 200, 48, Cm.ctypes.data, C.byref(cfg), None,
                               None)
        assert rc == 0 and np.array_equal(Cm.view(np.uint32), want.view(np.uint32))
        csr = __import__("paper_2412_11007_b200._abi", fromlist=["x"]).tcs_csr(
            300, 200, m.nnz, m.row_ptr.ctypes.data, m.col_idx.ctypes.data, m.values.ctypes.data)
        C2 = np.empty((300, 48), np.float32)
        rc = lib.tcs_spmm_csr_host(C.byref(csr), p, B.ctypes.data, 48, C2.ctypes.data, C.byref(cfg), None, None)
        assert rc == 0 and np.array_equal(C2.view(np.uint32), want.view(np.uint32))
        A = O.generate_random_dense(300, 20, 5)
        Bt = O.generate_random_dense(200, 20, 6)
        out = np.empty(8 * ref.nv, np.float32)
        rc = lib.tcs_sddmm_host(300, 200, p, ref.row_pointers.ctypes.data, ref.column_indices.ctypes.data,
                                ref.values.ctypes.data, A.ctypes.data, 300, 20, Bt.ctypes.data, 200, 20,
                                out.ctypes.data, C.byref(cfg), None, None)
        assert rc == 0 and np.array_equal(out.view(np.uint32), O.sddmm(ref, A, Bt).view(np.uint32))


@pytest.mark.parametrize("p", [0, 1])
@pytest.mark.parametrize("n", [128, 64, 32, 200])
def test_hub_windows_baseline16_bit_exact(p, n):
    """16x1 ablation on hub windows (split segments + ordered reduction)."""
    m = hub_matrix()
    ref = O.encode_mebcrs(m, p, vector_height=16)
    m16 = T.encode_mebcrs(dev(m), T.Precision(p), 1, vector_height=16)
    rp, ci, v = m16.to_host()
    assert np.array_equal(rp, ref.row_pointers) and np.array_equal(ci, ref.column_indices)
    assert np.array_equal(v.view(np.uint32), ref.values.view(np.uint32))
    B = O.generate_random_dense(m.cols, n, 5)
    want = O.spmm(ref, B)
    got = T.spmm_baseline16(m16, torch.from_numpy(B).cuda()).output.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if p == 0:
        m16h = T.encode_mebcrs(dev(m), T.Precision(p), 0, vector_height=16)
        got = T.spmm_baseline16(m16h, torch.from_numpy(B).cuda().half()).output.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("n", [128, 64, 32, 200])
@pytest.mark.parametrize("vdt", [0, 1])
def test_direct_mapping_bit_identical(n, vdt):
    """ThreadMapping::direct (the paper's ablation kernel) == coalesced, bit
    for bit (ref tests/acceptance.cpp:103-104), incl. split hub windows."""
    m = hub_matrix()
    ref = O.encode_mebcrs(m, 0)
    me = T.encode_mebcrs(dev(m), T.Precision.fp16, vdt)
    B = O.generate_random_dense(m.cols, n, 9)
    want = O.spmm(ref, B)
    for dense in (torch.from_numpy(B).cuda(), torch.from_numpy(B).cuda().half()):
        cfg = T.KernelConfig(T.Precision.fp16, mapping=T.ThreadMapping.direct)
        got = T.spmm(me, dense, cfg).output.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("defect", ["descending", "out_of_range"])
def test_pipelined_host_call_reports_late_chunk_format_errors(defect):
    """tcs_spmm_csr_host encodes its chunks without host round trips; a
    malformed row in the LAST chunk must still come back as the reference's
    FormatError (ref matrix.hpp validate), not as garbage output."""
    import paper_2412_11007_b200._abi as abi

    spec = G.GraphSpec("mid", 60_000, 3_000_000, alpha=1.2, cap=60.0, seed=7)
    rows, cols, rp, ci, v = G.power_law_csr(spec, values="int")
    m = to_oracle(rows, cols, rp, ci, v)
    ci_h = m.col_idx.copy()
    r = rows - 3  # a row of the last chunk with >= 2 entries
    while m.row_ptr[r + 1] - m.row_ptr[r] < 2:
        r -= 1
    e = int(m.row_ptr[r])
    if defect == "descending":
        ci_h[e], ci_h[e + 1] = ci_h[e + 1], ci_h[e]
    else:
        ci_h[int(m.row_ptr[r + 1]) - 1] = cols + 5
    csr = abi.tcs_csr(rows, cols, m.nnz, m.row_ptr.ctypes.data, ci_h.ctypes.data, m.values.ctypes.data)
    cfg = abi.tcs_kernel_config(0, 8, 1, 0)
    B = O.generate_random_dense(cols, 32, 3)
    Ch = np.empty((rows, 32), np.float32)
    lib = abi.load()
    rc = lib.tcs_spmm_csr_host(C.byref(csr), 0, B.ctypes.data, 32, Ch.ctypes.data, C.byref(cfg), None, None)
    assert rc == abi.TCS_ERR_FORMAT
    msg = lib.tcs_last_error().decode() if isinstance(lib.tcs_last_error(), bytes) else str(lib.tcs_last_error())
    assert ("ascending" if defect == "descending" else "out of range") in msg


@pytest.mark.gpu
@pytest.mark.parametrize("n", [128, 256, 200, 64, 32])
def test_f32_value_storage_equals_binary16_storage(n):
    """FP16 SpMM on f32-stored values (the drop-in adapter's bit-exact
    storage; the 128-feature kernels convert them to binary16 at the MMA)
    equals the same SpMM on binary16-stored values bit for bit: both round
    with RNE (ref precision.hpp round_to_fp16), so the MMA operands are the
    same.  Real values, hub windows (split items), residue steps."""
    import paper_2412_11007_b200._abi as abi

    spec = G.GraphSpec("mid_real", 60_000, 3_000_000, alpha=1.2, cap=60.0, seed=11)
    rows, cols, rp, ci, v = G.power_law_csr(spec, values="real")
    csr = T.CsrMatrix(rows, cols, rp, ci, v)
    m32 = T.encode_mebcrs(csr, T.Precision.fp16, abi.TCS_DTYPE_F32)
    m16 = T.encode_mebcrs(csr, T.Precision.fp16, abi.TCS_DTYPE_F16)
    B = G.dense(cols, n, 3, values="real", dtype=torch.float16)
    cfg = T.KernelConfig(T.Precision.fp16)
    got32 = T.spmm(m32, B, cfg).output
    got16 = T.spmm(m16, B, cfg).output
    assert torch.equal(got32.view(torch.int32), got16.view(torch.int32))
    m32.free()
    m16.free()
