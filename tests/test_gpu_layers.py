"""GPU: the GNN-layer glue (§8(f1)) -- row softmax over the ME-BCRS pattern,
the AGNN attention layer (SDDMM -> row softmax -> SpMM) and the GCN layer
(cuBLAS GEMM + SpMM), against plain PyTorch fp64 references of the same
ops (the reference library has no GNN layers)."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
T = L = None


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    global T, L
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_11007_b200.layers as layers
    import paper_2412_11007_b200.tcsparse as tcs

    T, L = tcs, layers


def dense_pattern(m: O.Csr):
    mask = np.zeros((m.rows, m.cols), bool)
    r = np.repeat(np.arange(m.rows), np.diff(m.row_ptr.astype(np.int64)))
    mask[r, m.col_idx] = m.values != 0
    return mask


def softmax_ref(S, mask, scale):
    S = torch.as_tensor(S, dtype=torch.float64) * scale
    M = torch.as_tensor(mask)
    S = S.masked_fill(~M, float("-inf"))
    P = torch.softmax(S, dim=1)
    return torch.nan_to_num(P, nan=0.0).masked_fill(~M, 0.0)


@pytest.mark.parametrize("p", [0, 1])
@pytest.mark.parametrize("out_f16", [False, True])
def test_row_softmax_matches_torch(p, out_f16):
    if p == 1 and out_f16:
        pytest.skip("TF32 stores f32")
    m = O.generate_random_sparse(203, 150, 0.08, 17, real=True)
    m.values[::7] = 0.0  # explicit zeros: stored vectors that are not live
    me = T.encode_mebcrs(T.CsrMatrix(m.rows, m.cols, torch.from_numpy(m.row_ptr.view(np.int32)).cuda(),
                                     torch.from_numpy(m.col_idx.view(np.int32)).cuda(),
                                     torch.from_numpy(m.values).cuda()), T.Precision(p), 1)
    A = torch.randn(m.rows, 24, device="cuda")
    Bt = torch.randn(m.cols, 24, device="cuda")
    scores = T.sddmm(T.SddmmOperands(me, A, Bt), T.KernelConfig(T.Precision(p))).output
    P = T.row_softmax(scores, me, 0.7, 0 if out_f16 else 1)
    rp, ci, sv = scores.to_host()
    pv = P.to_host()[2]
    # the kernel's own scores (a live score that is exactly 0 densifies to 0,
    # and the pattern mask keeps it live)
    S = O.mebcrs_to_dense(O.MeBcrs(m.rows, m.cols, p, rp, ci, sv))
    mask = dense_pattern(m)
    want = softmax_ref(S, mask, 0.7).numpy()
    got = O.mebcrs_to_dense(O.MeBcrs(m.rows, m.cols, p, rp, ci, pv))
    tol = 2e-3 if out_f16 or p == 0 else 1e-4
    assert np.abs(got - want).max() < tol
    assert np.all(got[~mask] == 0)
    # rows sum to 1 where the row has live entries
    sums = got.sum(1)
    live_rows = mask.any(1)
    assert np.allclose(sums[live_rows], 1.0, atol=5e-3)


def test_row_softmax_split_hub_windows():
    """Windows longer than the work-list segment: per-segment partials are
    merged (online softmax) before normalisation."""
    rng = np.random.default_rng(3)
    rows, cols = 40, 30000
    per_row = [25000] * 8 + [3] * 8 + [9000] * 8 + [0] * 8 + [100] * 8
    rp = np.zeros(rows + 1, np.uint32)
    cis = []
    for r, d in enumerate(per_row):
        cis.append(np.sort(rng.choice(cols, size=d, replace=False)).astype(np.uint32))
        rp[r + 1] = rp[r] + d
    ci = np.concatenate(cis)
    m = O.Csr(rows, cols, rp, ci, np.ones(ci.size, np.float32))
    me = T.encode_mebcrs(T.CsrMatrix(rows, cols, torch.from_numpy(rp.view(np.int32)).cuda(),
                                     torch.from_numpy(ci.view(np.int32)).cuda(),
                                     torch.from_numpy(m.values).cuda()), T.Precision.fp16, 1)
    assert me.max_window_vectors > 8 * 256  # several segments
    A = torch.randn(rows, 16, device="cuda")
    Bt = torch.randn(cols, 16, device="cuda")
    scores = T.sddmm(T.SddmmOperands(me, A, Bt), T.KernelConfig()).output
    P = T.row_softmax(scores, me, 2.0, 1)
    rph, cih, sv = scores.to_host()
    got = O.mebcrs_to_dense(O.MeBcrs(rows, cols, 0, rph, cih, P.to_host()[2]))
    S = O.mebcrs_to_dense(O.MeBcrs(rows, cols, 0, rph, cih, sv))
    want = softmax_ref(S, dense_pattern(m), 2.0).numpy()
    assert np.abs(got - want).max() < 1e-5 + 1e-4 * np.abs(want).max()


@pytest.mark.parametrize("p", [0, 1])
def test_agnn_layer_matches_dense_reference(p):
    n, F = 517, 32
    m = O.generate_random_sparse(n, n, 0.02, 23)
    rp = torch.from_numpy(m.row_ptr.view(np.int32)).cuda()
    ci = torch.from_numpy(m.col_idx.view(np.int32)).cuda()
    H = torch.randn(n, F, device="cuda")
    layer = L.AGNNLayer(n, rp, ci, beta=1.5, precision=T.Precision(p))
    got = layer(H).double().cpu()
    Hn = torch.nn.functional.normalize(H.double(), dim=1).cpu()
    mask = torch.as_tensor(dense_pattern(m) | (np.abs(O.Csr(n, n, m.row_ptr, m.col_idx, np.ones(m.nnz, np.float32))
                                                       .to_dense()) > 0))
    P = softmax_ref((Hn @ Hn.T).numpy(), mask.numpy(), 1.5)
    want = P @ H.double().cpu()
    err = (got - want).norm() / want.norm()
    assert err < (1e-2 if p == 0 else 1e-3), float(err)


@pytest.mark.parametrize("p", [0, 1])
def test_gcn_layer_matches_dense_reference(p):
    n, Fi, Fo = 700, 64, 128
    m = O.generate_random_sparse(n, n, 0.01, 29)
    rp = torch.from_numpy(m.row_ptr.view(np.int32)).cuda()
    ci = torch.from_numpy(m.col_idx.view(np.int32)).cuda()
    W = torch.randn(Fi, Fo, device="cuda") / Fi ** 0.5
    H = torch.randn(n, Fi, device="cuda")
    layer = L.GCNLayer(n, rp, ci, W.half() if p == 0 else W, precision=T.Precision(p))
    got = layer(H).double().cpu()
    A = torch.as_tensor(dense_pattern(O.Csr(n, n, m.row_ptr, m.col_idx, np.ones(m.nnz, np.float32)))).double()
    A = ((A + torch.eye(n, dtype=torch.float64)) > 0).double()
    dinv = A.sum(1).rsqrt()
    Ahat = dinv[:, None] * A * dinv[None, :]
    want = Ahat @ (H.double().cpu() @ W.double().cpu())
    err = (got - want).norm() / want.norm()
    assert err < (1e-2 if p == 0 else 1e-3), float(err)


def _fused_case(m, p, score_dt, out_dt, scale, F=24):
    me = T.encode_mebcrs(T.CsrMatrix(m.rows, m.cols, torch.from_numpy(m.row_ptr.view(np.int32)).cuda(),
                                     torch.from_numpy(m.col_idx.view(np.int32)).cuda(),
                                     torch.from_numpy(m.values).cuda()), T.Precision(p), 1)
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(m.rows, F, device="cuda", generator=g)
    Bt = torch.randn(m.cols, F, device="cuda", generator=g)
    ops = T.SddmmOperands(me, A, Bt)
    cfg = T.KernelConfig(T.Precision(p))
    fused = T.sddmm_row_softmax(ops, scale, cfg, score_dtype=score_dt, out_dtype=out_dt)
    static = T.sddmm_row_softmax(ops, scale, T.KernelConfig(T.Precision(p), static_mask=True),
                                 score_dtype=score_dt, out_dtype=out_dt)
    assert np.array_equal(static.to_host()[2].view(np.uint32), fused.to_host()[2].view(np.uint32))
    scores = T.sddmm(ops, cfg, out_dtype=score_dt).output
    two = T.row_softmax(scores, me, scale, out_dt)
    return fused.to_host()[2], two.to_host()[2]


@pytest.mark.parametrize("p,score_dt,out_dt", [(0, 1, 0), (0, 0, 0), (0, 1, 1), (0, 0, 1), (1, 1, 1)])
def test_fused_sddmm_softmax_equals_composition(p, score_dt, out_dt):
    """tcs_sddmm_row_softmax == tcs_sddmm -> tcs_mebcrs_row_softmax up to the
    order of the exp sums (max statistics are exact, dead slots exactly 0)."""
    m = O.generate_random_sparse(203, 150, 0.08, 17, real=True)
    m.values[::7] = 0.0  # stored but not live
    got, want = _fused_case(m, p, score_dt, out_dt, 0.7)
    tol = 2e-3 if out_dt == 0 else 1e-5
    assert np.abs(got - want).max() < tol


def test_fused_sddmm_softmax_split_windows():
    rng = np.random.default_rng(4)
    rows, cols = 40, 30000
    per_row = [25000] * 8 + [3] * 8 + [9000] * 8 + [0] * 8 + [100] * 8
    rp = np.zeros(rows + 1, np.uint32)
    cis = []
    for r, d in enumerate(per_row):
        cis.append(np.sort(rng.choice(cols, size=d, replace=False)).astype(np.uint32))
        rp[r + 1] = rp[r] + d
    ci = np.concatenate(cis)
    vals = np.ones(ci.size, np.float32)
    vals[::11] = 0.0
    m = O.Csr(rows, cols, rp, ci, vals)
    for p in (0, 1):
        got, want = _fused_case(m, p, 1, 1, 2.0, F=40)
        assert np.abs(got - want).max() < 1e-5 + 1e-4 * np.abs(want).max()


@pytest.mark.parametrize("f", [1, 12, 32, 45, 128, 130])
def test_rows_normalize_matches_torch(f):
    g = torch.Generator(device="cuda").manual_seed(f)
    h = torch.randn(1000, f, device="cuda", generator=g)
    h[7] = 0.0  # zero row: eps guard, like torch.nn.functional.normalize
    for dt in (torch.float16, torch.float32):
        hn, hc = T.rows_normalize(h, dt)
        want = torch.nn.functional.normalize(h, dim=1)
        assert torch.equal(hc, h.to(dt))
        assert (hn.float() - want).abs().max() < (1e-3 if dt == torch.float16 else 1e-6)


@pytest.mark.parametrize("n", [32, 20, 64, 128])
def test_agnn_aggregate_equals_materialised_softmax(n):
    """tcs_agnn_aggregate == spmm(sddmm_row_softmax(binary16 scores/P), Hc)
    bit for bit: the softmax applied in the SpMM's registers rounds exactly
    like the stored P.  Split hub windows, empty rows, dead (explicit-zero)
    mask entries, f32 and f16 operands, static and per-call mask."""
    rng = np.random.default_rng(n)
    rows = 3000
    per_row = rng.integers(0, 12, rows)
    per_row[8:16] = 2500   # a hub window longer than the work-list segment
    per_row[40:48] = 0     # an empty window
    rp = np.zeros(rows + 1, np.uint32)
    rp[1:] = np.cumsum(per_row)
    ci = np.concatenate([np.sort(rng.choice(rows, size=d, replace=False)) for d in per_row]).astype(np.uint32)
    vals = np.ones(ci.size, np.float32)
    vals[::13] = 0.0  # stored, not sampled
    m = O.Csr(rows, rows, rp, ci, vals)
    me = T.encode_mebcrs(T.CsrMatrix(rows, rows, torch.from_numpy(rp.view(np.int32)).cuda(),
                                     torch.from_numpy(ci.view(np.int32)).cuda(), torch.from_numpy(vals).cuda()),
                         T.Precision.fp16)
    g = torch.Generator(device="cuda").manual_seed(n)
    hn = torch.nn.functional.normalize(torch.randn(rows, 24, device="cuda", generator=g), dim=1)
    hc = torch.randn(rows, n, device="cuda", generator=g)
    for static in (False, True):
        cfg = T.KernelConfig(T.Precision.fp16, static_mask=static)
        for a_dt in (torch.float32, torch.float16):
            P = T.sddmm_row_softmax(T.SddmmOperands(me, hn.to(a_dt), hn.to(a_dt)), 0.9, cfg, score_dtype=0,
                                    out_dtype=0)
            want = T.spmm(P, hc.half(), T.KernelConfig()).output
            for h_dt in (torch.float32, torch.float16):
                got = T.agnn_aggregate(me, hn.to(a_dt), hc.to(h_dt), 0.9, cfg)
                assert torch.equal(got, want), (static, a_dt, h_dt)
    assert m.nnz == ci.size


def _attend_case(seed, rows, cols, hub=True):
    rng = np.random.default_rng(seed)
    per_row = rng.integers(0, 12, rows)
    if hub:
        per_row[8:16] = min(cols, 2500)  # a hub window longer than the work-list segment
    per_row[40:48] = 0                   # an empty window
    per_row[-1] = 0                      # an empty last row
    rp = np.zeros(rows + 1, np.uint32)
    rp[1:] = np.cumsum(per_row)
    ci = np.concatenate([np.sort(rng.choice(cols, size=d, replace=False)) for d in per_row]).astype(np.uint32)
    vals = np.ones(ci.size, np.float32)
    vals[::13] = 0.0  # stored, not sampled
    m = O.Csr(rows, cols, rp, ci, vals)
    me = T.encode_mebcrs(T.CsrMatrix(rows, cols, torch.from_numpy(rp.view(np.int32)).cuda(),
                                     torch.from_numpy(ci.view(np.int32)).cuda(), torch.from_numpy(vals).cuda()),
                         T.Precision.fp16)
    return m, me


def _attend_ref(m, h16, row0, scale, eps=1e-12):
    hf = h16.double().cpu()
    rn = 1.0 / hf.norm(dim=1).clamp_min(eps)
    hi = hf[row0:row0 + m.rows]
    S = (hi @ hf.T) * rn[row0:row0 + m.rows, None] * rn[None, :]
    P = softmax_ref(S, dense_pattern(m), scale)
    return (P @ hf).to(h16.device)


def _rel_l2(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))


@pytest.mark.parametrize("f", [32, 64])
def test_agnn_attend_matches_fp64(f):
    """Fused one-pass AGNN attention vs an fp64 dense PyTorch reference on
    the same f16 features: split hub windows, empty windows and rows, dead
    (explicit-zero) mask entries, static and per-call mask.  P is rounded to
    binary16 before the aggregation MMA, so the bound is FP16-level."""
    rows = 3000
    m, me = _attend_case(f, rows, rows)
    g = torch.Generator(device="cuda").manual_seed(f)
    h = torch.randn(rows, f, device="cuda", generator=g).half()
    want = _attend_ref(m, h, 0, 0.9)
    for static in (False, True):
        got = T.agnn_attend(me, h, 0.9, T.KernelConfig(T.Precision.fp16, static_mask=static))
        assert got.shape == (rows, f)
        assert _rel_l2(got, want) < 2e-3, (static, _rel_l2(got, want))
        assert torch.all(got[40:48] == 0) and torch.all(got[-1] == 0)


def test_agnn_attend_agrees_with_three_pass_aggregate():
    """The fused kernel and tcs_agnn_aggregate (SDDMM -> statistics ->
    softmax-applying SpMM, binary16 scores) compute the same layer."""
    rows, f = 3000, 32
    m, me = _attend_case(7, rows, rows)
    g = torch.Generator(device="cuda").manual_seed(7)
    h = torch.randn(rows, f, device="cuda", generator=g)
    hn, hc = T.rows_normalize(h, torch.float16)
    three = T.agnn_aggregate(me, hn, hc, 1.3)
    fused = T.agnn_attend(me, hc, 1.3)
    assert _rel_l2(fused, three) < 5e-3
    # only the pattern and liveness are read: a TF32-encoded mask (block
    # width 4) gives the same result
    me32 = T.encode_mebcrs(T.CsrMatrix(rows, rows, torch.from_numpy(m.row_ptr.view(np.int32)).cuda(),
                                       torch.from_numpy(m.col_idx.view(np.int32)).cuda(),
                                       torch.from_numpy(m.values).cuda()), T.Precision.tf32)
    assert _rel_l2(T.agnn_attend(me32, hc, 1.3), fused) < 1e-6


def test_agnn_attend_row_shard_and_large_scores():
    """A row shard (row0 > 0, mask rows < nodes, rows not a multiple of 8)
    and a large scale (scores up to +-40 in log2 units: the online
    max-rescaling must keep the sums finite)."""
    nodes, row0, rows, f = 4000, 1203, 1501, 32
    m, me = _attend_case(11, rows, nodes)
    g = torch.Generator(device="cuda").manual_seed(11)
    h = torch.randn(nodes, f, device="cuda", generator=g).half()
    for scale in (0.5, 30.0):
        want = _attend_ref(m, h, row0, scale)
        got = T.agnn_attend(me, h, scale, row0=row0)
        assert torch.isfinite(got).all()
        assert _rel_l2(got, want) < 4e-3, (scale, _rel_l2(got, want))


def test_agnn_attend_rejects_bad_arguments():
    rows = 64
    _, me = _attend_case(3, rows, rows, hub=False)
    h = torch.randn(rows, 48, device="cuda").half()
    with pytest.raises(T.ShapeError):
        T.agnn_attend(me, h)
    with pytest.raises(T.ArgumentError):
        T.agnn_attend(me, torch.randn(rows, 32, device="cuda"))
    with pytest.raises(T.ShapeError):
        T.agnn_attend(me, torch.randn(rows, 32, device="cuda").half(), row0=1)
