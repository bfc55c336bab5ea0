"""Seeded synthetic inputs of BASELINE.json's shapes, generated on the GPU
with torch (plumbing for bench.py and the large parity tests; no network
datasets exist here).

* ``power_law_csr`` -- Chung-Lu graph (both endpoints sampled in proportion
  to Pareto(alpha)+1 node weights, hub weights capped at ``cap`` x mean,
  duplicate edges merged): C3 "Reddit-shaped" (232,965 nodes, alpha 1.2,
  ~115 M nnz) and C4 "ogbn-products-shaped" (2,449,029 nodes, alpha 1.5).
* ``rmat_csr`` -- R-MAT (a, b, c, d) = (0.57, 0.19, 0.19, 0.05): C5.
* ``uniform_csr`` -- i.i.d. Bernoulli pattern (the shape of C1).

Values are either uniform [-1, 1) ("real") or small integers {-4..4}\\{0}
("int"), the reference's exactness trick (ref generate.hpp:13-18): with
them every FP16/TF32 product and fp32 sum is exact, so GPU results must be
bit-identical to the reference at any size.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class GraphSpec:
    name: str
    nodes: int
    target_nnz: int
    kind: str = "chung_lu"   # chung_lu | rmat | uniform
    alpha: float = 1.2
    cap: float = 60.0        # hub weight cap, x mean weight
    oversample: float = 1.10
    seed: int = 2412


C3_REDDIT = GraphSpec("reddit-shaped power law", 232_965, 115_000_000, alpha=1.2, cap=60.0, oversample=1.10)
C4_PRODUCTS = GraphSpec("ogbn-products-shaped power law", 2_449_029, 62_000_000, alpha=1.5, cap=400.0,
                        oversample=1.01)
C5_RMAT = GraphSpec("R-MAT scale 23", 1 << 23, 256_000_000, kind="rmat", oversample=1.04)


def _values(n, kind, gen, device):
    if kind == "int":
        m = torch.randint(0, 8, (n,), generator=gen, device=device)
        return torch.where(m < 4, m - 4, m - 3).to(torch.float32)
    return torch.rand(n, generator=gen, device=device) * 2.0 - 1.0


def _csr_from_edges(rows: torch.Tensor, cols: torch.Tensor, n_rows: int, n_cols: int):
    keys = torch.unique(rows.to(torch.int64) * n_cols + cols.to(torch.int64))  # sorted
    r = keys // n_cols
    c = (keys - r * n_cols).to(torch.int32)
    counts = torch.bincount(r, minlength=n_rows)
    row_ptr = torch.zeros(n_rows + 1, dtype=torch.int64, device=rows.device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    return row_ptr.to(torch.int32), c


def power_law_csr(spec: GraphSpec, values="real", device="cuda", rows_range=None):
    """Chung-Lu CSR on `device`; returns (rows, cols, row_ptr i32, col_idx i32, values f32)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed)
    n = spec.nodes
    u = torch.rand(n, generator=gen, device=device, dtype=torch.float64)
    w = (1.0 - u).pow(-1.0 / spec.alpha)
    w = torch.minimum(w, w.mean() * spec.cap)
    cdf = torch.cumsum(w / w.sum(), 0)
    cdf[-1] = 1.0
    m = int(spec.target_nnz * spec.oversample)
    rows = torch.empty(m, dtype=torch.int32, device=device)
    cols = torch.empty(m, dtype=torch.int32, device=device)
    chunk = 1 << 25
    for s in range(0, m, chunk):
        e = min(m, s + chunk)
        rows[s:e] = torch.searchsorted(cdf, torch.rand(e - s, generator=gen, device=device, dtype=torch.float64))
        cols[s:e] = torch.searchsorted(cdf, torch.rand(e - s, generator=gen, device=device, dtype=torch.float64))
    rows.clamp_(max=n - 1)
    cols.clamp_(max=n - 1)
    row_ptr, col_idx = _csr_from_edges(rows, cols, n, n)
    del rows, cols
    vals = _values(col_idx.numel(), values, gen, device)
    return n, n, row_ptr, col_idx, vals


def rmat_csr(spec: GraphSpec, values="real", device="cuda", abcd=(0.57, 0.19, 0.19, 0.05)):
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed)
    scale = int(spec.nodes).bit_length() - 1
    n = 1 << scale
    m = int(spec.target_nnz * spec.oversample)
    a, b, c, _ = abcd
    rows = torch.empty(m, dtype=torch.int32, device=device)
    cols = torch.empty(m, dtype=torch.int32, device=device)
    chunk = 1 << 25
    for s in range(0, m, chunk):
        e = min(m, s + chunk)
        r = torch.zeros(e - s, dtype=torch.int32, device=device)
        q = torch.zeros(e - s, dtype=torch.int32, device=device)
        for bit in range(scale):
            x = torch.rand(e - s, generator=gen, device=device)
            down = (x >= a + b).to(torch.int32)                      # quadrants c, d
            right = ((x >= a) & (x < a + b)) | (x >= a + b + c)      # quadrants b, d
            r |= down << bit
            q |= right.to(torch.int32) << bit
        rows[s:e], cols[s:e] = r, q
    row_ptr, col_idx = _csr_from_edges(rows, cols, n, n)
    del rows, cols
    return n, n, row_ptr, col_idx, _values(col_idx.numel(), values, gen, device)


def uniform_csr(rows_n, cols_n, density, seed=1, values="real", device="cuda"):
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    m = int(rows_n * cols_n * density)
    r = torch.randint(0, rows_n, (m,), generator=gen, device=device, dtype=torch.int64)
    c = torch.randint(0, cols_n, (m,), generator=gen, device=device, dtype=torch.int64)
    row_ptr, col_idx = _csr_from_edges(r, c, rows_n, cols_n)
    return rows_n, cols_n, row_ptr, col_idx, _values(col_idx.numel(), values, gen, device)


def _mt_stream(seed: int, n: int):
    """n raw std::mt19937 draws for `seed`: numpy's legacy RandomState seeds
    with init_genrand(seed) and returns raw 32-bit outputs for a full-range
    uint32 request, i.e. exactly std::mt19937(seed)()."""
    import numpy as np
    return np.random.RandomState(seed & 0xFFFFFFFF).randint(0, 1 << 32, size=n, dtype=np.uint32)


def _small_int(draws):
    import numpy as np
    m = (draws % 8).astype(np.int64)  # ref generate.hpp:15-18
    return np.where(m < 4, m - 4, m - 3).astype(np.float32)


def _uniform_real(draws):
    import numpy as np
    return (draws.astype(np.float32) * np.float32(2.0 ** -31) - np.float32(1.0)).astype(np.float32)  # :20-22


def reference_random_csr(rows_n, cols_n, density, seed, values="int"):
    """The reference's own CSR generator, ``generate_random_sparse`` /
    ``generate_random_sparse_real`` (ref generate.hpp:29-63): one raw
    mt19937 draw per position in row-major order, kept when below
    llround(density * 2^32), a kept position consuming one more draw for its
    small-integer value; "real" values come from a second stream seeded with
    seed ^ 0x9e3779b9.  Host numpy (BASELINE configs[0]/[1] size: 16.8 M
    draws); returns (row_ptr u32, col_idx u32, values f32) numpy arrays."""
    import numpy as np
    if rows_n <= 0 or cols_n <= 0 or not (0.0 < density <= 1.0):
        raise ValueError("rows and cols must be >= 1 and density in (0, 1]")
    cells = rows_n * cols_n
    thr = np.uint64(int(density * 4294967296.0 + 0.5))  # llround, density > 0
    # Draw d[i] is a position test unless it is the value draw of the kept
    # test right before it.  Over-draw, then walk the kept candidates.
    n = cells + max(64, int(cells * density * 1.5) + 6 * int((cells * density) ** 0.5) + 64)
    while True:
        d = _mt_stream(seed, n)
        kept, nxt = [], 0
        for c in np.flatnonzero(d.astype(np.uint64) < thr).tolist():
            if c >= nxt:  # a test draw, not the value draw of the kept test before it
                kept.append(c)
                nxt = c + 2
        if n - 1 - len(kept) >= cells:  # every cell tested, every kept value drawn
            break
        n *= 2
    kept = np.asarray(kept, dtype=np.int64)
    pos = kept - np.arange(kept.size, dtype=np.int64)  # cell = draw index - value draws before it
    kept, pos = kept[pos < cells], pos[pos < cells]
    vals = _small_int(d[kept + 1])
    if values == "real":
        vals = _uniform_real(_mt_stream(seed ^ 0x9E3779B9, kept.size))
    r = pos // cols_n
    row_ptr = np.zeros(rows_n + 1, np.uint32)
    np.cumsum(np.bincount(r, minlength=rows_n), out=row_ptr[1:])
    return row_ptr, (pos - r * cols_n).astype(np.uint32), vals


def reference_random_dense(rows_n, cols_n, seed, values="int"):
    """ref generate.hpp:65-79 (row-major, one draw per element)."""
    d = _mt_stream(seed, rows_n * cols_n)
    return (_uniform_real(d) if values == "real" else _small_int(d)).reshape(rows_n, cols_n)


def dense(rows_n, cols_n, seed, values="real", dtype=torch.float16, device="cuda"):
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    return _values(rows_n * cols_n, values, gen, device).reshape(rows_n, cols_n).to(dtype)


def row_slice(row_ptr, col_idx, vals, r0, r1):
    """Rows [r0, r1) of a CSR as a standalone CSR (row_ptr rebased)."""
    b, e = int(row_ptr[r0]), int(row_ptr[r1])
    return row_ptr[r0:r1 + 1] - b, col_idx[b:e], vals[b:e]
