"""Host-side logic of the multi-GPU layer at world size 2 over gloo (CPU):
nnz-balanced window sharding, shard-local CSR, dense broadcast and the
row all-gather -- checked end to end with the CPU oracle doing each shard's
SpMM: the gathered result must equal the single-process product bit for
bit (small-integer inputs)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2412_11007_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_windows_balance_and_cover():
    m = O.generate_random_sparse(200, 90, 0.08, 3)
    rp = torch.from_numpy(m.row_ptr.astype(np.int64))
    for world in (1, 2, 3, 4, 8):
        cuts = D.shard_windows(rp, m.rows, world)
        W = (m.rows + 7) // 8
        assert cuts[0] == 0 and cuts[-1] == W and all(a <= b for a, b in zip(cuts, cuts[1:]))
        nnz = [int(rp[min(8 * cuts[r + 1], m.rows)] - rp[min(8 * cuts[r], m.rows)]) for r in range(world)]
        assert sum(nnz) == m.nnz
        # each shard within one window's worth of nnz of the ideal share
        win = max(int(rp[min(8 * w + 8, m.rows)] - rp[8 * w]) for w in range(W))
        assert max(nnz) - m.nnz / world <= win


def test_shard_windows_by_nv():
    m = O.generate_random_sparse(160, 64, 0.1, 4)
    me = O.encode_mebcrs(m, 0)
    cuts = D.shard_windows(torch.from_numpy(m.row_ptr.astype(np.int64)), m.rows, 4, "nv",
                           torch.from_numpy(me.row_pointers.astype(np.int64)))
    assert cuts[0] == 0 and cuts[-1] == me.num_windows


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = O.generate_random_sparse(203, 120, 0.07, 11)  # 26 windows, last one partial
        rp = torch.from_numpy(m.row_ptr.astype(np.int64))
        ci = torch.from_numpy(m.col_idx.astype(np.int64))
        v = torch.from_numpy(m.values)
        B = torch.from_numpy(O.generate_random_dense(m.cols, 24, 12)) if rank == 0 else torch.zeros(m.cols, 24)
        D.broadcast_dense(B, src=0)
        cuts = D.shard_windows(rp, m.rows, world)
        sh = D.shard_of(cuts, rank, m.rows)
        lrp, lci, lv = D.local_rows(rp, ci, v, sh)
        local = O.Csr(sh.rows, m.cols, lrp.numpy().astype(np.uint32), lci.numpy().astype(np.uint32), lv.numpy())
        C_local = torch.from_numpy(O.spmm(O.encode_mebcrs(local, 0), B.numpy()))
        full = D.gather_rows(C_local, [D.shard_of(cuts, r, m.rows).rows for r in range(world)])
        want = O.spmm(O.encode_mebcrs(m, 0), B.numpy())
        out_q.put((rank, bool(np.array_equal(full.numpy().view(np.uint32), want.view(np.uint32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_world2_gloo_sharded_spmm_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=150) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert results == {0: True, 1: True}
