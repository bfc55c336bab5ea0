"""Worker for tests/test_gpu_distributed.py (run under torchrun, 2 ranks,
gloo, both ranks on the one visible GPU): two chained layers of the sharded
GCN and AGNN against the single-process layers on the same graph, chained
through full outputs and through each shard's local rows."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_11007_b200 import distributed as D, graphs as G, layers as L  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
torch.cuda.set_device(0)
rows, cols, rp, ci, v = G.power_law_csr(G.GraphSpec("t", 6000, 120_000, alpha=1.3, cap=50.0, seed=9), values="int")
g = torch.Generator(device="cuda").manual_seed(3)
H = torch.randn(rows, 64, device="cuda", generator=g)
W1 = torch.randn(64, 64, device="cuda", generator=g).half() / 8
W2 = torch.randn(64, 32, device="cuda", generator=g).half() / 8

gcn1, gcn2 = L.GCNLayer(rows, rp, ci, W1), L.GCNLayer(rows, rp, ci, W2)
want = gcn2(gcn1(H))
s1, s2 = D.ShardedGCNLayer(rows, rp, ci, W1), D.ShardedGCNLayer(rows, rp, ci, W2)
got = s2(s1(H))
gcn_err = float((got - want).norm() / want.norm())
# chaining on local rows: layer 1 keeps its shard, layer 2 takes it
got_local = s2(s1(H, gather=False))
gcn_err = max(gcn_err, float((got_local - want).norm() / want.norm()))

agnn = L.AGNNLayer(rows, rp, ci, beta=1.3)
want = agnn(agnn(H))
sa = D.ShardedAGNNLayer(rows, rp, ci, beta=1.3)
got = sa(sa(H))
agnn_exact = bool(torch.equal(got, want)) and bool(torch.equal(sa(sa(H, gather=False)), want))
agnn_err = float((got - want).norm() / want.norm())
print(f"RANK{rank} gcn_rel_l2={gcn_err:.3e} agnn_exact={agnn_exact} agnn_rel_l2={agnn_err:.3e}", flush=True)
dist.barrier()
dist.destroy_process_group()
