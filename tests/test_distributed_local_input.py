"""CPU: the sharded layers' input contract (all rows, or this shard's rows)."""
import pytest
import torch

from paper_2412_11007_b200 import distributed as D


def test_local_input_accepts_full_or_shard_rows():
    rows = 50
    rp = torch.arange(0, 2 * rows + 1, 2, dtype=torch.int32)
    cuts = D.shard_windows(rp, rows, 2)
    sh = D.shard_of(cuts, 1, rows)
    H = torch.arange(rows * 3, dtype=torch.float32).reshape(rows, 3)
    assert torch.equal(D.local_input(H, sh, rows), H[sh.r0:sh.r1])
    mine = H[sh.r0:sh.r1].clone()
    assert D.local_input(mine, sh, rows) is mine
    with pytest.raises(ValueError):
        D.local_input(H[:7], sh, rows)
