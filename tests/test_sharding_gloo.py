"""Multi-process (gloo, world size 2 and 4, CPU) tests of the multi-GPU layouts.

The GPU runs use the same functions over NCCL; here the attention itself is
replaced by a per-head reference operation so only the data movement is
tested: head ranges, the Ulysses sequence<->head all-to-all and its inverse,
and that "all-to-all, per-head op, all-to-all back" equals the op applied to
the unsharded tensor.
"""

import os
import socket
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_04648_b200.sharding import (gather_heads, head_range, head_to_seq, seq_to_head, shard_heads,
                                            ulysses_pipeline)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _per_head_op(x, heads):
    """Stand-in for attention: an op that mixes tokens within a head but never across heads."""
    scale = torch.arange(1, heads + 1, dtype=x.dtype).view(1, -1, 1)
    return torch.cumsum(x, dim=0) * scale + x.flip(0)


def _worker(rank, world, port, L, H, d, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(1234)
        full = torch.randn((L, H, d), generator=g)  # identical on every rank
        Ll = L // world
        local = full[rank * Ll:(rank + 1) * Ll].clone()
        # sequence -> head shard equals slicing the full tensor by this rank's heads
        hs = seq_to_head(local)
        hp = H // world
        assert torch.equal(hs, full[:, rank * hp:(rank + 1) * hp])
        # round trip
        assert torch.equal(head_to_seq(hs), local)
        # composition with a per-head op == op on the full tensor, resharded by sequence
        ref = _per_head_op(full, H)
        got = head_to_seq(_per_head_op_local(hs, rank, hp))
        assert torch.allclose(got, ref[rank * Ll:(rank + 1) * Ll], rtol=1e-6, atol=1e-5)
        # per-head-chunk pipeline (async all-to-alls around each chunk's compute) == the unchunked path
        for chunk in (1, 3, hp):
            got_p = ulysses_pipeline(local, local * 2, local * 3,
                                     lambda qc, kc, vc, c0, c1: _chunk_op(qc, kc, vc, rank * hp + c0), chunk)
            full_op = _chunk_op(full, full * 2, full * 3, 0)
            assert torch.allclose(got_p, full_op[rank * Ll:(rank + 1) * Ll], rtol=1e-6, atol=1e-5), chunk
        # head-parallel shard + gather (uneven head counts allowed)
        h0, h1 = head_range(rank, world, H + 1)
        full2 = torch.randn((L, H + 1, d), generator=torch.Generator().manual_seed(7))
        mine = shard_heads(full2, rank, world)
        assert mine.shape[1] == h1 - h0
        assert torch.equal(gather_heads(mine.contiguous()), full2)
        open(os.path.join(out_dir, f"ok{rank}"), "w").close()
    finally:
        dist.destroy_process_group()


def _chunk_op(q, k, v, h_first):
    """Per-head stand-in taking three inputs; the scale depends on the global head index."""
    scale = torch.arange(h_first + 1, h_first + q.shape[1] + 1, dtype=q.dtype).view(1, -1, 1)
    return torch.cumsum(q, dim=0) * scale + k.flip(0) - v * 0.5


def _per_head_op_local(x, rank, hp):
    """_per_head_op restricted to heads [rank*hp, (rank+1)*hp) (the global head index sets the scale)."""
    scale = torch.arange(rank * hp + 1, (rank + 1) * hp + 1, dtype=x.dtype).view(1, -1, 1)
    return torch.cumsum(x, dim=0) * scale + x.flip(0)


@pytest.mark.parametrize("world", [2, 4])
def test_ulysses_and_head_sharding_gloo(world):
    L, H, d = 48, 8, 16
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), L, H, d, tmp), nprocs=world, join=True)
        assert sorted(os.listdir(tmp)) == [f"ok{r}" for r in range(world)]


def test_head_range_partition():
    for heads in (1, 5, 12, 24, 40):
        for world in (1, 2, 3, 4, 8):
            ranges = [head_range(r, world, heads) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == heads
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h1 - h0 for h0, h1 in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        head_range(2, 2, 8)
