"""Multi-GPU layouts of the hot path: head-parallel shards and the Ulysses all-to-all.

Each (batch element, head) is an independent attention problem -- per-head
scales, window lists and outputs (the reference evaluates
heads independently, experiment.py:190-199) -- so N GPUs split the heads
with no data-path collective: rank r owns the contiguous head range
``head_range(r, N, H)`` and runs its own ``FpsaPlan`` on them.

Only when activations arrive *sequence*-sharded (rank r holds tokens
[r L/N, (r+1) L/N) of all heads, as a sequence-parallel video DiT produces
them) is a collective needed: ``UlyssesAttention`` transposes sequence
shards into head shards with one NCCL ``all_to_all_single`` per tensor,
runs the local head-parallel attention, and transposes the output back.
Quantisation happens after the all-to-all: a rank then holds whole tiles
and whole V columns, which the per-tile and per-channel scales need.

Everything here is plumbing over ``torch.distributed`` (NCCL on GPUs, gloo
in the CPU tests); the compute is ``FpsaPlan``.
"""

from __future__ import annotations


def head_range(rank: int, world: int, heads: int) -> tuple[int, int]:
    """Contiguous, balanced head range [h0, h1) of `rank` (the first heads % world ranks get one more)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} out of range for world size {world}")
    if heads < 1:
        raise ValueError(f"heads must be >= 1, got {heads}")
    base, extra = divmod(heads, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def shard_heads(x, rank: int, world: int, dim: int = 1):
    """View of the rank's heads of a [L, H, d] (dim=1) or [B, L, H, d] (dim=2) tensor."""
    h0, h1 = head_range(rank, world, x.shape[dim])
    return x.narrow(dim, h0, h1 - h0)


def gather_heads(local, group=None):
    """All ranks' [L, H_r, d] head shards concatenated to [L, H, d] (parity checks only)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [torch.zeros(1, dtype=torch.int64, device=local.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([local.shape[1]], dtype=torch.int64, device=local.device), group=group)
    hmax = int(max(int(s.item()) for s in sizes))
    pad = local.new_zeros((local.shape[0], hmax, local.shape[2]))
    pad[:, : local.shape[1]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:, : int(s.item())] for p, s in zip(parts, sizes)], dim=1)


def seq_to_head(x_local, group=None):
    """[L/P, H, d] sequence shard -> [L, H/P, d] head shard (one all_to_all_single)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    Ll, H, d = x_local.shape
    if H % world:
        raise ValueError(f"Ulysses needs heads ({H}) divisible by the world size ({world})")
    hp = H // world
    # [L/P, P, H/P, d] -> [P, L/P, H/P, d]: chunk j (rank j's heads) contiguous
    send = x_local.reshape(Ll, world, hp, d).transpose(0, 1).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv[i] = tokens of rank i for my heads -> [L, H/P, d] in token order
    return recv.reshape(world * Ll, hp, d)


def head_to_seq(y_heads, group=None):
    """[L, H/P, d] head shard -> [L/P, H, d] sequence shard (inverse of seq_to_head)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    L, hp, d = y_heads.shape
    if L % world:
        raise ValueError(f"sequence length {L} not divisible by the world size {world}")
    send = y_heads.reshape(world, L // world, hp, d).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv[j] = my tokens of rank j's heads -> [L/P, P, H/P, d] -> [L/P, H, d]
    return recv.transpose(0, 1).reshape(L // world, world * hp, d)


class UlyssesAttention:
    """Sliding-tile FP8 attention for sequence-sharded inputs (BASELINE config C3).

    ``__call__(q, k, v)`` takes this rank's [L/P, H, d] token shard of q, k, v
    (natural (t,h,w) order, rank r holding tokens [r L/P, (r+1) L/P)) and
    returns the [L/P, H, d] shard of the attention output.  The local
    attention runs on heads [r H/P, (r+1) H/P) of the full sequence.
    """

    def __init__(self, grid, tile, window, heads: int, d: int, group=None, device=None, **plan_kw):
        import torch.distributed as dist

        from .ops import FpsaPlan

        self.group = group
        self.world = dist.get_world_size(group)
        if heads % self.world:
            raise ValueError(f"Ulysses needs heads ({heads}) divisible by the world size ({self.world})")
        self.heads_local = heads // self.world
        self.plan = FpsaPlan(grid, tile, window, self.heads_local, d, device=device, **plan_kw)

    def __call__(self, q, k, v, out_dtype=None):
        qh, kh, vh = (seq_to_head(x, self.group) for x in (q, k, v))
        out = self.plan(qh, kh, vh, "lhd", out_dtype=out_dtype or q.dtype)
        return head_to_seq(out, self.group)
