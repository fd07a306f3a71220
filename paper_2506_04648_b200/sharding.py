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


def chunk_bounds(n: int, chunk: int) -> list[tuple[int, int]]:
    """[c0, c1) ranges of `chunk` items covering range(n) (the last one shorter)."""
    if chunk < 1:
        raise ValueError(f"chunk must be >= 1, got {chunk}")
    return [(c0, min(n, c0 + chunk)) for c0 in range(0, n, chunk)]


def seq_to_head_chunk(x_local, c0: int, c1: int, group=None, async_op: bool = False):
    """Heads [c0, c1) of every rank's head group: [L/P, H, d] sequence shard -> [L, c1 - c0, d]
    (this rank's heads r H/P + [c0, c1) over the whole sequence).  With async_op, returns
    (tensor, work); the tensor is valid once work.wait() returned (or, on NCCL, once the
    current stream has been made to wait by it)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    Ll, H, d = x_local.shape
    if H % world:
        raise ValueError(f"Ulysses needs heads ({H}) divisible by the world size ({world})")
    hp = H // world
    if not 0 <= c0 < c1 <= hp:
        raise ValueError(f"head chunk [{c0}, {c1}) outside [0, {hp})")
    send = x_local.reshape(Ll, world, hp, d)[:, :, c0:c1].transpose(0, 1).contiguous()  # [P, L/P, hc, d]
    recv = torch.empty_like(send)
    work = dist.all_to_all_single(recv, send, group=group, async_op=async_op)
    out = recv.view(world * Ll, c1 - c0, d)
    return (out, work) if async_op else out


def head_chunk_to_seq(y, c0: int, c1: int, out_local, group=None):
    """Inverse of seq_to_head_chunk for one head chunk, asynchronously: y [L, c1 - c0, d] goes back
    to the sequence shards; returns (work, finish) where finish() (after work.wait()) writes the
    received tokens into out_local[:, j H/P + c0 : j H/P + c1] for every rank j."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    L, hc, d = y.shape
    Ll, H, _ = out_local.shape
    hp = H // world
    send = y.reshape(world, L // world, hc, d).contiguous()
    recv = torch.empty_like(send)
    work = dist.all_to_all_single(recv, send, group=group, async_op=True)

    def finish():
        out_local.view(Ll, world, hp, d)[:, :, c0:c1] = recv.transpose(0, 1)

    return work, finish


def ulysses_pipeline(q, k, v, compute, chunk: int, group=None):
    """Sequence-sharded q, k, v [L/P, H, d] -> output [L/P, H, d] with per-head-chunk overlap.

    compute(qc, kc, vc, c0, c1) maps the [L, hc, d] head chunk [c0, c1) of this rank's heads to
    its [L, hc, d] output.  The all-to-all of chunk i+1's inputs and of chunk i-1's output run
    (NCCL stream) while chunk i computes: the per-head overlap SURVEY.md §8e asks for.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    hp = q.shape[1] // world
    bounds = chunk_bounds(hp, chunk)

    def issue(c0, c1):
        return [seq_to_head_chunk(x, c0, c1, group, async_op=True) for x in (q, k, v)]

    out = q.new_empty(q.shape)
    pending = issue(*bounds[0])
    tails = []
    for i, (c0, c1) in enumerate(bounds):
        cur = pending
        if i + 1 < len(bounds):
            pending = issue(*bounds[i + 1])
        for _, work in cur:
            work.wait()
        y = compute(cur[0][0], cur[1][0], cur[2][0], c0, c1)
        tails.append(head_chunk_to_seq(y.to(out.dtype), c0, c1, out, group))
    for work, finish in tails:
        work.wait()
        finish()
    return out


class UlyssesAttention:
    """Sliding-tile FP8 attention for sequence-sharded inputs (BASELINE config C3).

    ``__call__(q, k, v)`` takes this rank's [L/P, H, d] token shard of q, k, v
    (natural (t,h,w) order, rank r holding tokens [r L/P, (r+1) L/P)) and
    returns the [L/P, H, d] shard of the attention output.  The local
    attention runs on heads [r H/P, (r+1) H/P) of the full sequence.
    """

    def __init__(self, grid, tile, window, heads: int, d: int, group=None, device=None, chunk_heads: int | None = None,
                 **plan_kw):
        import torch.distributed as dist

        from .ops import FpsaPlan

        self.group = group
        self.world = dist.get_world_size(group)
        if heads % self.world:
            raise ValueError(f"Ulysses needs heads ({heads}) divisible by the world size ({self.world})")
        self.heads_local = heads // self.world
        self.plan = FpsaPlan(grid, tile, window, self.heads_local, d, device=device, **plan_kw)
        # chunk_heads < heads_local: per-head-chunk pipeline (all-to-all overlapped with compute)
        self.chunk = self.heads_local if chunk_heads is None else max(1, min(int(chunk_heads), self.heads_local))
        self.chunk_plans = {}
        if self.chunk < self.heads_local:
            for c0, c1 in chunk_bounds(self.heads_local, self.chunk):
                if c1 - c0 not in self.chunk_plans:
                    self.chunk_plans[c1 - c0] = FpsaPlan(grid, tile, window, c1 - c0, d, device=device, **plan_kw)

    def __call__(self, q, k, v, out_dtype=None):
        dt = out_dtype or q.dtype
        if not self.chunk_plans:
            qh, kh, vh = (seq_to_head(x, self.group) for x in (q, k, v))
            out = self.plan(qh, kh, vh, "lhd", out_dtype=dt)
            return head_to_seq(out, self.group)

        def compute(qc, kc, vc, c0, c1):
            return self.chunk_plans[c1 - c0](qc, kc, vc, "lhd", out_dtype=dt)

        out = ulysses_pipeline(q, k, v, compute, self.chunk, self.group)
        return out if out.dtype == dt else out.to(dt)
