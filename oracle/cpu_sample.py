"""Bounded CPU sample of the reference algorithm, for bench.py's cpu_baseline / --impl reference legs.

TEST/BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py).  Runs the
oracle's restatement of fp8sta.fp8_sparse_forward (attention.py:179-208)
restricted to a subset of query tiles of one head: Q is quantised for the
sampled tiles, K and V for the key tiles their windows touch (V's
per-channel scale still uses the column max over all rows,
quantize.py:127-134), then the two-pass engine (attention.py:91-149) runs
on each sampled tile.  Work per sampled tile is identical to the full
call, so throughput = algorithmic FLOPs of the sampled tiles / time.
Tiles are processed by a thread pool (the reference's own concurrency
model, experiment.py:166-175) with BLAS pinned to one thread per worker.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .fpsa_oracle import E4M3, _softmax_scale, _tile_attention, block_scales, decode, encode

try:
    from threadpoolctl import threadpool_limits
except ImportError:  # pragma: no cover
    threadpool_limits = None


def sample_tiles(M: int, n: int) -> np.ndarray:
    """n query tiles spread evenly over [0, M)."""
    n = max(1, min(M, n))
    return np.unique(np.linspace(0, M - 1, n).round().astype(np.int64))


def sample_forward(q, k, v, tv: int, offs, ids, tiles, fmt=E4M3, threads: int | None = None):
    """Reference algorithm on `tiles` of one head; returns (outputs dict, flops, seconds)."""
    threads = threads or os.cpu_count() or 1
    d = q.shape[1]
    t0 = time.perf_counter()
    key_tiles = np.unique(np.concatenate([ids[offs[u]:offs[u + 1]] for u in tiles]))
    vs = block_scales(np.abs(v.astype(np.float64)).max(axis=0), fmt)
    v_fac = (vs * (1.0 / 448.0)).astype(np.float32)
    scale = _softmax_scale(d, None)

    def quant_tile(x, t):
        blk = x[t * tv:(t + 1) * tv].astype(np.float64)
        s = block_scales(np.array([np.abs(blk).max()]), fmt)[0]
        return decode(encode(blk / s, fmt), fmt), np.float32(s)

    def quant_v_tile(t):
        blk = v[t * tv:(t + 1) * tv].astype(np.float64)
        return decode(encode(blk / vs[None, :], fmt), fmt)

    def work(u):
        qv, qf = quant_tile(q, u)
        return u, qv, qf

    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    try:
        if ctx:
            ctx.__enter__()
        with ThreadPoolExecutor(max_workers=threads) as pool:
            kq = dict(zip(key_tiles, pool.map(lambda t: quant_tile(k, t), key_tiles)))
            vq = dict(zip(key_tiles, pool.map(quant_v_tile, key_tiles)))
            qq = list(pool.map(work, tiles))

            def attend(item):
                u, qv, qf = item
                keys = ids[offs[u]:offs[u + 1]]
                # local re-indexing: query tile 0, key tiles 1..n in ascending order
                kv = np.concatenate([kq[t][0] for t in keys])
                vv = np.concatenate([vq[t] for t in keys])
                k_fac = np.array([kq[t][1] for t in keys], dtype=np.float32)
                o = _tile_attention(qv, kv, vv, tv, np.array([0, len(keys)]), np.arange(len(keys)),
                                    np.array([qf], np.float32), k_fac, v_fac, scale, quant_p=True)
                return u, o

            outs = dict(pool.map(attend, qq))
    finally:
        if ctx:
            ctx.__exit__(None, None, None)
    secs = time.perf_counter() - t0
    flops = int(sum((offs[u + 1] - offs[u]) for u in tiles)) * 4 * tv * tv * d
    return outs, flops, secs
