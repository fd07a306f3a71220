"""Quantised sliding-tile sparse attention forward (mirror of fp8sta/attention.py).

``fp8_sparse_forward(inputs, config)`` keeps the reference signature and
semantics of its inputs (single head, rows already tile-contiguous,
fp8sta/attention.py:36-61 / :179-208) and runs quantisation and attention
on the GPU.  numpy inputs give a numpy float32 result (a drop-in for the CPU
path); CUDA tensor inputs give a CUDA tensor.  ``passthrough`` (the
full-precision branch, attention.py:192-194) runs the bf16 tcgen05 kernel
(``PassthroughPlan``): operands rounded to bf16, softmax and accumulation in
f32.  There is no CPU fallback.

``ForwardConfig.p_mode`` (extension) selects the softmax-weight semantics:
``"normalized"`` (default) is the reference's arithmetic -- exact row max, f64
row sum, P = e4m3(448 * p) of the normalised weights (attention.py:133-145) --
in a three-pass kernel; ``"onepass"`` is the fast path of the batched API
(unnormalised weights re-quantised per key block).  Plans are
cached per (shape, window, format, mode, device, stream, thread).  Head dims
other than 64 / 128 (the tcgen05 operand widths) are zero-padded to the next
one: zero columns change no tile or channel amax, no logit and no kept output
column, so codes and scales of the real columns are unchanged.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np

from .fp8 import E4M3, Fp8Format
from .grid import TileMap
from .sparsity import WindowSpec


@dataclass(frozen=True)
class AttentionInputs:
    """Single-head q, k, v in tile-contiguous row order plus their tile map."""

    q: object
    k: object
    v: object
    tile_map: TileMap

    def __post_init__(self) -> None:
        L, d = self.tile_map.grid.tokens, self.tile_map.grid.d_model
        for name in ("q", "k", "v"):
            arr = getattr(self, name)
            if _is_torch(arr):
                import torch

                if tuple(arr.shape) != (L, d):
                    raise ValueError(f"{name} must have shape ({L}, {d}), got {tuple(arr.shape)}")
                if not bool(torch.isfinite(arr).all()):
                    raise ValueError(f"{name} contains non-finite values")
                continue
            arr = np.ascontiguousarray(arr, dtype=np.float32)
            if arr.shape != (L, d):
                raise ValueError(f"{name} must have shape ({L}, {d}), got {arr.shape}")
            if not np.isfinite(arr).all():
                raise ValueError(f"{name} contains non-finite values")
            object.__setattr__(self, name, arr)

    @property
    def d_model(self) -> int:
        return self.tile_map.grid.d_model


@dataclass(frozen=True)
class ForwardConfig:
    """Knobs of the quantised sparse forward (attention.py:64-80).

    ``tau`` (extension, log2 units) is the lazy-rescale headroom of the
    one-pass GPU softmax; see DESIGN.md.
    """

    window: WindowSpec
    fmt: Fp8Format = E4M3
    softmax_scale: float | None = None
    passthrough: bool = False
    tau: float = 8.0
    p_mode: str = "normalized"

    def __post_init__(self) -> None:
        if self.softmax_scale is not None and not self.softmax_scale > 0:
            raise ValueError("softmax_scale must be > 0")
        if self.p_mode not in ("normalized", "onepass"):
            raise ValueError(f"p_mode must be 'normalized' or 'onepass', got {self.p_mode!r}")


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _resolve_scale(scale, d: int) -> np.float32:
    if scale is None:
        return np.float32(1.0 / math.sqrt(d))
    if not scale > 0:
        raise ValueError("softmax_scale must be > 0")
    return np.float32(scale)


_PLAN_CACHE: dict = {}
_PLAN_LOCK = threading.Lock()
MAX_HEAD_DIM = 128


def _padded_dim(d: int) -> int:
    """Operand width of the tcgen05 kernels for head dim d (64 or 128)."""
    if d > MAX_HEAD_DIM:
        raise NotImplementedError(f"head dim {d} > {MAX_HEAD_DIM} is not supported by the sm_100a kernels")
    return 64 if d <= 64 else 128


def _cached_plan(kind: str, tmap: TileMap, config: ForwardConfig, dp: int, device):
    import torch

    from .ops import FpsaPlan, PassthroughPlan, cache_get

    stream = torch.cuda.current_stream(device).cuda_stream
    key = (kind, tmap.grid.dims, tmap.scheme.dims, config.window.dims, dp, config.fmt.name, config.p_mode,
           float(config.tau), str(device), stream, threading.get_ident())

    def make():
        if kind == "passthrough":
            return PassthroughPlan(tmap.grid.dims, tmap.scheme.dims, config.window, 1, dp, device=device)
        return FpsaPlan(tmap.grid.dims, tmap.scheme.dims, config.window, 1, dp, config.fmt, device=device,
                        tau=config.tau, p_mode=config.p_mode)

    with _PLAN_LOCK:
        plan = cache_get(_PLAN_CACHE, key, make)
    return plan


def fp8_sparse_forward(inputs: AttentionInputs, config: ForwardConfig):
    """Joint tile-wise FP8 quantisation with sliding-tile sparse attention (attention.py:179-208)."""
    import torch

    tmap = inputs.tile_map
    d = inputs.d_model
    scale = _resolve_scale(config.softmax_scale, d)  # of the real head dim, before any padding
    dp = _padded_dim(d)
    host = not _is_torch(inputs.q)

    def dev(x):
        t = torch.from_numpy(x) if host else x
        t = t.cuda()
        t = t if t.dtype in (torch.float32, torch.bfloat16) else t.float()
        if dp != d:
            t = torch.nn.functional.pad(t, (0, dp - d))
        return t

    q, k, v = dev(inputs.q), dev(inputs.k), dev(inputs.v)
    out = torch.empty((tmap.grid.tokens, dp), dtype=torch.float32, device=q.device)
    if config.passthrough:
        pplan = _cached_plan("passthrough", tmap, config, dp, q.device)
        pplan.gather(q, k, v, layout="ld", tile_order=True)
        pplan.attention(out, layout="ld", tile_order=True, softmax_scale=float(scale))
    else:
        plan = _cached_plan("fp8", tmap, config, dp, q.device)
        plan.quantize(q, k, v, layout="ld", tile_order=True)
        plan.attention(out, layout="ld", tile_order=True, softmax_scale=float(scale))
        plan.check_finite()
    if dp != d:
        out = out[:, :d].contiguous()
    return out.cpu().numpy() if host else out
