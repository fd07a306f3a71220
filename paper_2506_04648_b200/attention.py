"""Quantised sliding-tile sparse attention forward (mirror of fp8sta/attention.py).

``fp8_sparse_forward(inputs, config)`` keeps the reference signature and
semantics of its inputs (single head, rows already tile-contiguous,
fp8sta/attention.py:36-61 / :179-208) and runs quantisation and attention
on the GPU.  numpy inputs give a numpy float32 result (a drop-in for the CPU
path); CUDA tensor inputs give a CUDA tensor.  ``passthrough`` (the
full-precision branch, attention.py:192-194) runs the bf16 tcgen05 kernel
(``PassthroughPlan``): operands rounded to bf16, softmax and accumulation in
f32.  There is no CPU fallback.
"""

from __future__ import annotations

import math
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

    def __post_init__(self) -> None:
        if self.softmax_scale is not None and not self.softmax_scale > 0:
            raise ValueError("softmax_scale must be > 0")


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


def fp8_sparse_forward(inputs: AttentionInputs, config: ForwardConfig):
    """Joint tile-wise FP8 quantisation with sliding-tile sparse attention (attention.py:179-208)."""
    import torch

    from .ops import FpsaPlan

    tmap = inputs.tile_map
    scale = _resolve_scale(config.softmax_scale, inputs.d_model)
    host = not _is_torch(inputs.q)

    def dev(x):
        t = torch.from_numpy(x) if host else x
        t = t.cuda()
        return t if t.dtype in (torch.float32, torch.bfloat16) else t.float()

    q, k, v = dev(inputs.q), dev(inputs.k), dev(inputs.v)
    out = torch.empty((tmap.grid.tokens, inputs.d_model), dtype=torch.float32, device=q.device)
    if config.passthrough:
        from .ops import PassthroughPlan

        pplan = PassthroughPlan(tmap.grid.dims, tmap.scheme.dims, config.window, 1, inputs.d_model, device=q.device)
        pplan.gather(q, k, v, layout="ld", tile_order=True)
        pplan.attention(out, layout="ld", tile_order=True, softmax_scale=float(scale))
        return out.cpu().numpy() if host else out
    plan = FpsaPlan(tmap.grid.dims, tmap.scheme.dims, config.window, 1, inputs.d_model, config.fmt,
                    device=q.device, tau=config.tau)
    plan.quantize(q, k, v, layout="ld", tile_order=True)
    plan.attention(out, layout="ld", tile_order=True, softmax_scale=float(scale))
    plan.check_finite()
    return out.cpu().numpy() if host else out
