"""FLOPs accounting of the hot path (mirror of fp8sta/metrics.py:91-102)."""

from __future__ import annotations


def flops_dense(L: int, d: int) -> int:
    """4 L^2 d: the two attention GEMMs at 2 FLOPs per MAC."""
    if L < 1 or d < 1:
        raise ValueError(f"L and d must be >= 1, got L={L}, d={d}")
    return 4 * L * L * d


def flops_sparse(L: int, d: int, density: float) -> int:
    """Dense FLOPs scaled by the admissible-pair density, rounded to int."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    return round(density * flops_dense(L, d))
