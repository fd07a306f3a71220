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


def fidelity_from_sums(sxy: float, sxx: float, syy: float, see: float, mx: float, my: float,
                       n: int) -> tuple[float, float, float]:
    """(cosine, mse, snr_db) from device sums (ops.device_fidelity), with the
    reference's conventions (fp8sta/metrics.py:41-88): two zero vectors have
    cosine 1 and one zero vector 0; the cosine is clamped to [-1, 1]; SNR is
    reference-anchored (x = reference), +inf for zero error, and undefined
    (ValueError) for an all-zero reference."""
    import math

    if mx == 0.0 and my == 0.0:
        cos = 1.0
    elif mx == 0.0 or my == 0.0:
        cos = 0.0
    else:
        cos = min(1.0, max(-1.0, sxy / math.sqrt(sxx * syy)))
    err = see / n
    if mx == 0.0:
        raise ValueError("SNR is undefined for an all-zero reference")
    snr = math.inf if see == 0.0 else 10.0 * math.log10(sxx / see)
    return cos, err, snr
