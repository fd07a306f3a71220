"""FP8 format descriptors (mirror of fp8sta/fp8.py:28-61, :135-150).

The element codec itself runs on the GPU inside the quantisation kernels
(paper_2506_04648_b200/csrc/fpsa_quant.cu), bit-identical to fp8.encode.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Fp8Format:
    name: str
    exponent_bits: int
    mantissa_bits: int
    exponent_bias: int
    max_value: float
    min_normal: float
    has_inf: bool

    @property
    def abi_id(self) -> int:
        return {"e4m3": 0, "e5m2": 1}[self.name]


E4M3 = Fp8Format("e4m3", 4, 3, 7, 448.0, 2.0 ** -6, False)
E5M2 = Fp8Format("e5m2", 5, 2, 15, 57344.0, 2.0 ** -14, True)
FORMATS = {"e4m3": E4M3, "e5m2": E5M2}


def compute_scale(values, fmt: Fp8Format) -> float:
    """max|values| / max_value, 1.0 for an all-zero block (fp8.py:135-150)."""
    arr = np.asarray(values, dtype=np.float64)
    if arr.size == 0:
        raise ValueError("cannot compute a scale for an empty block")
    if not np.isfinite(arr).all():
        raise ValueError("non-finite value in scale block")
    peak = float(np.max(np.abs(arr)))
    if peak == 0.0:
        return 1.0
    return max(peak / fmt.max_value, np.finfo(np.float64).tiny)
