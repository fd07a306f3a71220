"""Tensor-level FP8 quantisation policies (mirror of fp8sta/quantize.py).

``quantize_qk_tilewise`` and ``quantize_v_channelwise`` run the sm_100a
kernels of libfpsa and return the reference's ``QuantizedTensor``: uint8
codes in the input row order and float64 scales, bit-identical to the
reference (fp8sta/quantize.py:111-134) for f32, bf16 and f64 input of any
width d (f64 data is quantised in f64, as the reference does; d other than
64 / 128 and f64 run the general exact kernels).  ``dequantize`` /
``dequantize_tensor`` reconstruct decode(code) * scale in float64 on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .fp8 import Fp8Format
from .grid import TileMap

GRANULARITY_KINDS = ("per_tile_3d", "per_channel", "per_tensor", "per_token", "per_group")
P_FIXED_SCALE = 1.0 / 448.0  # softmax weights: 1.0 maps onto the E4M3 max (quantize.py:27)


@dataclass(frozen=True)
class Granularity:
    kind: str
    group_size: int | None = None

    def __post_init__(self) -> None:
        if self.kind not in GRANULARITY_KINDS:
            raise ValueError(f"unknown granularity {self.kind!r}; expected one of {GRANULARITY_KINDS}")
        if self.kind == "per_group":
            if self.group_size is None or self.group_size < 1:
                raise ValueError("per_group requires group_size >= 1")
        elif self.group_size is not None:
            raise ValueError(f"group_size only applies to per_group, not {self.kind}")


@dataclass(frozen=True)
class QuantizedTensor:
    """FP8 codes plus scale metadata (quantize.py:47-99)."""

    codes: np.ndarray
    scales: np.ndarray
    granularity: Granularity
    fmt: Fp8Format
    block_rows: int | None = None

    def element_scales(self) -> np.ndarray:
        kind = self.granularity.kind
        if kind == "per_tensor":
            return self.scales.reshape(1, 1)
        if kind == "per_channel":
            return self.scales[None, :]
        if kind == "per_tile_3d":
            s = self.scales.cpu().numpy() if hasattr(self.scales, "cpu") else self.scales
            return np.repeat(s, self.block_rows)[:, None]
        raise NotImplementedError(f"{kind} is a comparison granularity outside the hot path")

    def dequantize(self):
        """decode(code) * scale in float64 (quantize.py:95-98), on the GPU (fpsa_decode).  numpy codes give
        numpy, CUDA codes a CUDA tensor."""
        import torch

        from .fp8 import _decode_dev, _scale_arg

        host = not isinstance(self.codes, torch.Tensor)
        codes = torch.from_numpy(np.ascontiguousarray(self.codes)) if host else self.codes
        shape = tuple(codes.shape)
        codes = codes.reshape(-1).contiguous().cuda()
        es = self.element_scales()
        scales = _scale_arg(es.cpu() if isinstance(es, torch.Tensor) else es, shape, codes.device)
        out = _decode_dev(codes, self.fmt, torch.float64, scales).reshape(shape)
        return out.cpu().numpy() if host else out




def _device_matrix(matrix):
    """(torch CUDA tensor [R, d], host_out) from numpy or torch input."""
    import torch

    if isinstance(matrix, torch.Tensor):
        x = matrix
        if x.dtype not in (torch.float32, torch.bfloat16, torch.float64):
            x = x.double()
        return x.contiguous().cuda(), False
    arr = np.asarray(matrix)
    if arr.dtype != np.float32:
        arr = arr.astype(np.float64)  # the reference quantises in float64 (quantize.py:115, :128)
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda(), True


def _run(kind: str, matrix, grid, tile, fmt: Fp8Format, n_scales: int):
    import torch

    x, host = _device_matrix(matrix)
    if x.dim() != 2:
        raise ValueError(f"expected a 2D matrix, got shape {tuple(x.shape)}")
    R, d = x.shape
    codes = torch.empty((R, d), dtype=torch.uint8, device=x.device)
    scales = torch.empty(n_scales, dtype=torch.float64, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    st = torch.cuda.current_stream().cuda_stream
    dt = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}[x.dtype]
    L = _lib.lib()
    tv = tile[0] * tile[1] * tile[2]
    if kind == "qk":
        _lib.check(L.fpsa_quantize_qk(x.data_ptr(), dt, d, 0, 1, _lib.dims3(grid), _lib.dims3(tile), d, tv,
                                      _lib.ORDER_TILE, fmt.abi_id, codes.data_ptr(), scales.data_ptr(),
                                      err.data_ptr(), st))
    else:
        ws = torch.empty(2 * d, dtype=torch.int32, device=x.device)  # f64 channel maxima on the general path
        _lib.check(L.fpsa_quantize_v(x.data_ptr(), dt, d, 0, 1, _lib.dims3(grid), _lib.dims3(tile), d, tv,
                                     _lib.ORDER_TILE, fmt.abi_id, codes.data_ptr(), scales.data_ptr(),
                                     ws.data_ptr(), err.data_ptr(), st))
    if int(err.item()):
        raise ValueError("non-finite value in quantization input")
    if host:
        return codes.cpu().numpy(), scales.cpu().numpy()
    return codes, scales


def quantize_qk_tilewise(matrix, tmap: TileMap, fmt: Fp8Format) -> QuantizedTensor:
    """One scale per 3D tile over all channels of its rows; rows tile-contiguous (quantize.py:111-124)."""
    shape = tuple(matrix.shape)
    L = tmap.grid.tokens
    if len(shape) != 2 or shape[0] != L:
        raise ValueError(f"expected an L x d matrix with L={L}, got shape {shape}")
    codes, scales = _run("qk", matrix, tmap.grid.dims, tmap.scheme.dims, fmt, tmap.tiles_total)
    return QuantizedTensor(codes, scales, Granularity("per_tile_3d"), fmt, block_rows=tmap.tile_volume)


def quantize_v_channelwise(matrix, fmt: Fp8Format) -> QuantizedTensor:
    """One scale per channel, column max over all rows (quantize.py:127-134)."""
    shape = tuple(matrix.shape)
    if len(shape) != 2 or shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"expected a non-empty 2D matrix, got shape {shape}")
    R, d = shape
    codes, scales = _run("v", matrix, (1, 1, R), (1, 1, R), fmt, d)
    return QuantizedTensor(codes, scales, Granularity("per_channel"), fmt)


def dequantize_tensor(q: QuantizedTensor):
    """Elementwise decode(code) * scale(block) (quantize.py:183-185)."""
    return q.dequantize()
