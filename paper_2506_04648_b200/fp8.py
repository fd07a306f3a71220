"""FP8 format descriptors and the element codec (mirror of fp8sta/fp8.py:28-61, :135-234).

``encode`` / ``decode`` / ``quantize_dequantize`` run on the GPU (fpsa_encode /
fpsa_decode in csrc/fpsa_quant.cu, bit-identical to the reference); the
quantisation kernels use the same rounding inline.
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


# ---------------------------------------------------------------------------- element codec (GPU)
def _torch():
    import torch

    return torch


def _to_device(x, allow=("float32", "float64", "bfloat16")):
    """(CUDA tensor, dtype id, host?, scalar?) of numpy / Python / torch input."""
    from . import _lib

    torch = _torch()
    if isinstance(x, torch.Tensor):
        t, host, scalar = x, False, x.dim() == 0
        if str(t.dtype).replace("torch.", "") not in allow:
            t = t.double()
    else:
        a = np.asarray(x)
        scalar = a.ndim == 0
        if a.dtype != np.float32:
            a = a.astype(np.float64)
        t, host = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)), True
    t = t.reshape(-1).contiguous().cuda()
    dt = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16}[t.dtype]
    return t, dt, host, scalar


def _scale_arg(scale, shape, device):
    torch = _torch()
    s = scale if isinstance(scale, torch.Tensor) else torch.from_numpy(np.asarray(scale, dtype=np.float64))
    return torch.broadcast_to(s.to(device=device, dtype=torch.float64), shape).reshape(-1).contiguous()


def _encode_dev(t, dt, fmt: Fp8Format, scale=None):
    from . import _lib

    torch = _torch()
    codes = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
    err = torch.zeros(1, dtype=torch.int32, device=t.device)
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().fpsa_encode(t.data_ptr(), dt, None if scale is None else scale.data_ptr(), t.numel(),
                                          fmt.abi_id, codes.data_ptr(), err.data_ptr(),
                                          torch.cuda.current_stream(t.device).cuda_stream))
    e = int(err.item())
    if e & 1:
        raise ValueError("cannot encode NaN")
    if e & 2:
        raise ValueError(f"cannot encode infinity in {fmt.name}")
    return codes


def _decode_dev(codes, fmt: Fp8Format, out_dtype, scale=None):
    from . import _lib

    torch = _torch()
    out = torch.empty(codes.numel(), dtype=out_dtype, device=codes.device)
    err = torch.zeros(1, dtype=torch.int32, device=codes.device)
    odt = _lib.F32 if out_dtype == torch.float32 else _lib.F64
    with torch.cuda.device(codes.device):
        _lib.check(_lib.lib().fpsa_decode(codes.data_ptr(), codes.numel(), fmt.abi_id,
                                          None if scale is None else scale.data_ptr(), out.data_ptr(), odt,
                                          err.data_ptr(), torch.cuda.current_stream(codes.device).cuda_stream))
    if int(err.item()) & 1:
        raise ValueError(f"NaN code pattern for {fmt.name}")
    return out


def encode(x, fmt: Fp8Format):
    """Round to nearest even onto the format's codes, saturating, sign kept on zero (fp8.py:153-188).

    Scalars return ``int``, numpy input ``np.uint8`` of the same shape, CUDA tensors a uint8 tensor.
    NaN raises; infinity raises unless the format has one.  Runs on the GPU (fpsa_encode)."""
    shape = np.shape(x) if not isinstance(x, _torch().Tensor) else tuple(x.shape)
    t, dt, host, scalar = _to_device(x)
    codes = _encode_dev(t, dt, fmt)
    if scalar:
        return int(codes.item())
    return codes.cpu().numpy().reshape(shape) if host else codes.reshape(shape)


def decode(code, fmt: Fp8Format):
    """Exact float32 value of codes; NaN bit patterns raise (fp8.py:191-205).  Runs on the GPU (fpsa_decode)."""
    torch = _torch()
    if isinstance(code, torch.Tensor):
        c, host, scalar, shape = code.to(torch.uint8).reshape(-1).contiguous().cuda(), False, code.dim() == 0, \
            tuple(code.shape)
    else:
        a = np.asarray(code, dtype=np.uint8)
        c, host, scalar, shape = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda(), True, a.ndim == 0, \
            a.shape
    out = _decode_dev(c, fmt, torch.float32)
    if scalar:
        return float(out.item())
    return out.cpu().numpy().reshape(shape) if host else out.reshape(shape)


def quantize_dequantize(x, scale, fmt: Fp8Format):
    """decode(encode(x / scale)) * scale, all in float64 (fp8.py:219-234); scale broadcasts against x."""
    torch = _torch()
    if not bool(np.all(np.asarray(scale.cpu() if isinstance(scale, torch.Tensor) else scale) > 0)):
        raise ValueError("scale must be strictly positive")
    shape = np.shape(x) if not isinstance(x, torch.Tensor) else tuple(x.shape)
    t, dt, host, scalar = _to_device(x, allow=("float64",))
    if not bool(torch.isfinite(t).all()):
        raise ValueError("quantize_dequantize requires finite input")
    s = _scale_arg(scale, shape, t.device)
    out = _decode_dev(_encode_dev(t, dt, fmt, s), fmt, torch.float64, s)
    if scalar or (not isinstance(x, (np.ndarray, torch.Tensor)) and np.ndim(x) == 0):
        return float(out.item())
    return out.cpu().numpy().reshape(shape) if host else out.reshape(shape)


def code_table(fmt: Fp8Format) -> np.ndarray:
    """All 256 decoded values in code order, float64, NaN patterns as nan (fp8.py:214-216); decoded on the
    GPU (fpsa_decode, whose NaN flag is expected here)."""
    from . import _lib

    torch = _torch()
    codes = torch.arange(256, dtype=torch.uint8, device="cuda")
    out = torch.empty(256, dtype=torch.float64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().fpsa_decode(codes.data_ptr(), 256, fmt.abi_id, None, out.data_ptr(), _lib.F64,
                                      err.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy()


def is_nan_code(code, fmt: Fp8Format):
    """True where a byte is one of the format's NaN patterns (fp8.py:208-211)."""
    return np.isnan(code_table(fmt)[np.asarray(code, dtype=np.uint8)])
