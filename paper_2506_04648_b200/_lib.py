"""ctypes binding of libfpsa.so (the C ABI declared in include/fpsa.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2506_04648_b200.build``).  There is no fallback: if the
library is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("FPSA_LIB", "libfpsa.so"))  # FPSA_LIB: in-tree variant (experiments)

FPSA_OK = 0
FPSA_EINVAL = 1
FPSA_EINDIVISIBLE = 2
FPSA_ENONFINITE = 3
FPSA_ECUDA = 4
FPSA_EUNSUPPORTED = 5
FPSA_ERANGE = 6
FPSA_ECAPACITY = 7

F32, BF16, F16, F64 = 0, 1, 2, 3
E4M3_ID, E5M2_ID = 0, 1
ORDER_TILE, ORDER_NATURAL = 0, 1
P_ONEPASS, P_NORMALIZED = 0, 1  # fpsa_p_mode


class Dims3(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32)]


class FpsaError(RuntimeError):
    """Raised for CUDA / library failures (FPSA_ECUDA, FPSA_ECAPACITY)."""


_lock = threading.Lock()
_lib = None

_c = ctypes
_i32, _i64, _f32, _dbl, _vp = _c.c_int32, _c.c_int64, _c.c_float, _c.c_double, _c.c_void_p
_pi32, _pi64 = _c.POINTER(_i32), _c.POINTER(_i64)

# name -> (restype, argtypes); mirrors include/fpsa.h exactly
SIGNATURES = {
    "fpsa_last_error": (_c.c_char_p, []),
    "fpsa_version": (_c.c_int, []),
    "fpsa_tile_grid": (_c.c_int, [Dims3, Dims3, _c.POINTER(Dims3)]),
    "fpsa_tile_perm": (_c.c_int, [Dims3, Dims3, _pi64]),
    "fpsa_window_nnz": (_c.c_int, [Dims3, Dims3, _pi64]),
    "fpsa_window_csr": (_c.c_int, [Dims3, Dims3, _pi32, _pi32, _i64, _pi64]),
    "fpsa_regime_of": (_c.c_int, [_i32, _i32, _dbl, _dbl, _pi32]),
    "fpsa_quantize_qk": (_c.c_int, [_vp, _c.c_int, _i64, _i64, _i32, Dims3, Dims3, _i32, _i32, _c.c_int, _c.c_int,
                                    _vp, _vp, _vp, _vp]),
    "fpsa_quantize_v": (_c.c_int, [_vp, _c.c_int, _i64, _i64, _i32, Dims3, Dims3, _i32, _i32, _c.c_int, _c.c_int,
                                   _vp, _vp, _vp, _vp, _vp]),
    "fpsa_quantize_qkv": (_c.c_int, [_vp, _vp, _vp, _c.c_int, _i64, _i64, _i32, Dims3, Dims3, _i32, _i32,
                                     _c.c_int, _c.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fpsa_quantize_workspace_bytes": (_c.c_int, [_i32, _i32, _pi64]),
    "fpsa_quantize_qkv_amax": (_c.c_int, [_vp, _vp, _vp, _c.c_int, _i64, _i64, _i32, Dims3, Dims3, _i32, _i32,
                                          _c.c_int, _c.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                          _vp]),
    "fpsa_encode": (_c.c_int, [_vp, _c.c_int, _vp, _i64, _c.c_int, _vp, _vp, _vp]),
    "fpsa_decode": (_c.c_int, [_vp, _i64, _c.c_int, _vp, _vp, _c.c_int, _vp, _vp]),
    "fpsa_attn_worklist": (_c.c_int, [_i32, Dims3, _i32, _pi32, _pi32, _i64, _pi64]),
    "fpsa_attn_workspace_bytes": (_c.c_int, [_i32, _pi64]),
    "fpsa_attn_fwd": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, Dims3, Dims3, _i32, _i32, _vp, _vp, _vp, _i32,
                                 _f32, _c.c_int, _f32, _c.c_int, _vp, _c.c_int, _i64, _i64, _c.c_int, _vp, _i64,
                                 _vp]),
    "fpsa_tile_gather_bf16": (_c.c_int, [_vp, _c.c_int, _i64, _i64, _i32, Dims3, Dims3, _i32, _i32, _c.c_int, _vp,
                                         _vp]),
    "fpsa_attn_bf16_fwd": (_c.c_int, [_vp, _vp, _vp, _i32, Dims3, Dims3, _i32, _i32, _vp, _vp, _vp, _i32, _f32, _vp,
                                      _c.c_int, _i64, _i64, _c.c_int, _vp, _i64, _vp]),
    "fpsa_fidelity": (_c.c_int, [_vp, _c.c_int, _vp, _c.c_int, _i64, _i32, _i32, _i64, _i64, _vp, _vp]),
    "fpsa_copy2d": (_c.c_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
}


def lib():
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise FpsaError(
                    f"{LIB_PATH} is missing: build the CUDA library first "
                    "(python -c 'import __graft_entry__ as g; g.build()')")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int) -> None:
    """Map an fpsa_status to the reference's exception types."""
    if status == FPSA_OK:
        return
    msg = lib().fpsa_last_error().decode()
    if status in (FPSA_EINVAL, FPSA_EINDIVISIBLE, FPSA_ENONFINITE):
        raise ValueError(msg)
    if status == FPSA_ERANGE:
        raise IndexError(msg)
    if status == FPSA_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise FpsaError(msg)


def dims3(v) -> Dims3:
    t, h, w = (int(x) for x in v)
    return Dims3(t, h, w)
