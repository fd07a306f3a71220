"""numpy restatement of the reference ``fp8sta`` hot path (test infrastructure).

Written independently of the reference code: the FP8 encoder works on
frexp/rint arithmetic instead of the reference's searchsorted boundary tables,
the tile permutation is a reshape/transpose instead of index arithmetic, and
the window lists are built per axis as integer intervals instead of an M x M
boolean mask.  Semantics (rounding, saturation, signed zero, error types) are
those of the cited reference lines and are pinned by the golden vectors in
``tests/golden``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Fmt", "E4M3", "E5M2", "FORMATS",
    "decode", "encode", "grid_round",
    "block_scales", "quantize_qk_tilewise", "quantize_v_channelwise",
    "tile_perm", "tile_grid_dims",
    "axis_interval", "window_lists", "density_of", "flops_sparse_of",
    "regime_of", "schedule_valid",
    "fp8_sparse_forward", "sparse_forward_f32", "onepass_forward", "bf16_round", "passthrough_emulation",
    "normalized_rows", "fp8_sparse_rows", "p_flip_budget", "packed_keys",
    "cosine", "max_abs", "gen_inputs",
]


# --------------------------------------------------------------------------
# FP8 formats -- fp8sta/fp8.py:28-61
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Fmt:
    name: str
    ebits: int
    mbits: int
    bias: int
    max_value: float
    has_inf: bool

    @property
    def min_normal(self) -> float:
        return 2.0 ** (1 - self.bias)

    @property
    def sub_step_exp(self) -> int:
        # exponent of the subnormal spacing, fp8.py:79-80 (m * 2^(1-bias-mbits))
        return 1 - self.bias - self.mbits

    @property
    def max_code(self) -> int:
        # largest finite non-negative code: fp8.py:86-87
        return 0x7E if not self.has_inf else 0x7B


E4M3 = Fmt("e4m3", 4, 3, 7, 448.0, False)       # fp8.py:41-49
E5M2 = Fmt("e5m2", 5, 2, 15, 57344.0, True)     # fp8.py:51-59
FORMATS = {"e4m3": E4M3, "e5m2": E5M2}


def _code_values(fmt: Fmt) -> np.ndarray:
    """Value of each of the 256 codes (NaN where the pattern is NaN), fp8.py:73-84."""
    codes = np.arange(256)
    sign = np.where(codes & 0x80, -1.0, 1.0)
    e = (codes >> fmt.mbits) & ((1 << fmt.ebits) - 1)
    m = codes & ((1 << fmt.mbits) - 1)
    mag = np.where(
        e == 0,
        np.ldexp(m.astype(np.float64), fmt.sub_step_exp),
        np.ldexp((m + (1 << fmt.mbits)).astype(np.float64), e - fmt.bias - fmt.mbits),
    )
    top = (1 << fmt.ebits) - 1
    if fmt.has_inf:
        mag = np.where(e == top, np.where(m == 0, np.inf, np.nan), mag)
    else:
        mag = np.where((e == top) & (m == (1 << fmt.mbits) - 1), np.nan, mag)
    return sign * mag


_VALUES = {f.name: _code_values(f) for f in (E4M3, E5M2)}


def decode(codes, fmt: Fmt = E4M3) -> np.ndarray:
    """codes -> exact float32 values; NaN patterns raise (fp8.py:191-205)."""
    c = np.asarray(codes, dtype=np.uint8)
    out = _VALUES[fmt.name][c].astype(np.float32)
    if np.isnan(out).any():
        raise ValueError(f"NaN code pattern for {fmt.name}")
    return out


def encode(x, fmt: Fmt = E4M3) -> np.ndarray:
    """Round to nearest, ties to even, saturating; sign kept on zero (fp8.py:153-188).

    Restated with frexp arithmetic: the spacing of the grid around |x| is
    2^max(e - mbits, 1 - bias - mbits); ``np.rint`` gives ties-to-even on the
    multiple count, which coincides with ties to the even code.
    """
    a = np.asarray(x)
    if a.dtype != np.float32:
        a = a.astype(np.float64)
    if np.isnan(a).any():
        raise ValueError("cannot encode NaN")
    mag = np.abs(a).astype(np.float64)
    inf = np.isinf(mag)
    if inf.any() and not fmt.has_inf:
        raise ValueError(f"cannot encode infinity in {fmt.name}")
    mag = np.where(inf, 0.0, mag)
    _, ex = np.frexp(mag)
    step_exp = np.maximum(ex - 1 - fmt.mbits, fmt.sub_step_exp)
    k = np.rint(np.ldexp(mag, -step_exp))
    val = np.minimum(np.ldexp(k, step_exp), fmt.max_value)
    # value -> code
    fr, ex2 = np.frexp(val)
    normal = val >= fmt.min_normal
    mant = np.where(normal, np.ldexp(fr, fmt.mbits + 1) - (1 << fmt.mbits), 0.0)
    code_normal = ((ex2 - 1 + fmt.bias) << fmt.mbits) + mant.astype(np.int64)
    code_sub = np.ldexp(val, -fmt.sub_step_exp).astype(np.int64)
    code = np.where(normal, code_normal, code_sub).astype(np.uint8)
    if fmt.has_inf:
        code = np.where(inf, np.uint8(0x7C), code)
    code = code | (np.signbit(a).astype(np.uint8) << 7)
    return code.astype(np.uint8)


def grid_round(v: np.ndarray, fmt: Fmt = E4M3) -> np.ndarray:
    """RNE of non-negative float32 onto the fp8 grid, saturating (fp8.py:237-253)."""
    if v.dtype != np.float32:
        raise TypeError("grid_round expects float32")
    return decode(encode(v, fmt), fmt)


# --------------------------------------------------------------------------
# quantisation policies -- fp8sta/quantize.py
# --------------------------------------------------------------------------
def block_scales(peaks: np.ndarray, fmt: Fmt = E4M3) -> np.ndarray:
    """max(peak/max_value, f64 tiny); exactly 1.0 for an all-zero block (quantize.py:102-108)."""
    peaks = np.asarray(peaks, dtype=np.float64)
    if not np.isfinite(peaks).all():
        raise ValueError("non-finite value in quantization input")
    s = np.maximum(peaks / fmt.max_value, np.finfo(np.float64).tiny)
    return np.where(peaks == 0.0, 1.0, s)


def quantize_qk_tilewise(x: np.ndarray, tv: int, fmt: Fmt = E4M3):
    """One f64 scale per tile of tv tile-contiguous rows (quantize.py:111-124)."""
    m = np.asarray(x, dtype=np.float64)
    L, d = m.shape
    if L % tv:
        raise ValueError(f"L={L} not a multiple of the tile volume {tv}")
    tiles = m.reshape(L // tv, tv * d)
    scales = block_scales(np.abs(tiles).max(axis=1), fmt)
    codes = encode(tiles / scales[:, None], fmt).reshape(L, d)
    return codes, scales


def quantize_v_channelwise(x: np.ndarray, fmt: Fmt = E4M3):
    """One f64 scale per column over all rows (quantize.py:127-134)."""
    m = np.asarray(x, dtype=np.float64)
    scales = block_scales(np.abs(m).max(axis=0), fmt)
    return encode(m / scales[None, :], fmt), scales


# --------------------------------------------------------------------------
# layout -- fp8sta/grid.py
# --------------------------------------------------------------------------
def tile_grid_dims(grid: tuple[int, int, int], tile: tuple[int, int, int]) -> tuple[int, int, int]:
    """Tiles per axis, rejecting indivisible axes with the reference message (grid.py:91-109)."""
    out = []
    for axis, g, s in zip("thw", grid, tile):
        if g % s:
            raise ValueError(f"indivisible grid: axis {axis} has {g} tokens, not divisible by tile extent {s}")
        out.append(g // s)
    return tuple(out)


def tile_perm(grid: tuple[int, int, int], tile: tuple[int, int, int]) -> np.ndarray:
    """Gather permutation to tile-major order (grid.py:132-154).

    x[perm] lists tiles row-major over the tile grid, tokens row-major inside
    a tile.  Restated as a 6-axis reshape/transpose of the token index grid.
    """
    gt, gh, gw = tile_grid_dims(grid, tile)
    st, sh, sw = tile
    idx = np.arange(grid[0] * grid[1] * grid[2], dtype=np.int64)
    return idx.reshape(gt, st, gh, sh, gw, sw).transpose(0, 2, 4, 1, 3, 5).reshape(-1)


# --------------------------------------------------------------------------
# sliding-tile windows -- fp8sta/sparsity.py
# --------------------------------------------------------------------------
def axis_interval(x: int, dim: int, extent: int) -> tuple[int, int]:
    """Admissible key coordinates [lo, hi] for query coordinate x (sparsity.py:43-45, :96-109)."""
    back, fwd = (extent - 1) // 2, extent // 2
    return max(0, x - back), min(dim - 1, x + fwd)


def window_lists(dims: tuple[int, int, int], window: tuple[int, int, int]):
    """CSR of ascending admissible key tiles per query tile (sparsity.py:63-75, :112-132)."""
    dt, dh, dw = dims
    if min(dims) < 1:
        raise ValueError(f"tile grid dims must be >= 1, got {dims}")
    offs = [0]
    ids = []
    for ut in range(dt):
        t0, t1 = axis_interval(ut, dt, window[0])
        for uh in range(dh):
            h0, h1 = axis_interval(uh, dh, window[1])
            for uw in range(dw):
                w0, w1 = axis_interval(uw, dw, window[2])
                for vt in range(t0, t1 + 1):
                    for vh in range(h0, h1 + 1):
                        base = (vt * dh + vh) * dw
                        ids.extend(range(base + w0, base + w1 + 1))
                offs.append(len(ids))
    return np.asarray(offs, dtype=np.int32), np.asarray(ids, dtype=np.int32)


def density_of(offs: np.ndarray) -> float:
    """Admissible-pair fraction (sparsity.py:141-144)."""
    m = len(offs) - 1
    return int(offs[-1]) / (m * m)


def flops_sparse_of(L: int, d: int, density: float) -> int:
    """round(density * 4 L^2 d) (metrics.py:91-102)."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    return round(density * 4 * L * L * d)


# --------------------------------------------------------------------------
# schedule -- fp8sta/schedule.py
# --------------------------------------------------------------------------
def regime_of(t: int, total: int, alpha1: float, alpha2: float) -> str:
    """Step -> regime with boundary steps in the earlier regime (schedule.py:41-50)."""
    if not 1 <= t <= total:
        raise ValueError(f"step {t} out of range [1, {total}]")
    if t <= math.floor(alpha1 * total):
        return "early"
    if t <= math.floor(alpha2 * total):
        return "mid"
    return "late"


def schedule_valid(alpha1, alpha2, total, tile_vols, win_vols) -> bool:
    """Ordering rules of schedule.validate (schedule.py:76-104); vols = (early, mid, late)."""
    ge, gm, gl = tile_vols
    we, wm, wl = win_vols
    return (0 < alpha1 < alpha2 < 1) and total >= 1 and ge > gl > gm and wm > wl > we


# --------------------------------------------------------------------------
# attention -- fp8sta/attention.py
# --------------------------------------------------------------------------
def _softmax_scale(d: int, scale) -> np.float32:
    """f32(1/sqrt(d)) unless given; must be > 0 (attention.py:83-88)."""
    if scale is None:
        return np.float32(1.0 / math.sqrt(d))
    if not scale > 0:
        raise ValueError("softmax_scale must be > 0")
    return np.float32(scale)


def _tile_attention(qv, kv, vv, tv, offs, ids, q_fac, k_fac, v_fac, scale, quant_p: bool):
    """Per-query-tile masked attention with a two-pass softmax (attention.py:91-149).

    f32 logits from the decoded values, per-(tile,tile) factor applied after
    the GEMM, f64 denominator, normalised weights rounded to E4M3 at 448 when
    ``quant_p``, f32 output GEMM scaled by per-channel factors.
    """
    L, d = qv.shape
    M = L // tv
    out = np.empty((L, d), dtype=np.float32)
    lanes = np.arange(tv, dtype=np.int64)
    for u in range(M):
        keys = ids[offs[u]:offs[u + 1]].astype(np.int64)
        rows = (keys[:, None] * tv + lanes[None, :]).reshape(-1)
        k_blk, v_blk = kv[rows], vv[rows]
        col_fac = np.repeat(k_fac[keys], tv) * (q_fac[u] * scale)
        for r0 in range(u * tv, (u + 1) * tv, 1024):
            r1 = min(r0 + 1024, (u + 1) * tv)
            s = qv[r0:r1] @ k_blk.T
            s *= col_fac[None, :]
            if not np.isfinite(s).all():
                raise FloatingPointError("non-finite attention logits")
            s -= s.max(axis=1, keepdims=True)
            np.exp(s, out=s)
            den = s.sum(axis=1, dtype=np.float64, keepdims=True)
            s /= den.astype(np.float32)
            if quant_p:
                s *= np.float32(448.0)
                s = grid_round(s, E4M3)
            o = s @ v_blk
            o *= v_fac[None, :]
            out[r0:r1] = o
    return out


def fp8_sparse_forward(q, k, v, tv, offs, ids, fmt: Fmt = E4M3, softmax_scale=None):
    """Quantised sparse forward on tile-contiguous single-head inputs (attention.py:179-208).

    Returns (out f32 [L,d], dict of the intermediate codes/scales).
    """
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    for name, a in (("q", q), ("k", k), ("v", v)):
        if not np.isfinite(a).all():
            raise ValueError(f"{name} contains non-finite values")
    scale = _softmax_scale(q.shape[1], softmax_scale)
    qc, qs = quantize_qk_tilewise(q, tv, fmt)
    kc, ks = quantize_qk_tilewise(k, tv, fmt)
    vc, vs = quantize_v_channelwise(v, fmt)
    out = _tile_attention(
        decode(qc, fmt), decode(kc, fmt), decode(vc, fmt), tv, offs, ids,
        qs.astype(np.float32), ks.astype(np.float32), (vs * (1.0 / 448.0)).astype(np.float32),
        scale, quant_p=True,
    )
    return out, dict(q_codes=qc, q_scales=qs, k_codes=kc, k_scales=ks, v_codes=vc, v_scales=vs)


def normalized_rows(q, k, v, tv, offs, ids, rows, fmt: Fmt = E4M3, softmax_scale=None):
    """Per-row intermediates of the reference's quantised forward for selected rows (attention.py:179-208,
    _engine :118-149): yields (row, x = f32(p) * 448 before rounding, decoded V rows of its keys, v_fac).
    The same arithmetic as _tile_attention restricted to single rows (the f32 GEMM of one row)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    scale = _softmax_scale(q.shape[1], softmax_scale)
    qc, qs = quantize_qk_tilewise(q, tv, fmt)
    kc, ks = quantize_qk_tilewise(np.asarray(k, np.float32), tv, fmt)
    vc, vs = quantize_v_channelwise(np.asarray(v, np.float32), fmt)
    qv, kv, vv = decode(qc, fmt), decode(kc, fmt), decode(vc, fmt)
    q_fac, k_fac = qs.astype(np.float32), ks.astype(np.float32)
    v_fac = (vs * (1.0 / 448.0)).astype(np.float32)
    lanes = np.arange(tv, dtype=np.int64)
    for r in rows:
        u = int(r) // tv
        keys = ids[offs[u]:offs[u + 1]].astype(np.int64)
        kr = (keys[:, None] * tv + lanes[None, :]).reshape(-1)
        s = qv[r:r + 1] @ kv[kr].T
        s *= (np.repeat(k_fac[keys], tv) * (q_fac[u] * scale))[None, :]
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)
        s /= s.sum(axis=1, dtype=np.float64, keepdims=True).astype(np.float32)
        s *= np.float32(448.0)
        yield int(r), s[0], vv[kr], v_fac


def fp8_sparse_rows(q, k, v, tv, offs, ids, rows, fmt: Fmt = E4M3, softmax_scale=None) -> np.ndarray:
    """fp8_sparse_forward's output for selected query rows only ([len(rows), d] f32): the same arithmetic
    (attention.py:133-149) one row at a time, for tiles too large for the full-matrix pass (24576 tokens)."""
    out = np.empty((len(rows), np.asarray(q).shape[1]), dtype=np.float32)
    for i, (_, x, vrows, v_fac) in enumerate(normalized_rows(q, k, v, tv, offs, ids, rows, fmt, softmax_scale)):
        out[i] = (grid_round(x, E4M3)[None, :] @ vrows)[0] * v_fac
    return out


def p_flip_budget(q, k, v, tv, offs, ids, rows, fmt: Fmt = E4M3, softmax_scale=None, rel: float = 2.0 ** -19):
    """Bound on how far a correct implementation of the normalised-P forward may move each output element
    of `rows` away from the reference through P-code flips.

    The reference rounds x = 448 p onto the E4M3 grid (attention.py:143-145).  x itself depends on a float32
    GEMM, exp and division whose last bits differ between numpy builds and a GPU (numpy's f32 exp is not
    correctly rounded: up to 2 ulp), so an x within `rel` (relative) of a rounding midpoint may round to
    either neighbour.  Each such weight can move output channel c by (hi - lo) |V_j,c| v_fac[c].  Returns
    (budget [len(rows), d] float64, number of ambiguous weights)."""
    grid = _VALUES["e4m3"][:0x7F].astype(np.float64)  # non-negative finite E4M3 values, ascending
    d = np.asarray(q).shape[1]
    budget = np.zeros((len(rows), d), dtype=np.float64)
    n_amb = 0
    for i, (_, x, vrows, v_fac) in enumerate(normalized_rows(q, k, v, tv, offs, ids, rows, fmt, softmax_scale)):
        xd = x.astype(np.float64)
        hi_i = np.clip(np.searchsorted(grid, xd, side="left"), 1, len(grid) - 1)
        lo, hi = grid[hi_i - 1], grid[hi_i]
        amb = np.abs(xd - 0.5 * (lo + hi)) <= rel * np.maximum(xd, 2.0 ** -6)
        amb &= xd < grid[-1]
        if amb.any():
            n_amb += int(amb.sum())
            budget[i] = ((hi - lo)[amb][:, None] * np.abs(vrows[amb].astype(np.float64))).sum(0) * v_fac
    return budget, n_amb


def sparse_forward_f32(q, k, v, tv, offs, ids, softmax_scale=None):
    """Full-precision sparse oracle == the passthrough branch (attention.py:165-176, :192-194)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    M = q.shape[0] // tv
    ones = np.ones(M, dtype=np.float32)
    return _tile_attention(q, np.asarray(k, np.float32), np.asarray(v, np.float32), tv, offs, ids,
                           ones, ones, np.ones(q.shape[1], np.float32),
                           _softmax_scale(q.shape[1], softmax_scale), quant_p=False)


POLY_PER8 = 4  # softmax.cuh FPSA_POLY_PER8


def _poly_columns(block: int = 128, per8: int = POLY_PER8) -> np.ndarray:
    """Columns of a key block whose exp2 the GPU kernel evaluates with its polynomial
    (softmax.cuh softmax_chunk32): columns 2, 3, 6, 7 of every group of 8 (per8 = 4, the
    build default), columns 6 and 7 (per8 = 2), 2-7 (6), all (8) or none (0); the rest use MUFU ex2."""
    col = np.arange(block) % 8
    if per8 == 8:
        return np.ones(block, dtype=bool)
    if per8 == 6:
        return col >= 2
    if per8 == 4:
        return col % 4 >= 2
    if per8 == 2:
        return col >= 6
    return np.zeros(block, dtype=bool)


def _exp2_poly(x: np.ndarray) -> np.ndarray:
    """The kernel's FMA-pipe exp2: x clamped to [-126, 130], j = rint(x), degree-2 minimax on x - j."""
    x = np.clip(x, -126.0, 130.0)
    j = np.rint(x)
    f = x - j
    y = (np.float32(0.238487109541893) * f + np.float32(0.703453540802002)) * f + np.float32(1.0004364252090454)
    return np.ldexp(y, j.astype(np.int64))


def packed_keys(tv: int) -> bool:
    """Whether the kernel runs packed key blocks for tile volume tv (fpsa_attn.cu fpsa_attn_fwd: 128
    consecutive keys of the concatenated window tiles per block, no padding keys)."""
    return tv % 16 == 0 and tv > 128 and tv % 128 != 0


def onepass_forward(codes: dict, tv, offs, ids, fmt: Fmt = E4M3, softmax_scale=None, block=128, tau=0.0,
                    poly=False, return_redo=False, packed=None):
    """Emulation of the GPU kernel's schedule (NOT the reference semantics).

    Work item = 128 query rows of a tile.  Keys are visited per key tile in
    `block`-key blocks (the last block of a tile is shorter).  The reference
    max m of a row is the max of its first key block; the unnormalised weights
    448 * 2^(x - m - tau) are rounded to E4M3 before the PV product and the
    denominator is the sum of the rounded weights (the kernel accumulates it
    with the PV MMA through a column of ones).  If any rounded weight of an
    item reaches 448 (possible saturation), the item is recomputed with the
    exact row max and tau = 0 (the kernel's redo launch).  Used to check the
    CUDA kernel tightly; the reference-facing check is against
    ``fp8_sparse_forward``.  With packed key blocks (``packed_keys(tv)``) a
    key's column in its block -- which decides polynomial or MUFU exp2 -- is
    its position in the concatenated key stream modulo 128.
    """
    if packed is None:
        packed = packed_keys(tv)
    qv = decode(codes["q_codes"], fmt).astype(np.float64)
    kv = decode(codes["k_codes"], fmt).astype(np.float64)
    vv = decode(codes["v_codes"], fmt).astype(np.float64)
    qs, ks, vs = codes["q_scales"], codes["k_scales"], codes["v_scales"]
    L, d = qv.shape
    M = L // tv
    scale = float(_softmax_scale(d, softmax_scale))
    sl = float(np.float32(scale / math.log(2.0)))
    out = np.empty((L, d), dtype=np.float64)
    redo = []
    pc_all = _poly_columns(block)
    for u in range(M):
        for r0 in range(0, tv, 128):
            rows = slice(u * tv + r0, u * tv + min(r0 + 128, tv))
            qrows = qv[rows]
            blocks = []
            for i, vt in enumerate(ids[offs[u]:offs[u + 1]]):
                c = float(np.float32(np.float32(np.float32(qs[u]) * np.float32(ks[vt])) * np.float32(sl)))
                if packed:
                    # first block of the stream separate (it sets the reference max), then whole tiles
                    starts = [0, block] if i == 0 else [0]
                    ends = [block, tv] if i == 0 else [tv]
                    for b0, b1 in zip(starts, ends):
                        blocks.append((c, vt * tv + b0, vt * tv + b1, (i * tv + b0) % block))
                else:
                    for b0 in range(0, tv, block):
                        b1 = min(b0 + block, tv)
                        blocks.append((c, vt * tv + b0, vt * tv + b1, 0))

            def run(m, t):
                lsum = np.zeros(qrows.shape[0])
                acc = np.zeros((qrows.shape[0], d))
                over = False
                for c, k0, k1, col0 in blocks:
                    x = (qrows @ kv[k0:k1].T) * c
                    xe = x - m[:, None] + (math.log2(448.0) - t)
                    p = np.exp2(xe)
                    if poly:
                        pc = pc_all[(col0 + np.arange(x.shape[1])) % block]
                        p[:, pc] = _exp2_poly(xe[:, pc])
                    pq = grid_round(p.astype(np.float32), E4M3).astype(np.float64)
                    over |= bool(np.any(pq >= 448.0))
                    lsum += pq.sum(axis=1)
                    acc += pq @ vv[k0:k1]
                return acc / lsum[:, None] * vs[None, :], over

            c0, k0, k1, _ = blocks[0]
            o, over = run((qrows @ kv[k0:k1].T).max(axis=1) * c0, tau)
            if over:
                m = np.max([((qrows @ kv[a:b].T) * c).max(axis=1) for c, a, b, _ in blocks], axis=0)
                o, _ = run(m, 0.0)
                redo.append((u, r0 // 128))
            out[rows] = o
    res = out.astype(np.float32)
    return (res, redo) if return_redo else res


def bf16_round(x) -> np.ndarray:
    """f32 -> nearest-even bfloat16, returned as f32 (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def passthrough_emulation(q, k, v, tv, offs, ids, softmax_scale=None, block=128):
    """Emulation of the GPU passthrough kernel's schedule (fpsa_attn_bf16.cu), NOT the reference.

    Operands rounded to bf16; per 128-row work item the keys are visited in
    `block`-key blocks (per key tile, the last block of a tile shorter); the
    reference max m of a row is the max of its first key block (x units:
    s * f32(scale log2 e)); P = 2^(x - m) is summed unrounded into l and
    rounded to bf16 for the PV product; out = O / l.  (The kernel's exact-max
    redo triggers only when l overflows f32, which these inputs never do.)
    """
    qv = bf16_round(q).astype(np.float64)
    kv = bf16_round(k).astype(np.float64)
    vv = bf16_round(v).astype(np.float64)
    L, d = qv.shape
    M = L // tv
    c = float(np.float32(np.float32(_softmax_scale(d, softmax_scale)) * np.float32(1.4426950408889634)))
    out = np.empty((L, d), dtype=np.float64)
    for u in range(M):
        blocks = [(vt * tv + b0, vt * tv + min(b0 + block, tv))
                  for vt in ids[offs[u]:offs[u + 1]] for b0 in range(0, tv, block)]
        for r0 in range(0, tv, 128):
            rows = slice(u * tv + r0, u * tv + min(r0 + 128, tv))
            qrows = qv[rows]
            k0, k1 = blocks[0]
            m = (qrows @ kv[k0:k1].T).astype(np.float32).max(axis=1).astype(np.float64) * c
            lsum = np.zeros(qrows.shape[0])
            acc = np.zeros((qrows.shape[0], d))
            for k0, k1 in blocks:
                x = (qrows @ kv[k0:k1].T).astype(np.float32).astype(np.float64) * c - m[:, None]
                p = np.exp2(x).astype(np.float32)
                lsum += p.sum(axis=1, dtype=np.float64)
                acc += bf16_round(p).astype(np.float64) @ vv[k0:k1]
            out[rows] = acc / lsum[:, None]
    return out.astype(np.float32)


# --------------------------------------------------------------------------
# metrics used as parity checkers -- fp8sta/metrics.py:41-62
# --------------------------------------------------------------------------
def cosine(a, b) -> float:
    x = np.asarray(a, np.float64).ravel()
    y = np.asarray(b, np.float64).ravel()
    mx, my = np.abs(x).max(), np.abs(y).max()
    if mx == 0.0 and my == 0.0:
        return 1.0
    if mx == 0.0 or my == 0.0:
        return 0.0
    x, y = x / mx, y / my
    return float(min(1.0, max(-1.0, np.dot(x, y) / math.sqrt(np.dot(x, x) * np.dot(y, y)))))


def max_abs(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


# --------------------------------------------------------------------------
# synthetic inputs -- fp8sta/experiment.py:90-115 (Philox keyed by coordinates)
# --------------------------------------------------------------------------
def gen_inputs(seed: int, step: int, head: int, L: int, d: int, dist: str = "gaussian",
               sigma: float = 1.0, lo: float = -1.0, hi: float = 1.0):
    """q, k, v float32 [L, d] exactly as the reference draws them (tile-contiguous rows)."""
    out = []
    for tag in (1, 2, 3):  # q, k, v
        key = ((((step << 24) | (head << 8) | tag)) << 64) | (seed & 0xFFFFFFFFFFFFFFFF)
        gen = np.random.Generator(np.random.Philox(key=key))
        if dist == "gaussian":
            x = np.float32(sigma) * gen.standard_normal((L, d), dtype=np.float32)
        elif dist == "uniform":
            x = gen.random((L, d), dtype=np.float32) * np.float32(hi - lo) + np.float32(lo)
        elif dist == "heavy":
            col = (10.0 ** gen.uniform(-1.0, 1.0, size=d)).astype(np.float32)
            x = gen.standard_normal((L, d), dtype=np.float32) * col[None, :]
        else:
            raise ValueError(f"unknown distribution {dist!r}")
        out.append(x)
    return tuple(out)
