"""The quantiser's exact-tie table (fpsa_quant.cu: build_tie_table / resolve_tie), restated in numpy and checked
against the oracle's f64 encoding (quantize.py:111-134: codes = encode(x_f64 / RN64(peak / maxv))).

With bf16 data x and a bf16 peak P, the GPU's f32 fast path brackets x * f32(maxv / P) by +-2^-20; when the two
bracket ends encode differently the element is an exact tie (the quotient x * maxv / P is a rounding midpoint
o * 2^f of the fp8 grid), and the reference's code then depends only on P's significand and on o.  These tests
check both statements on many random bf16 pairs, on CPU, independently of the GPU kernel.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

FMTS = {"e4m3": (O.E4M3, 448.0, 3), "e5m2": (O.E5M2, 57344.0, 2)}


def tie_odd(k, mbits):
    m = 1 << mbits
    return 2 * m + 1 + 2 * k if k < m else 2 * (k - m) + 1


def tie_class(code, mbits):
    mag = int(code) & 0x7F
    m = mag & ((1 << mbits) - 1)
    return m if (mag >> mbits) else (1 << mbits) + m


def tie_table(maxv, mbits):
    """(up, even, valid) bit masks per peak significand 128..255, the same IEEE f64 steps as the kernel."""
    classes = 2 << mbits
    table = []
    for pm in range(128, 256):
        up = even = valid = 0
        s = np.float64(pm) / np.float64(maxv)
        for k in range(classes):
            o = tie_odd(k, mbits)
            xo = np.float64(o * pm)
            x = xo / np.float64(maxv)
            if Fraction(float(x)) * Fraction(maxv) != Fraction(o * pm):
                continue  # the tying input is not representable: this class cannot tie
            valid |= 1 << k
            q = x / s
            if q > o:
                up |= 1 << k
            elif q == o:
                even |= 1 << k
        table.append((up, even, valid))
    return table


def bf16(a):
    """Round float32 values to bf16 (RNE) and return them as float32."""
    u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("fmt_name", ["e4m3", "e5m2"])
def test_ambiguous_elements_are_exact_ties_and_the_table_decides_them(fmt_name):
    fmt, maxv, mbits = FMTS[fmt_name]
    table = tie_table(maxv, mbits)
    rng = np.random.default_rng(5)
    n_amb = 0
    for trial in range(60):
        # tie-rich blocks: multiples of peak / 2^k, plus Gaussian ones, with peaks of every significand class
        peak = bf16(np.float32(np.ldexp(1.0 + rng.integers(0, 128) / 128.0, int(rng.integers(-8, 9)))))
        if trial % 2:
            x = bf16(rng.integers(-255, 256, 4096).astype(np.float32) * (peak / np.float32(256)))
        else:
            x = bf16(rng.standard_normal(4096).astype(np.float32) * peak / np.float32(4))
        x = np.concatenate([x, [peak]]).astype(np.float32)
        p = np.float32(np.abs(x).max())
        s = np.float64(p) / np.float64(maxv)
        ref = O.encode(x.astype(np.float64) / s, fmt)  # the reference: f64 quotient, RNE
        r = np.float32(maxv) / p  # the kernel's bracket (bracket_f32)
        lo = O.encode((x * np.float32(r * np.float32(0.99999904632568359375))).astype(np.float32), fmt)
        hi = O.encode((x * np.float32(r * np.float32(1.00000095367431640625))).astype(np.float32), fmt)
        assert np.array_equal(lo[lo == hi], ref[lo == hi])  # the fast path
        pm = int((p.view(np.uint32) >> 16) & 0x7F)
        up, even, valid = table[pm]
        for i in np.flatnonzero(lo != hi):
            q = Fraction(float(x[i])) * Fraction(maxv) / Fraction(float(p))
            mid = (Fraction(float(O.decode(np.uint8(lo[i] & 0x7F), fmt))) +
                   Fraction(float(O.decode(np.uint8(hi[i] & 0x7F), fmt)))) / 2
            assert abs(q) == mid, "an ambiguous element that is not an exact tie"
            bit = 1 << tie_class(lo[i], mbits)
            assert valid & bit
            code = hi[i] if up & bit else ((hi[i] if lo[i] & 1 else lo[i]) if even & bit else lo[i])
            assert code == ref[i]
            n_amb += 1
    print(f"{fmt_name}: {n_amb} ambiguous elements, all exact ties decided by the table")
    assert n_amb > 100  # the tie-rich blocks exercise the table
