"""Pin the CPU oracle (oracle/fpsa_oracle.py) to the reference's own outputs.

The fixtures in tests/golden were produced by tests/golden/make_golden.py,
which imports the reference package fp8sta (/root/reference/pkg/src) in the
build container.  Bit-exact: code tables, encode (f64 and f32 inputs, both
formats), adversarial near-tie tile quantisation, tile permutations, window
lists, densities, schedule regimes, per-case codes/scales and the Philox
input generator.  Tolerance-pinned: attention outputs (float32 BLAS summation
order is platform dependent), here ≤ 1e-5 · max|ref|.
"""

import numpy as np
import pytest

import oracle as O
from oracle import fpsa_oracle as OF
from conftest import CASE_NAMES, golden_cases

FMTS = [O.E4M3, O.E5M2]


# ----------------------------------------------------------------- FP8 codec (fp8.py)
@pytest.mark.parametrize("fmt", FMTS, ids=lambda f: f.name)
def test_code_table(codec_golden, fmt):
    ref = codec_golden[f"table_{fmt.name}"]
    got = OF._code_values(fmt)
    assert np.array_equal(np.isnan(ref), np.isnan(got))
    ok = ~np.isnan(ref)
    assert np.array_equal(ref[ok], got[ok])
    assert np.array_equal(np.signbit(ref[ok]), np.signbit(got[ok]))


@pytest.mark.parametrize("fmt", FMTS, ids=lambda f: f.name)
@pytest.mark.parametrize("kind", ["enc", "enc32"])
def test_encode_matches_reference(codec_golden, fmt, kind):
    x = codec_golden[f"{kind}_x_{fmt.name}"]
    ref = codec_golden[f"{kind}_c_{fmt.name}"]
    if not fmt.has_inf:
        # the reference raises on inf for E4M3; the fixture holds only finite values there
        assert np.isfinite(x).all()
    assert np.array_equal(O.encode(x, fmt), ref)


def test_encode_kats():
    """Known answers of test_fp8.py:55-110: ties, saturation, subnormal, signed zero, errors."""
    e = O.E4M3
    assert O.encode(np.array([1.0625]), e)[0] == O.encode(np.array([1.0]), e)[0]  # tie -> even
    assert O.encode(np.array([1.1875]), e)[0] == O.encode(np.array([1.25]), e)[0]  # tie -> even (up)
    assert O.encode(np.array([1e9]), e)[0] == 0x7E  # saturate to 448
    assert O.encode(np.array([-1e9]), e)[0] == 0xFE
    assert O.encode(np.array([2.0 ** -9]), e)[0] == 0x01  # smallest subnormal
    assert O.encode(np.array([2.0 ** -10]), e)[0] == 0x00  # tie to even zero
    assert O.encode(np.array([-0.0]), e)[0] == 0x80
    assert O.encode(np.array([-(2.0 ** -11)]), e)[0] == 0x80  # rounds to -0
    with pytest.raises(ValueError):
        O.encode(np.array([np.nan]), e)
    with pytest.raises(ValueError):
        O.encode(np.array([np.inf]), e)
    assert O.encode(np.array([np.inf]), O.E5M2)[0] == 0x7C
    with pytest.raises(ValueError):
        O.decode(np.array([0x7F], np.uint8), e)


def test_all_codes_round_trip():
    for fmt in FMTS:
        vals = OF._code_values(fmt)
        codes = np.arange(256, dtype=np.uint8)
        ok = np.isfinite(vals)
        assert np.array_equal(O.encode(vals[ok], fmt), codes[ok])


def test_grid_round_matches_decode_encode():
    """round_to_grid on grid points, midpoints and +-1 ulp (test_fp8.py:216-233)."""
    vals = OF._code_values(O.E4M3)[:127].astype(np.float32)
    mids = ((vals[:-1].astype(np.float64) + vals[1:]) / 2).astype(np.float32)
    xs = np.concatenate([vals, mids, np.nextafter(mids, np.float32(0)), np.nextafter(mids, np.float32(1e9)),
                         np.float32([448.0, 464.0, 500.0])])
    got = O.grid_round(xs, O.E4M3)
    assert got.max() == 448.0
    assert np.array_equal(got, O.decode(O.encode(xs, O.E4M3), O.E4M3))


# ----------------------------------------------------------------- quantisation (quantize.py)
def test_adversarial_tile_quantisation(codec_golden):
    x = codec_golden["adv_x"]
    rows = int(codec_golden["adv_tile_rows"])
    codes, scales = O.quantize_qk_tilewise(x, rows, O.E4M3)
    assert np.array_equal(scales, codec_golden["adv_scales"])
    assert np.array_equal(codes, codec_golden["adv_codes"])


def test_scale_kats():
    """quantize.py:102-108 / test_quantize.py:26-94."""
    assert O.block_scales(np.array([3.0]))[0] == 3.0 / 448.0
    assert O.block_scales(np.array([0.0]))[0] == 1.0
    assert O.block_scales(np.array([1e-320]))[0] == np.finfo(np.float64).tiny
    with pytest.raises(ValueError):
        O.block_scales(np.array([np.inf]))
    x = np.zeros((4, 2), np.float32)
    x[:, 0] = [1, -7, 2, 0]
    x[:, 1] = [0.5, 0.25, -1, 1]
    codes, scales = O.quantize_v_channelwise(x)
    assert np.array_equal(scales, [7 / 448, 1 / 448])
    assert codes[1, 0] == 0xFE  # -7/(7/448) = -448


@pytest.mark.parametrize("name", CASE_NAMES)
def test_case_inputs_and_codes(attn_golden, name):
    """Philox restatement (experiment.py:90-115) + codes and scales of every golden case."""
    c = golden_cases(attn_golden)[name]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    s = attn_golden[name + "__in_sum"]
    assert q.astype(np.float64).sum() == s[0] and k.astype(np.float64).sum() == s[1]
    assert v.astype(np.float64).sum() == s[2] and q[0, 0] == s[3] and v[-1, -1] == s[4]
    fmt = O.FORMATS[c["fmt"]]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    rows = attn_golden[name + "__rows"]
    for nm, x in (("q", q), ("k", k)):
        codes, scales = O.quantize_qk_tilewise(x, tv, fmt)
        assert np.array_equal(scales, attn_golden[f"{name}__{nm}_scales"])
        got = codes if L <= 256 else codes[rows]
        assert np.array_equal(got, attn_golden[f"{name}__{nm}_codes_rows"])
    codes, scales = O.quantize_v_channelwise(v, fmt)
    assert np.array_equal(scales, attn_golden[f"{name}__v_scales"])
    assert np.array_equal(codes if L <= 256 else codes[rows], attn_golden[f"{name}__v_codes_rows"])


# ----------------------------------------------------------------- layout / windows / schedule
@pytest.mark.parametrize("key", ["perm_4_8_8_2_4_4", "perm_6_8_8_3_4_4", "perm_6_10_16_3_10_4",
                                 "perm_7_9_16_7_9_8", "perm_4_6_10_2_3_5"])
def test_tile_perm(codec_golden, key):
    v = [int(x) for x in key.split("_")[1:]]
    assert np.array_equal(O.tile_perm(tuple(v[:3]), tuple(v[3:])), codec_golden[key])


def test_tile_perm_kat_and_errors():
    # grid 1x2x2, tile 1x1x2 -> tiles rows: [0,1],[2,3]; tile 1x2x1 -> [0,2],[1,3] (test_grid.py:68-76)
    assert O.tile_perm((1, 2, 2), (1, 2, 1)).tolist() == [0, 2, 1, 3]
    with pytest.raises(ValueError, match="indivisible grid: axis h has 30 tokens, not divisible by tile extent 4"):
        O.tile_grid_dims((21, 30, 52), (3, 4, 4))


MASK_KEYS = ["2_2_2_2_2_2", "7_3_13_3_3_5", "7_9_5_3_3_3", "7_9_5_5_5_3", "4_4_4_6_6_6", "3_5_2_1_4_2",
             "11_9_5_5_5_3", "3_3_5_3_3_1", "3_5_10_3_3_3"]


@pytest.mark.parametrize("key", MASK_KEYS)
def test_window_lists(codec_golden, key):
    v = [int(x) for x in key.split("_")]
    offs, ids = O.window_lists(tuple(v[:3]), tuple(v[3:]))
    assert np.array_equal(offs.astype(np.int64), codec_golden[f"mask_offs_{key}"])
    assert np.array_equal(ids.astype(np.int64), codec_golden[f"mask_ids_{key}"])
    assert O.density_of(offs) == float(codec_golden[f"mask_density_{key}"])


def test_window_kats():
    """1D densities [2,3,3,2] -> 0.625 (test_sparsity.py:73-76); even window reach."""
    offs, ids = O.window_lists((1, 1, 4), (1, 1, 3))
    assert np.diff(offs).tolist() == [2, 3, 3, 2] and O.density_of(offs) == 0.625
    assert O.axis_interval(5, 10, 4) == (4, 7)  # back 1, forward 2
    assert O.axis_interval(0, 10, 6) == (0, 3)


def test_schedule_regimes(codec_golden):
    assert [["early", "mid", "late"].index(O.regime_of(t, 50, 0.2, 0.7)) for t in range(1, 51)] == \
        codec_golden["sched_regimes_50"].tolist()
    for D, a1, a2 in [(7, 0.3, 0.6), (1000, 0.2, 0.7), (13, 0.5, 0.9)]:
        got = [["early", "mid", "late"].index(O.regime_of(t, D, a1, a2)) for t in range(1, D + 1)]
        assert got == codec_golden[f"sched_regimes_{D}_{a1}_{a2}"].tolist()


def test_flops_accounting():
    offs, _ = O.window_lists((7, 9, 5), (5, 5, 3))
    L, d, tv = 75600, 128, 240
    assert O.flops_sparse_of(L, d, O.density_of(offs)) == int(offs[-1]) * 4 * tv * tv * d


# ----------------------------------------------------------------- attention (attention.py)
@pytest.mark.parametrize("name", ["c0_toy", "c0_toy_full", "small_d128", "tv120_d128", "tv256_d64"])
def test_attention_vs_reference(attn_golden, name):
    c = golden_cases(attn_golden)[name]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    out, _ = O.fp8_sparse_forward(q, k, v, tv, offs, ids, O.FORMATS[c["fmt"]])
    rows = attn_golden[name + "__rows"]
    ref = attn_golden[name + "__out"]
    assert O.max_abs(out[rows], ref) <= 1e-5 * float(np.abs(ref).max())
    if name + "__sparse_ref" in attn_golden.files:
        f32 = O.sparse_forward_f32(q, k, v, tv, offs, ids)
        sref = attn_golden[name + "__sparse_ref"]
        assert O.max_abs(f32[rows], sref) <= 1e-5 * float(np.abs(sref).max())


@pytest.mark.parametrize("name", CASE_NAMES)
def test_passthrough_vs_reference(attn_golden, name):
    """The oracle's full-precision branch == the reference's sparse_reference / passthrough
    (attention.py:165-176, :192-194) on every golden case; the GPU passthrough kernel's
    emulation (bf16 operands, first-block max, bf16 P) stays within bf16 error of it."""
    c = golden_cases(attn_golden)[name]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    rows = attn_golden[name + "__rows"]
    sref = attn_golden[name + "__sparse_ref"]
    f32 = O.sparse_forward_f32(q, k, v, tv, offs, ids)
    assert O.max_abs(f32[rows], sref) <= 1e-5 * float(np.abs(sref).max())
    # bf16 operands: logit error ~ |s| 2^-9, largest for the heavy-tailed inputs (3.5e-2 rel there)
    emu = O.passthrough_emulation(q, k, v, tv, offs, ids)
    assert O.cosine(emu[rows], sref) >= 0.9999
    assert O.max_abs(emu[rows], sref) <= 5e-2 * float(np.abs(sref).max())
    # on bf16-exact inputs only the bf16 rounding of P remains
    rb = O.sparse_forward_f32(O.bf16_round(q), O.bf16_round(k), O.bf16_round(v), tv, offs, ids)
    assert O.cosine(emu, rb) >= 0.999995
    assert O.max_abs(emu, rb) <= 5e-3 * float(np.abs(rb).max())


def test_attention_row_stochastic_and_full_window_dense():
    """Full window == dense attention; exactly representable inputs are lossless in Q/K/V."""
    L, d, tv = 64, 16, 16
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((L, d)).astype(np.float32) for _ in range(3))
    offs, ids = O.window_lists((1, 1, 4), (1, 1, 8))
    f32 = O.sparse_forward_f32(q, k, v, tv, offs, ids)
    s = (q @ k.T) * np.float32(1 / np.sqrt(d))
    p = np.exp(s - s.max(1, keepdims=True))
    dense = (p / p.sum(1, keepdims=True)) @ v
    assert np.abs(f32 - dense).max() < 1e-5


def test_onepass_emulation_close_to_reference(attn_golden):
    """The GPU kernel's schedule (oracle.onepass_forward) stays within the stated tolerance."""
    c = golden_cases(attn_golden)["small_d128"]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    ref, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    emu = O.onepass_forward(codes, tv, offs, ids, tau=8.0, poly=True)
    assert O.cosine(emu, ref) >= 0.999
    assert O.max_abs(emu, ref) <= 0.1 * float(np.abs(ref).max())



@pytest.mark.parametrize("name", CASE_NAMES)
def test_sampled_rows_vs_reference(attn_golden, name):
    """oracle.fp8_sparse_rows (the large-tile parity checker: one query row at a time) against the
    reference's own outputs on the golden rows (attention.py:179-208)."""
    c = golden_cases(attn_golden)[name]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    rows = attn_golden[name + "__rows"]
    ref = attn_golden[name + "__out"]
    got = O.fp8_sparse_rows(q, k, v, tv, offs, ids, rows, O.FORMATS[c["fmt"]])
    budget, _ = O.p_flip_budget(q, k, v, tv, offs, ids, rows, O.FORMATS[c["fmt"]])
    assert (np.abs(got.astype(np.float64) - ref) <= 1e-5 * float(np.abs(ref).max()) + budget).all()
