"""Drop-in breadth of the reference API on the GPU: the element codec (encode / decode /
quantize_dequantize / dequantize_tensor), f64 and any-width quantisation, head dims other than 64 / 128
in fp8_sparse_forward, and natural-order tiles above 2048 tokens (the reference default_schedule's
3072- and 24576-token tiles).  Bit-exact against the reference's golden vectors or the oracle."""

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fpsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_04648_b200 as m

    return m


@pytest.mark.parametrize("fmt", ["e4m3", "e5m2"])
def test_encode_decode_vs_reference_goldens(fpsa, codec_golden, fmt):
    """fp8.encode of 40k f64 and f32 reals (incl. ties, saturation, subnormals, signed zero) and fp8.decode of
    every non-NaN code equal the reference's outputs (tests/golden/codec_layout.npz)."""
    F = fpsa.FORMATS[fmt]
    assert np.array_equal(fpsa.encode(codec_golden[f"enc_x_{fmt}"], F), codec_golden[f"enc_c_{fmt}"])
    assert np.array_equal(fpsa.encode(codec_golden[f"enc32_x_{fmt}"], F), codec_golden[f"enc32_c_{fmt}"])
    table = codec_golden[f"table_{fmt}"]
    ok = ~np.isnan(table)
    dec = fpsa.decode(np.arange(256, dtype=np.uint8)[ok], F)
    assert dec.dtype == np.float32 and np.array_equal(dec.astype(np.float64), table[ok])
    bad = int(np.flatnonzero(~ok)[0])
    with pytest.raises(ValueError, match="NaN code"):
        fpsa.decode(bad, F)
    with pytest.raises(ValueError, match="NaN"):
        fpsa.encode(np.array([1.0, np.nan]), F)
    if fmt == "e4m3":
        with pytest.raises(ValueError, match="infinity"):
            fpsa.encode(np.inf, F)
    else:
        assert fpsa.encode(-np.inf, F) == 0xFC
    assert isinstance(fpsa.encode(1.0, F), int) and isinstance(fpsa.decode(0x38, F), float)
    ct = fpsa.code_table(F)
    assert np.array_equal(np.isnan(ct), np.isnan(table)) and np.array_equal(ct[ok], table[ok])
    assert np.array_equal(fpsa.is_nan_code(np.arange(256), F), ~ok)


def test_quantize_dequantize_and_dequantize_tensor(fpsa):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 48)) * np.exp2(rng.uniform(-6, 6, (64, 1)))
    scale = np.abs(x).max(axis=1, keepdims=True) / 448.0
    got = fpsa.quantize_dequantize(x, scale, fpsa.E4M3)
    ref = O.decode(O.encode(x / scale), O.E4M3).astype(np.float64) * scale
    assert got.dtype == np.float64 and np.array_equal(got, ref)
    with pytest.raises(ValueError, match="strictly positive"):
        fpsa.quantize_dequantize(x, 0.0, fpsa.E4M3)
    # QuantizedTensor.dequantize / dequantize_tensor: decode(code) * element scale in f64
    tmap = fpsa.build_tile_map(fpsa.GridShape(2, 4, 8, 48), fpsa.TileScheme(1, 4, 8))
    qt = fpsa.quantize_qk_tilewise(x, tmap, fpsa.E4M3)
    deq = fpsa.dequantize_tensor(qt)
    c, s = O.quantize_qk_tilewise(x, 32)
    assert np.array_equal(deq, O.decode(c).astype(np.float64) * np.repeat(s, 32)[:, None])
    qv = fpsa.quantize_v_channelwise(x, fpsa.E5M2)
    c, s = O.quantize_v_channelwise(x, O.E5M2)
    assert np.array_equal(qv.dequantize(), O.decode(c, O.E5M2).astype(np.float64) * s[None, :])


@pytest.mark.parametrize("d", [3, 16, 48, 64, 100])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_standalone_quantisers_any_width_and_f64(fpsa, d, dtype):
    """quantize_qk_tilewise / quantize_v_channelwise quantise float64 input in float64 (no narrowing to f32,
    quantize.py:115, :128) and accept any d; codes and scales equal the oracle's (pinned to the reference)."""
    rng = np.random.default_rng(d)
    x = rng.standard_normal((4 * 24, d)) * 3.0  # f64 values, most not f32-representable
    if dtype == "f32":
        x = x.astype(np.float32)
    tmap = fpsa.build_tile_map(fpsa.GridShape(4, 4, 6, d), fpsa.TileScheme(2, 2, 6))
    qt = fpsa.quantize_qk_tilewise(x, tmap, fpsa.E4M3)
    c, s = O.quantize_qk_tilewise(x, 24)
    assert np.array_equal(qt.scales, s) and np.array_equal(qt.codes, c)
    qv = fpsa.quantize_v_channelwise(x, fpsa.E4M3)
    c, s = O.quantize_v_channelwise(x)
    assert np.array_equal(qv.scales, s) and np.array_equal(qv.codes, c)
    if dtype == "f64":
        # narrowing to f32 first would change some codes: the f64 path is really taken
        c32, _ = O.quantize_v_channelwise(x.astype(np.float32))
        assert not np.array_equal(c32, qv.codes) or not np.array_equal(
            O.quantize_v_channelwise(x.astype(np.float32))[1], qv.scales)


@pytest.mark.parametrize("d", [8, 16, 96])
def test_fp8_sparse_forward_any_head_dim(fpsa, d):
    """Head dims the tcgen05 operands do not take directly (the reference's own test configs use d = 16 and
    8, conftest.py:26, test_attention.py:140-157) run zero-padded to 64 / 128: normalised-P parity."""
    grid, tile, win = (6, 8, 8), (3, 4, 4), (3, 3, 3)
    L = 6 * 8 * 8
    tv = 48
    q, k, v = O.gen_inputs(2, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                  fpsa.ForwardConfig(window=fpsa.WindowSpec(*win)))
    assert out.shape == (L, d) and out.dtype == np.float32
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, _ = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    budget, n_amb = O.p_flip_budget(q, k, v, tv, offs, ids, np.arange(L))
    err = np.abs(out.astype(np.float64) - ref)
    peak = float(np.abs(ref).max())
    print(f"d={d}: max rel err {err.max() / peak:.3e}, ambiguous weights {n_amb}")
    assert (err <= 1e-5 * peak + budget).all()
    pt = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                 fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), passthrough=True))
    assert O.cosine(pt, O.sparse_forward_f32(q, k, v, tv, offs, ids)) >= 0.9999


def test_natural_order_large_tiles(fpsa):
    """Tiles of 3072 and 24576 tokens (default_schedule's late and early regimes, schedule.py:58-64) in
    natural token order: bit-exact codes and normalised-P attention against the oracle."""
    for grid, tile, win in (((24, 32, 64), (12, 16, 16), (3, 3, 3)), ((24, 32, 64), (24, 32, 32), (1, 1, 1))):
        H, d = 1, 64
        L = grid[0] * grid[1] * grid[2]
        tv = tile[0] * tile[1] * tile[2]
        q, k, v = O.gen_inputs(9, 1, 0, L, d)
        perm = O.tile_perm(grid, tile)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(L)
        nat = [torch.from_numpy(x[inv]).cuda().view(L, 1, d) for x in (q, k, v)]  # natural (t,h,w) order
        plan = fpsa.FpsaPlan(grid, tile, win, H, d, p_mode="normalized")
        out = torch.empty((L, 1, d), dtype=torch.float32, device="cuda")
        plan.quantize(*nat, "lhd")
        plan.attention(out, "lhd")
        torch.cuda.synchronize()
        c, s = O.quantize_qk_tilewise(q, tv)
        M = L // tv
        assert np.array_equal(plan.q_scales.cpu().numpy(), s)
        assert np.array_equal(plan.q_codes.view(M, plan.pitch, d)[:, :tv].reshape(L, d).cpu().numpy(), c)
        offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
        got = out[:, 0].cpu().numpy()[perm]
        rows = np.unique(np.linspace(0, L - 1, 256).astype(np.int64))
        ref = O.fp8_sparse_rows(q, k, v, tv, offs, ids, rows).astype(np.float64)  # the oracle on the sampled rows
        budget, n_amb = O.p_flip_budget(q, k, v, tv, offs, ids, rows)
        err = np.abs(got[rows].astype(np.float64) - ref)
        peak = float(np.abs(ref).max())
        print(f"tile {tile}: max rel err {err.max() / peak:.3e}, ambiguous {n_amb}")
        assert (err <= 1e-5 * peak + budget).all()
