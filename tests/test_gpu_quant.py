"""GPU parity of the FP8 quantisers (K1 per-tile Q/K, K2 per-channel V): bit-exact vs the oracle.

The oracle (oracle/fpsa_oracle.py) is itself pinned bit-exactly to the
reference fp8sta by tests/test_oracle_golden.py.
"""

import numpy as np
import pytest

import oracle as O
from conftest import CASE_NAMES, golden_cases

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fpsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_04648_b200 as m

    return m


def _case_inputs(c):
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    return O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_quantize_matches_golden_reference(fpsa, attn_golden, name):
    """Codes and f64 scales equal the reference's (tests/golden from fp8sta itself)."""
    c = golden_cases(attn_golden)[name]
    q, k, v = _case_inputs(c)
    fmt = fpsa.FORMATS[c["fmt"]]
    tmap = fpsa.build_tile_map(fpsa.GridShape(*c["grid"], c["d"]), fpsa.TileScheme(*c["tile"]))
    rows = attn_golden[name + "__rows"]
    L = tmap.grid.tokens
    for nm, x in (("q", q), ("k", k)):
        qt = fpsa.quantize_qk_tilewise(x, tmap, fmt)
        assert np.array_equal(qt.scales, attn_golden[f"{name}__{nm}_scales"])
        got = qt.codes if L <= 256 else qt.codes[rows]
        assert np.array_equal(got, attn_golden[f"{name}__{nm}_codes_rows"])
    qv = fpsa.quantize_v_channelwise(v, fmt)
    assert np.array_equal(qv.scales, attn_golden[f"{name}__v_scales"])
    got = qv.codes if L <= 256 else qv.codes[rows]
    assert np.array_equal(got, attn_golden[f"{name}__v_codes_rows"])


def test_adversarial_near_tie_tiles(fpsa, codec_golden):
    """Quotients on and one f32 ulp beside every E4M3 midpoint, peaks over 2^+-20."""
    x = codec_golden["adv_x"]
    rows = int(codec_golden["adv_tile_rows"])
    tmap = fpsa.build_tile_map(fpsa.GridShape(x.shape[0] // rows, 1, rows, x.shape[1]), fpsa.TileScheme(1, 1, rows))
    qt = fpsa.quantize_qk_tilewise(x, tmap, fpsa.E4M3)
    assert np.array_equal(qt.scales, codec_golden["adv_scales"])
    assert np.array_equal(qt.codes, codec_golden["adv_codes"])


@pytest.mark.parametrize("fmt_name", ["e4m3", "e5m2"])
def test_random_scales_bit_exact(fpsa, fmt_name):
    rng = np.random.default_rng(5)
    L, d = 64 * 40, 128
    x = (rng.standard_normal((L, d)) * np.exp2(rng.uniform(-30, 30, (L // 64, 1))).repeat(64, 0)).astype(np.float32)
    fmt = fpsa.FORMATS[fmt_name]
    tmap = fpsa.build_tile_map(fpsa.GridShape(40, 8, 8, d), fpsa.TileScheme(1, 8, 8))
    qt = fpsa.quantize_qk_tilewise(x, tmap, fmt)
    codes, scales = O.quantize_qk_tilewise(x, 64, O.FORMATS[fmt_name])
    assert np.array_equal(qt.scales, scales)
    assert np.array_equal(qt.codes, codes)
    qv = fpsa.quantize_v_channelwise(x, fmt)
    vc, vs = O.quantize_v_channelwise(x, O.FORMATS[fmt_name])
    assert np.array_equal(qv.scales, vs)
    assert np.array_equal(qv.codes, vc)


def test_zero_tile_and_signed_zero(fpsa):
    """All-zero tile -> scale exactly 1.0; -0 and negative underflow -> 0x80 (quantize.py:107-108, fp8.py:185)."""
    d = 64
    x = np.zeros((32 * 3, d), dtype=np.float32)
    x[32:64] = -0.0
    x[64:96, 0] = 448.0
    x[64:96, 1] = -1e-6
    tmap = fpsa.build_tile_map(fpsa.GridShape(3, 4, 8, d), fpsa.TileScheme(1, 4, 8))
    qt = fpsa.quantize_qk_tilewise(x, tmap, fpsa.E4M3)
    assert qt.scales[0] == 1.0 and qt.scales[1] == 1.0 and qt.scales[2] == 1.0
    assert (qt.codes[:32] == 0x00).all()
    assert (qt.codes[32:64] == 0x80).all()
    assert (qt.codes[64:96, 0] == 0x7E).all() and (qt.codes[64:96, 1] == 0x80).all()


def test_nonfinite_raises(fpsa):
    x = np.ones((64, 64), dtype=np.float32)
    x[3, 5] = np.inf
    tmap = fpsa.build_tile_map(fpsa.GridShape(1, 8, 8, 64), fpsa.TileScheme(1, 8, 8))
    with pytest.raises(ValueError, match="non-finite"):
        fpsa.quantize_qk_tilewise(torch.from_numpy(x), tmap, fpsa.E4M3)
    x[3, 5] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        fpsa.quantize_v_channelwise(torch.from_numpy(x), fpsa.E4M3)


@pytest.mark.parametrize("shape", [
    ((21, 30, 52), (3, 10, 4), 3),   # Wan2.1-1.3B 480p, 3 heads
    ((21, 45, 80), (3, 5, 16), 2),   # Wan2.1-14B 720p, 2 heads
])
def test_natural_order_multihead_bf16(fpsa, shape):
    """Fast path: bf16 [L, H, d] in (t,h,w) order, gathered to padded tile-major codes in one pass."""
    grid, tile, H = shape
    d = 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((L, H, d), generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    plan = fpsa.FpsaPlan(grid, tile, (3, 3, 3), H, d)
    plan.quantize(x, x, x, "lhd")
    torch.cuda.synchronize()
    perm = O.tile_perm(grid, tile)
    tv, M = plan.tv, plan.M
    codes = plan.q_codes.view(H, M, plan.pitch, d).cpu().numpy()
    vcodes = plan.v_codes.view(H, M, plan.pitch, d).cpu().numpy()
    xs = x.float().cpu().numpy()
    for h in range(H):
        xt = xs[perm, h, :]
        c, s = O.quantize_qk_tilewise(xt, tv)
        assert np.array_equal(plan.q_scales.view(H, M)[h].cpu().numpy(), s)
        assert np.array_equal(codes[h, :, :tv, :].reshape(L, d), c)
        assert (codes[h, :, tv:, :] == 0).all()
        vc, vs = O.quantize_v_channelwise(xt)
        assert np.array_equal(plan.v_scales.view(H, d)[h].cpu().numpy(), vs)
        assert np.array_equal(vcodes[h, :, :tv, :].reshape(L, d), vc)


@pytest.mark.parametrize("fmt_name", ["e4m3", "e5m2"])
@pytest.mark.parametrize("peak_mant", [0x88, 0x8C, 0xE0])
def test_bf16_tie_table_every_class(fpsa, fmt_name, peak_mant):
    """The tie table of the TMA quantiser (exact ties of bf16 data resolved without f64 arithmetic) against
    the oracle, bit for bit, with tiles whose values are multiples of the peak / 2^k and the peak's
    significand 0x88 (136: not a multiple of 7, so only the classes with 7 | o tie), 0x8C (140 = 7 * 20) or
    0xE0 (224 = 7 * 32: every class can tie), in both formats."""
    fmt = fpsa.E4M3 if fmt_name == "e4m3" else fpsa.E5M2
    grid, tile, H, d = (6, 10, 32), (3, 5, 16), 2, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(3)
    peak = float(np.frombuffer(np.array([peak_mant << 16 | (130 << 23)], dtype=np.uint32).tobytes(), np.float32)[0])
    k = torch.randint(-255, 256, (L, H, d), generator=gen, device="cuda").float() * (peak / 256.0)
    k[0::240, :, 0] = peak
    x = k.to(torch.bfloat16)
    plan = fpsa.FpsaPlan(grid, tile, (3, 3, 3), H, d, fmt)
    plan.quantize(x, x, x, "lhd")
    torch.cuda.synchronize()
    perm = O.tile_perm(grid, tile)
    tv, M = plan.tv, plan.M
    qc = plan.q_codes.view(H, M, plan.pitch, d).cpu().numpy()
    vc = plan.v_codes.view(H, M, plan.pitch, d).cpu().numpy()
    xs = x.float().cpu().numpy()
    ofmt = O.FORMATS[fmt_name]
    for h in range(H):
        xt = xs[perm, h, :]
        c, s = O.quantize_qk_tilewise(xt, tv, ofmt)
        assert np.array_equal(plan.q_scales.view(H, M)[h].cpu().numpy(), s)
        assert np.array_equal(qc[h, :, :tv, :].reshape(L, d), c)
        c, s = O.quantize_v_channelwise(xt, ofmt)
        assert np.array_equal(plan.v_scales.view(H, d)[h].cpu().numpy(), s)
        assert np.array_equal(vc[h, :, :tv, :].reshape(L, d), c)


@pytest.mark.parametrize("tie_rich", [False, True])
def test_bf16_exact_ties_natural_order(fpsa, tie_rich):
    """bf16 data hits exact fp8 midpoints often (e.g. 448*0.796875/4.25 == 84); ties go to even.

    tie_rich draws every value from k/64 with a 4.25 peak per tile, so most
    quotients are exact midpoints -- exercises the queued exact path and its
    overflow fallback in the TMA quantiser.
    """
    grid, tile, H, d = (6, 10, 32), (3, 5, 16), 2, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(7)
    if tie_rich:
        k = torch.randint(-255, 256, (L, H, d), generator=gen, device="cuda").float() / 64.0
        k[0::240, :, 0] = 4.25
        x = k.to(torch.bfloat16)
    else:
        x = torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16)
    plan = fpsa.FpsaPlan(grid, tile, (3, 3, 3), H, d)
    plan.quantize(x, x, x, "lhd")
    torch.cuda.synchronize()
    perm = O.tile_perm(grid, tile)
    tv, M = plan.tv, plan.M
    qc = plan.q_codes.view(H, M, plan.pitch, d).cpu().numpy()
    vc = plan.v_codes.view(H, M, plan.pitch, d).cpu().numpy()
    xs = x.float().cpu().numpy()
    for h in range(H):
        xt = xs[perm, h, :]
        c, s = O.quantize_qk_tilewise(xt, tv)
        assert np.array_equal(plan.q_scales.view(H, M)[h].cpu().numpy(), s)
        assert np.array_equal(qc[h, :, :tv, :].reshape(L, d), c)
        c, s = O.quantize_v_channelwise(xt)
        assert np.array_equal(plan.v_scales.view(H, d)[h].cpu().numpy(), s)
        assert np.array_equal(vc[h, :, :tv, :].reshape(L, d), c)


def _check_plan_codes(plan, xs, perm):
    """Every head's q, k, v codes and scales in `plan` against the oracle (bit-exact)."""
    H, M, tv, d, L = plan.heads, plan.M, plan.tv, plan.d, plan.L
    bufs = [(plan.q_codes, plan.q_scales, False), (plan.k_codes, plan.k_scales, False),
            (plan.v_codes, plan.v_scales, True)]
    for x, (codes, scales, chan) in zip(xs, bufs):
        cc = codes.view(H, M, plan.pitch, d).cpu().numpy()
        sc = scales.cpu().numpy()
        xf = x.float().cpu().numpy()
        for h in range(H):
            xt = xf[perm, h, :]
            c, s = O.quantize_v_channelwise(xt) if chan else O.quantize_qk_tilewise(xt, tv)
            assert np.array_equal(sc.reshape(H, -1)[h], s)
            assert np.array_equal(cc[h, :, :tv, :].reshape(L, d), c)
            assert (cc[h, :, tv:, :] == 0).all()


def test_fused_quantiser_distinct_qkv_many_heads(fpsa):
    """The fused one-launch quantiser (v channel-amax tiles -> q, k tiles -> v code tiles waiting on the
    head's maxima) with distinct q, k, v over 6 heads of the C2 grid: all codes / scales bit-exact."""
    grid, tile, H, d = (21, 45, 80), (3, 5, 16), 6, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(11)
    xs = [(torch.randn((L, H, d), generator=gen, device="cuda") * s).to(torch.bfloat16) for s in (1.0, 3.0, 0.5)]
    plan = fpsa.FpsaPlan(grid, tile, (3, 3, 3), H, d)
    for _ in range(2):  # the second call reuses the workspace (counters re-zeroed by the call)
        plan.quantize(*xs, "lhd")
    torch.cuda.synchronize()
    plan.check_finite()
    _check_plan_codes(plan, xs, O.tile_perm(grid, tile))


@pytest.mark.parametrize("given", ["qkv", "v", "qk"])
def test_quantize_with_amax_hook(fpsa, given):
    """f3 fusion hook: caller-supplied tile / channel maxima give the same codes and scales as the
    self-reducing quantiser (and those are the reference's)."""
    grid, tile, H, d = (6, 10, 32), (3, 5, 16), 3, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(5)
    xs = [torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3)]
    plan = fpsa.FpsaPlan(grid, tile, (3, 3, 3), H, d)
    perm = torch.from_numpy(O.tile_perm(grid, tile)).cuda()
    tv, M = plan.tv, plan.M

    def tile_amax(x):  # [L, H, d] natural order -> [H, M] f32 max|x| per tile
        return x.float()[perm].abs().view(M, tv, H, d).amax(dim=(1, 3)).t().contiguous()

    qa = tile_amax(xs[0]) if "q" in given else None
    ka = tile_amax(xs[1]) if "k" in given else None
    va = xs[2].float().abs().amax(dim=0).contiguous() if "v" in given else None
    plan.quantize_with_amax(*xs, qa, ka, va, layout="lhd")
    torch.cuda.synchronize()
    _check_plan_codes(plan, xs, O.tile_perm(grid, tile))
