"""GPU parity of the sparse FP8 attention forward (K4) against the reference and the oracle.

Tolerances: the one-pass kernel re-quantises the
unnormalised softmax weights per key block, the reference quantises the
normalised weights (fp8sta/attention.py:133-145), so outputs agree within a
stated tolerance, not bitwise:
    cosine >= 0.999   and   max|out - ref| <= 0.1 * max|ref|
and, for sigma=1 Gaussian inputs at the BASELINE video shapes, max-abs <= 2e-2.
Against the oracle's emulation of the kernel's own schedule
(oracle.onepass_forward, same block order / lazy max / rounding points) the
agreement is much tighter: cosine >= 0.99999.
"""

import numpy as np
import pytest

import oracle as O
from conftest import CASE_NAMES, golden_cases

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

COS_REF = 0.999
REL_REF = 0.1
COS_EMU = 0.99999
REL_EMU = 1e-2  # max|out - emulation| / max|emulation|


@pytest.fixture(scope="module")
def fpsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_04648_b200 as m

    return m


def _run_case(fpsa, c, tau=8.0):
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    tmap = fpsa.build_tile_map(fpsa.GridShape(*c["grid"], c["d"]), fpsa.TileScheme(*c["tile"]))
    cfg = fpsa.ForwardConfig(window=fpsa.WindowSpec(*c["window"]), fmt=fpsa.FORMATS[c["fmt"]], tau=tau)
    return (q, k, v), fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), cfg)


@pytest.mark.parametrize("name", CASE_NAMES)
def test_attention_vs_reference_golden(fpsa, attn_golden, name):
    c = golden_cases(attn_golden)[name]
    _, out = _run_case(fpsa, c)
    rows = attn_golden[name + "__rows"]
    ref = attn_golden[name + "__out"]
    got = out[rows]
    cos = O.cosine(got, ref)
    rel = O.max_abs(got, ref) / float(np.abs(ref).max())
    print(f"{name}: cos={cos:.6f} max-abs={O.max_abs(got, ref):.3e} rel={rel:.3e}")
    assert np.isfinite(out).all()
    assert cos >= COS_REF, cos
    assert rel <= REL_REF, rel


@pytest.mark.parametrize("name", CASE_NAMES)
def test_attention_vs_onepass_emulation(fpsa, attn_golden, name):
    c = golden_cases(attn_golden)[name]
    (q, k, v), out = _run_case(fpsa, c)
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    fmt = O.FORMATS[c["fmt"]]
    _, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids, fmt)
    emu = O.onepass_forward(codes, tv, offs, ids, fmt, tau=8.0, poly=True)
    cos = O.cosine(out, emu)
    # per-row least-squares scale: a normalisation error (e.g. padding keys in the row sum) is a row
    # scale, which the cosine barely sees
    scale = (out * emu).sum(1) / np.maximum((emu * emu).sum(1), 1e-30)
    rel = O.max_abs(out, emu) / float(np.abs(emu).max())
    print(f"{name}: cos(emu)={cos:.7f} max-abs/max={rel:.3e} row scale [{scale.min():.5f}, {scale.max():.5f}]")
    assert cos >= COS_EMU, cos
    assert rel <= REL_EMU, rel
    assert np.abs(scale - 1.0).max() <= 5e-3, (scale.min(), scale.max())
    assert abs(scale.mean() - 1.0) <= 1e-3, scale.mean()  # no systematic normalisation bias


def test_tile_order_vs_natural_order_multihead(fpsa):
    """[L,H,d] natural-order bf16 fast path == per-head reference-layout path, unpermuted."""
    grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 3, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = fpsa.fps_attention(q, k, v, grid, tile, win, layout="lhd", out_dtype=torch.float32)
    perm = fpsa.tile_contiguous_order(fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile)))
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    cfg = fpsa.ForwardConfig(window=fpsa.WindowSpec(*win))
    for h in range(H):
        qt = q[:, h, :].float()[perm].contiguous()
        kt = k[:, h, :].float()[perm].contiguous()
        vt = v[:, h, :].float()[perm].contiguous()
        ref_h = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(qt, kt, vt, tmap), cfg)
        got_h = out[:, h, :][perm]
        assert torch.equal(got_h, ref_h), (h, (got_h - ref_h).abs().max().item())


@pytest.mark.parametrize("shape", [
    ((21, 30, 52), (3, 10, 4), (3, 3, 5)),   # C1 Wan2.1-1.3B 480p
    ((21, 45, 80), (3, 5, 16), (3, 3, 3)),   # C2 Wan2.1-14B 720p
])
def test_full_size_head_vs_oracle(fpsa, shape):
    """One head at the BASELINE video shapes vs the reference algorithm (oracle), sigma=1 Gaussian."""
    grid, tile, win = shape
    d = 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(3, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), fpsa.ForwardConfig(window=fpsa.WindowSpec(*win)))
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, _ = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    cos = O.cosine(out, ref)
    mabs = O.max_abs(out, ref)
    print(f"{grid}: cos={cos:.6f} max-abs={mabs:.3e} rel={mabs / np.abs(ref).max():.3e}")
    assert cos >= COS_REF
    assert mabs <= 2e-2


def test_exact_redo_path_forced(fpsa, attn_golden):
    """tau = 0: every item whose later key blocks exceed the first block's max saturates e4m3 and is
    recomputed by the exact-max launch; the result follows the oracle's emulation of that schedule."""
    c = golden_cases(attn_golden)["tv240_d128"]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    plan = fpsa.FpsaPlan(c["grid"], c["tile"], c["window"], 1, c["d"], tau=0.0)
    out = torch.empty((L, c["d"]), dtype=torch.float32, device="cuda")
    args = [torch.from_numpy(x).cuda() for x in (q, k, v)]
    plan.quantize(*args, layout="ld", tile_order=True)
    plan.attention(out, layout="ld", tile_order=True)
    n_redo = plan.redo_count()
    got = out.cpu().numpy()
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    ref, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    emu, redo = O.onepass_forward(codes, tv, offs, ids, tau=0.0, poly=True, return_redo=True)
    print(f"redo items: kernel {n_redo}, emulation {len(redo)} of {plan.n_items}; "
          f"cos(emu)={O.cosine(got, emu):.7f} cos(ref)={O.cosine(got, ref):.6f}")
    assert n_redo == len(redo) > 0
    assert O.cosine(got, emu) >= COS_EMU
    assert O.cosine(got, ref) >= COS_REF


def test_full_size_head_large_tile(fpsa):
    """The C4 early regime at the 14B 720p grid: tile (7,15,16) (1680 tokens, 14 key blocks), window (3,3,1)."""
    grid, tile, win, d = (21, 45, 80), (7, 15, 16), (3, 3, 1), 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(5, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), fpsa.ForwardConfig(window=fpsa.WindowSpec(*win)))
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    cos = O.cosine(out, ref)
    mabs = O.max_abs(out, ref)
    print(f"tile {tile}: cos={cos:.6f} max-abs={mabs:.3e}")
    assert cos >= COS_REF
    assert mabs <= 2e-2


@pytest.mark.parametrize("grid,tile,win,d", [
    ((6, 10, 20), (3, 5, 5), (3, 3, 3), 128),   # tv = 75: a tail block with 75 keys (not a multiple of 4)
    ((4, 6, 9), (1, 3, 3), (3, 3, 3), 64),      # tv = 9
    ((6, 10, 26), (3, 5, 13), (3, 3, 1), 128),  # tv = 195: 128 + 67
])
def test_odd_tile_volumes(fpsa, grid, tile, win, d):
    """Tile volumes that are not multiples of 8 (the reference accepts any tile): per-column masking of
    the tail block in the max, the codes and the row sum."""
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(21, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    inputs = fpsa.AttentionInputs(q, k, v, tmap)
    out = fpsa.fp8_sparse_forward(inputs, fpsa.ForwardConfig(window=fpsa.WindowSpec(*win)))
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    emu = O.onepass_forward(codes, tv, offs, ids, tau=8.0, poly=True)
    scale = (out * emu).sum(1) / np.maximum((emu * emu).sum(1), 1e-30)
    print(f"tv={tv}: cos(ref)={O.cosine(out, ref):.6f} cos(emu)={O.cosine(out, emu):.7f} "
          f"row scale [{scale.min():.5f}, {scale.max():.5f}]")
    assert O.cosine(out, ref) >= COS_REF
    assert O.cosine(out, emu) >= COS_EMU
    # few keys per row here (window (3,3,1): 780), so single code flips from the exp approximations move
    # a peaked row by up to ~1.5 % (the emulation with exact exp2 differs from itself with the polynomial
    # as much); a normalisation bug is a systematic bias instead
    assert abs(scale.mean() - 1.0) <= 2e-3, scale.mean()
    assert np.abs(scale - 1.0).max() <= 3e-2
    pt = fpsa.fp8_sparse_forward(inputs, fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), passthrough=True))
    f32 = O.sparse_forward_f32(q, k, v, tv, offs, ids)
    assert O.cosine(pt, f32) >= 0.9999


def test_full_size_head_e5m2(fpsa):
    """E5M2 Q/K/V (P stays E4M3, attention.py:208) at the C2 shape, window (3,3,3), against the oracle."""
    grid, tile, win, d = (21, 45, 80), (3, 5, 16), (3, 3, 3), 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(4, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                  fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), fmt=fpsa.E5M2))
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, _ = O.fp8_sparse_forward(q, k, v, tv, offs, ids, O.E5M2)
    cos, mabs = O.cosine(out, ref), O.max_abs(out, ref)
    print(f"e5m2 {grid}: cos={cos:.6f} max-abs={mabs:.3e}")
    assert cos >= COS_REF
    assert mabs <= 2e-2


def test_full_size_head_passthrough(fpsa):
    """Passthrough at the C2 shape, window (3,3,3): bf16 operands against the oracle's f32 sparse attention."""
    grid, tile, win, d = (21, 45, 80), (3, 5, 16), (3, 3, 3), 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(5, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                  fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), passthrough=True))
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref = O.sparse_forward_f32(q, k, v, tv, offs, ids)
    cos, mabs = O.cosine(out, ref), O.max_abs(out, ref)
    print(f"passthrough {grid}: cos={cos:.7f} max-abs={mabs:.3e}")
    assert cos >= 0.9999
    assert mabs <= 1e-2 * float(np.abs(ref).max())
