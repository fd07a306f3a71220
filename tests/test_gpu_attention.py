"""GPU parity of the sparse FP8 attention forward (K4) against the reference and the oracle.

Two softmax-weight modes:

* normalised-P (``p_mode="normalized"``, the drop-in default): the reference's
  arithmetic step for step (exact row max, f64 row sum, P = e4m3(448 p),
  fp8sta/attention.py:133-145).  Contract: |out - ref| <= 1e-5 * max|ref| per
  element, plus, only where a weight 448 p lies within 2^-19 (relative) of an
  e4m3 rounding midpoint, the output move of that one code flip
  (oracle.p_flip_budget: numpy's f32 exp is itself off by up to 2 ulp, so such
  a code is not determined by the algorithm).  Rows without such a weight must
  meet 1e-5 * max|ref| outright.
* one-pass (``p_mode="onepass"``, the fast path of the batched API and of
  bench.py): unnormalised weights re-quantised per key block, so outputs agree
  within a stated tolerance, not bitwise:
      cosine >= 0.999   and   max|out - ref| <= 0.1 * max|ref|
  and, for sigma=1 Gaussian inputs at the BASELINE video shapes,
  max-abs <= 2e-2.  Against the oracle's emulation of the kernel's own
  schedule (oracle.onepass_forward, same block order / lazy max / rounding
  points) the agreement is much tighter: cosine >= 0.99999.
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
REL_NORM = 1e-5  # normalised-P mode: max|out - ref| / max|ref| outside code flips


@pytest.fixture(scope="module")
def fpsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_04648_b200 as m

    return m


def _run_case(fpsa, c, tau=8.0, p_mode="onepass"):
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    tmap = fpsa.build_tile_map(fpsa.GridShape(*c["grid"], c["d"]), fpsa.TileScheme(*c["tile"]))
    cfg = fpsa.ForwardConfig(window=fpsa.WindowSpec(*c["window"]), fmt=fpsa.FORMATS[c["fmt"]], tau=tau,
                             p_mode=p_mode)
    return (q, k, v), fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), cfg)


def _check_normalized(got, ref, q, k, v, tv, offs, ids, rows, fmt, label):
    """The normalised-P contract (module docstring) on `rows`; returns (max rel err outside flips, flips)."""
    budget, n_amb = O.p_flip_budget(q, k, v, tv, offs, ids, rows, fmt)
    tol = REL_NORM * float(np.abs(ref).max())
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    clean = budget.max(axis=1) == 0.0
    worst_clean = float(err[clean].max()) / float(np.abs(ref).max()) if clean.any() else 0.0
    over = err > tol
    print(f"{label}: max rel err {err.max() / np.abs(ref).max():.3e} (rows without ambiguous weights "
          f"{worst_clean:.3e}); ambiguous weights {n_amb}, elements above 1e-5 rel {int(over.sum())}, all "
          f"within their flip budget: {bool((err <= tol + budget).all())}")
    assert np.isfinite(got).all()
    assert worst_clean <= REL_NORM, worst_clean
    assert (err <= tol + budget).all(), float((err - tol - budget).max())
    return worst_clean, n_amb


@pytest.mark.parametrize("name", CASE_NAMES)
def test_normalized_vs_reference_golden(fpsa, attn_golden, name):
    """Normalised-P mode against the reference's own outputs (tests/golden, fp8sta.fp8_sparse_forward)."""
    c = golden_cases(attn_golden)[name]
    (q, k, v), out = _run_case(fpsa, c, p_mode="normalized")
    rows = attn_golden[name + "__rows"]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    _check_normalized(out[rows], attn_golden[name + "__out"], q, k, v, tv, offs, ids, rows,
                      O.FORMATS[c["fmt"]], name)


@pytest.mark.parametrize("name", CASE_NAMES)
def test_attention_vs_reference_golden(fpsa, attn_golden, name):
    """One-pass mode against the reference's outputs (tolerance contract, module docstring)."""
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
    cfg = fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), p_mode="onepass")
    for h in range(H):
        qt = q[:, h, :].float()[perm].contiguous()
        kt = k[:, h, :].float()[perm].contiguous()
        vt = v[:, h, :].float()[perm].contiguous()
        ref_h = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(qt, kt, vt, tmap), cfg)
        got_h = out[:, h, :][perm]
        assert torch.equal(got_h, ref_h), (h, (got_h - ref_h).abs().max().item())


_ORACLE_CACHE: dict = {}


def _oracle_full(grid, tile, win, seed, fmt=O.E4M3, d=128):
    """(inputs, oracle output, tv, offs, ids) of one head, cached across the tests of this module."""
    key = (grid, tile, win, seed, fmt.name, d)
    if key not in _ORACLE_CACHE:
        L = grid[0] * grid[1] * grid[2]
        tv = tile[0] * tile[1] * tile[2]
        q, k, v = O.gen_inputs(seed, 1, 0, L, d)
        offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
        ref, _ = O.fp8_sparse_forward(q, k, v, tv, offs, ids, fmt)
        _ORACLE_CACHE[key] = ((q, k, v), ref, tv, offs, ids)
    return _ORACLE_CACHE[key]


def _sample_rows(L, n=384):
    """First rows, last rows and an even spread (both query blocks of many tiles)."""
    return np.unique(np.concatenate([np.arange(64), np.linspace(0, L - 1, n).astype(np.int64),
                                     np.arange(L - 64, L)]))


FULL_SHAPES = [
    ((21, 30, 52), (3, 10, 4), (3, 3, 5)),   # C1 Wan2.1-1.3B 480p
    ((21, 45, 80), (3, 5, 16), (3, 3, 3)),   # C2 Wan2.1-14B 720p, late-regime window
    ((21, 45, 80), (3, 5, 16), (5, 5, 3)),   # C2 at the benchmarked window
    ((33, 45, 80), (3, 5, 16), (5, 5, 3)),   # C3 HunyuanVideo 720p
]


@pytest.mark.parametrize("p_mode", ["onepass", "normalized"])
@pytest.mark.parametrize("shape", FULL_SHAPES)
def test_full_size_head_vs_oracle(fpsa, shape, p_mode):
    """One head at the BASELINE video shapes vs the reference algorithm (oracle), sigma=1 Gaussian."""
    grid, tile, win = shape
    d = 128
    (q, k, v), ref, tv, offs, ids = _oracle_full(grid, tile, win, 3)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                  fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), p_mode=p_mode))
    cos = O.cosine(out, ref)
    mabs = O.max_abs(out, ref)
    print(f"{grid} {win} {p_mode}: cos={cos:.7f} max-abs={mabs:.3e} rel={mabs / np.abs(ref).max():.3e}")
    assert cos >= COS_REF
    assert mabs <= 2e-2
    if p_mode == "normalized":
        rows = _sample_rows(q.shape[0])
        _check_normalized(out[rows], ref[rows], q, k, v, tv, offs, ids, rows, O.E4M3, f"{grid} {win}")


def test_bench_config_40_heads_bf16(fpsa):
    """The exact path bench.py times: C2 at window (5,5,3), 40 heads, bf16 [L, H, d] natural-order input,
    bf16 output written in natural order by the one-pass kernel (fpsa_attn_kernel<128, E4M3, BF16>).
    Heads 0 and 39 against the oracle on the same (bf16 -> f32, exact) inputs gathered to tile order."""
    grid, tile, win, H, d = (21, 45, 80), (3, 5, 16), (5, 5, 3), 40, 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    gen = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
    plan = fpsa.FpsaPlan(grid, tile, win, H, d)
    out = torch.empty_like(q)
    plan.quantize(q, k, v, "lhd")
    plan.attention(out, "lhd")
    torch.cuda.synchronize()
    perm = O.tile_perm(grid, tile)
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    for h in (0, H - 1):
        qh, kh, vh = (x[:, h, :].float().cpu().numpy()[perm] for x in (q, k, v))
        ref, codes = O.fp8_sparse_forward(qh, kh, vh, tv, offs, ids)
        # the plan's codes / scales of this head are the reference's, bit for bit
        M = L // tv
        qc = plan.q_codes.view(H, M, plan.pitch, d)[h, :, :tv].reshape(L, d).cpu().numpy()
        assert np.array_equal(qc, codes["q_codes"])
        assert np.array_equal(plan.q_scales.view(H, M)[h].cpu().numpy(), codes["q_scales"])
        assert np.array_equal(plan.v_scales.view(H, d)[h].cpu().numpy(), codes["v_scales"])
        got = out[:, h, :].float().cpu().numpy()[perm]
        cos, mabs = O.cosine(got, ref), O.max_abs(got, ref)
        print(f"head {h}: cos={cos:.6f} max-abs={mabs:.3e} rel={mabs / np.abs(ref).max():.3e}")
        assert cos >= COS_REF
        assert mabs <= 2e-2


def test_redo_path_full_size(fpsa):
    """The exact-max redo launch at C2 (5,5,3): tau = 0 sends every item whose later key blocks exceed the
    first block's max to the second launch; the result still meets the one-pass contract vs the oracle."""
    grid, tile, win, d = (21, 45, 80), (3, 5, 16), (5, 5, 3), 128
    (q, k, v), ref, tv, offs, ids = _oracle_full(grid, tile, win, 3)
    plan = fpsa.FpsaPlan(grid, tile, win, 1, d, tau=0.0)
    out = torch.empty((q.shape[0], d), dtype=torch.float32, device="cuda")
    plan.quantize(*(torch.from_numpy(x).cuda() for x in (q, k, v)), layout="ld", tile_order=True)
    plan.attention(out, layout="ld", tile_order=True)
    n_redo = plan.redo_count()
    got = out.cpu().numpy()
    cos, mabs = O.cosine(got, ref), O.max_abs(got, ref)
    print(f"redo items {n_redo} of {plan.n_items}: cos={cos:.6f} max-abs={mabs:.3e}")
    assert n_redo > plan.n_items // 4
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
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    for p_mode in ("onepass", "normalized"):
        out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                      fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), p_mode=p_mode))
        cos = O.cosine(out, ref)
        mabs = O.max_abs(out, ref)
        print(f"tile {tile} {p_mode}: cos={cos:.7f} max-abs={mabs:.3e}")
        assert cos >= COS_REF
        assert mabs <= 2e-2
    rows = _sample_rows(L, 256)
    _check_normalized(out[rows], ref[rows], q, k, v, tv, offs, ids, rows, O.E4M3, f"tile {tile}")


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
    out = fpsa.fp8_sparse_forward(inputs, fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), p_mode="onepass"))
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
    # normalised-P mode (the default): per-column masking of the tail block in max, sum and P
    nout = fpsa.fp8_sparse_forward(inputs, fpsa.ForwardConfig(window=fpsa.WindowSpec(*win)))
    rows = _sample_rows(L, 256)
    _check_normalized(nout[rows], ref[rows], q, k, v, tv, offs, ids, rows, O.E4M3, f"tv={tv}")


def test_full_size_head_e5m2(fpsa):
    """E5M2 Q/K/V (P stays E4M3, attention.py:208) at the C2 shape, window (3,3,3), against the oracle."""
    grid, tile, win, d = (21, 45, 80), (3, 5, 16), (3, 3, 3), 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(4, 1, 0, L, d)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap),
                                  fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), fmt=fpsa.E5M2,
                                                     p_mode="onepass"))
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


@pytest.mark.parametrize("grid,tile,win,d", [
    ((4, 6, 9), (1, 3, 3), (3, 3, 3), 64),     # tv = 9: cheap max / sum passes, many steps per item
    ((6, 8, 8), (3, 4, 4), (3, 3, 3), 128),    # tv = 48
])
@pytest.mark.parametrize("p_mode", ["normalized", "onepass"])
def test_split_issue_repeated_launches(fpsa, grid, tile, win, d, p_mode):
    """The split QK / PV issue under repetition: 300 launches of the multi-pass modes (normalised P: three
    passes; one-pass with tau = 0: saturating items go to the exact-max redo launch, two passes) on small
    tiles.  Their max / sum passes store no P~, so without the p_free wait before each p_ready signal one
    softmax part could signal two phases of its p_ready barrier while the PV warp waits for the other
    part, a deadlock the first split build hit twice in full GPU-suite runs (K4).
    The race is timing-dependent and this test did not reproduce it on demand (2 x 1200 launches of the
    unfixed build passed), so it guards the schedule's determinism: every repetition must reproduce the
    first output bit for bit."""
    L = grid[0] * grid[1] * grid[2]
    q, k, v = O.gen_inputs(5, 1, 0, L, d)
    plan = fpsa.FpsaPlan(grid, tile, win, 1, d, p_mode=p_mode, tau=0.0 if p_mode == "onepass" else 8.0)
    out = torch.empty((L, d), dtype=torch.float32, device="cuda")
    args = [torch.from_numpy(x).cuda() for x in (q, k, v)]
    plan.quantize(*args, layout="ld", tile_order=True)
    plan.attention(out, layout="ld", tile_order=True)
    first = out.clone()
    for _ in range(300):
        plan.attention(out, layout="ld", tile_order=True)
    torch.cuda.synchronize()
    assert torch.equal(out, first)
