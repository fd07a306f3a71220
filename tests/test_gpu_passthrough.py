"""GPU parity of the full-precision passthrough path (bf16 tcgen05 kind::f16 kernel).

The reference's passthrough / sparse_reference (fp8sta/attention.py:152-154,
:165-176, :192-194) is f32 attention over the window's key tiles.  The GPU
kernel computes it on bf16 operands with f32 softmax and accumulation, so:
  * against the oracle's emulation of the kernel (oracle.passthrough_emulation:
    same bf16 rounding, first-block max, bf16 P):  cosine >= 0.999999
  * against the reference's f32 output (golden):   cosine >= 0.9999,
    max|out - ref| <= 5e-2 max|ref| (the heavy-tailed case; 1e-2 otherwise)
Device fidelity sums (fpsa_fidelity) are checked against the host metrics.
"""

import math

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


def _case(c):
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    return L, tv, (q, k, v), offs, ids


@pytest.mark.parametrize("name", CASE_NAMES)
def test_passthrough_vs_reference_and_emulation(fpsa, attn_golden, name):
    c = golden_cases(attn_golden)[name]
    L, tv, (q, k, v), offs, ids = _case(c)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*c["grid"], c["d"]), fpsa.TileScheme(*c["tile"]))
    cfg = fpsa.ForwardConfig(window=fpsa.WindowSpec(*c["window"]), passthrough=True)
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), cfg)
    assert isinstance(out, np.ndarray) and out.dtype == np.float32 and np.isfinite(out).all()
    rows = attn_golden[name + "__rows"]
    sref = attn_golden[name + "__sparse_ref"]
    emu = O.passthrough_emulation(q, k, v, tv, offs, ids)
    cos_e, cos_r = O.cosine(out, emu), O.cosine(out[rows], sref)
    rel_r = O.max_abs(out[rows], sref) / float(np.abs(sref).max())
    print(f"{name}: cos(emu)={cos_e:.8f} max-abs(emu)={O.max_abs(out, emu):.2e} cos(ref)={cos_r:.7f} rel(ref)={rel_r:.2e}")
    assert cos_e >= 0.999999
    assert O.max_abs(out, emu) <= 2e-3 * float(np.abs(emu).max())
    assert cos_r >= 0.9999
    assert rel_r <= (5e-2 if c["dist"] == "heavy" else 1e-2)


def test_passthrough_multihead_natural_order_bf16(fpsa):
    """[L, H, d] bf16 natural order == per-head tile-order calls, unpermuted (bit-identical)."""
    grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 3, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(2)
    q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
    plan = fpsa.PassthroughPlan(grid, tile, win, H, d)
    out = plan(q, k, v, "lhd", out_dtype=torch.float32)
    tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
    perm = torch.from_numpy(fpsa.tile_contiguous_order(tmap)).cuda()
    one = fpsa.PassthroughPlan(grid, tile, win, 1, d)
    for h in range(H):
        ref = one(q[:, h][perm].contiguous(), k[:, h][perm].contiguous(), v[:, h][perm].contiguous(), "ld",
                  out_dtype=torch.float32, tile_order=True)
        got = out[:, h][perm]
        assert torch.equal(got, ref), (h, (got - ref).abs().max().item())
    # bf16 inputs are exact: the only deviation from f32 attention is the bf16 P
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    h = 1
    qt, kt, vt = (x[:, h][perm].float().cpu().numpy() for x in (q, k, v))
    ref32 = O.sparse_forward_f32(qt, kt, vt, tile[0] * tile[1] * tile[2], offs, ids)
    assert O.cosine(out[:, h][perm].cpu().numpy(), ref32) >= 0.999995


def test_passthrough_overflow_redo(fpsa):
    """Logits more than 127 (log2 units) above the first key block's row max overflow the one-pass
    sum; those items go through the exact-max launch and still match f32 attention."""
    grid, tile, win, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 128
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    rng = np.random.default_rng(5)
    q = O.bf16_round(rng.standard_normal((L, d)).astype(np.float32) * 12)
    k = O.bf16_round(rng.standard_normal((L, d)).astype(np.float32) * 12)
    v = O.bf16_round(rng.standard_normal((L, d)).astype(np.float32))
    plan = fpsa.PassthroughPlan(grid, tile, win, 1, d)
    out = torch.empty((L, d), dtype=torch.float32, device="cuda")
    plan.gather(*(torch.from_numpy(x).cuda() for x in (q, k, v)), layout="ld", tile_order=True)
    plan.attention(out, layout="ld", tile_order=True)
    n_redo = plan.redo_count()
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref = O.sparse_forward_f32(q, k, v, tv, offs, ids)
    got = out.cpu().numpy()
    print(f"redo items {n_redo} of {plan.n_items}; cos={O.cosine(got, ref):.7f} max-abs={O.max_abs(got, ref):.2e}")
    assert n_redo > 0
    assert np.isfinite(got).all()
    assert O.cosine(got, ref) >= 0.99999


def test_device_fidelity_matches_host_metrics(fpsa):
    L, H, d = 3000, 3, 64
    gen = torch.Generator(device="cuda").manual_seed(4)
    ref = torch.randn((L, H, d), generator=gen, device="cuda")
    app = (ref + 0.01 * torch.randn((L, H, d), generator=gen, device="cuda")).to(torch.bfloat16)
    app32 = app.float()
    got = fpsa.device_fidelity(ref, app32, "lhd")
    for h in range(H):
        x = ref[:, h].double().cpu().numpy().ravel()
        y = app32[:, h].double().cpu().numpy().ravel()
        cos, mse, snr = got[h]
        assert abs(cos - O.cosine(x, y)) < 1e-12
        assert abs(mse - float(((x - y) ** 2).mean())) <= 1e-12 * max(1.0, mse)
        assert abs(snr - 10 * math.log10((x @ x) / ((x - y) @ (x - y)))) < 1e-9
    # mixed dtypes and identical inputs
    same = fpsa.device_fidelity(app, app, "lhd")
    assert all(m[0] == pytest.approx(1.0, abs=1e-15) and m[1] == 0.0 and m[2] == math.inf for m in same)


def test_schedule_runner_fidelity_columns(fpsa):
    """ScheduleRunner(fidelity=True) fills the reference CSV's cosine / mse / snr columns."""
    from paper_2506_04648_b200.grid import TileScheme
    from paper_2506_04648_b200.schedule import RegimeParams, ScheduleConfig
    from paper_2506_04648_b200.sparsity import WindowSpec

    grid, H, d = (6, 10, 32), 2, 128
    sched = ScheduleConfig(alpha1=0.2, alpha2=0.7,
                           early=RegimeParams(TileScheme(6, 10, 16), WindowSpec(1, 1, 1)),
                           mid=RegimeParams(TileScheme(3, 5, 16), WindowSpec(3, 3, 3)),
                           late=RegimeParams(TileScheme(3, 10, 16), WindowSpec(1, 1, 2)),
                           total_steps=5)
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(6)
    q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = torch.empty((L, H, d), dtype=torch.float32, device="cuda")
    runner = fpsa.ScheduleRunner(grid, sched, H, d, use_graphs=False, fidelity=True)
    rows = runner.run(q, k, v, out)
    csv = fpsa.rows_to_csv(rows).splitlines()
    assert len(csv) == 6 and "nan" not in ",".join(csv[1:])
    for r in rows:
        assert 0.99 < r.cosine_sim <= 1.0 and r.mse > 0 and r.snr_db > 20, r
