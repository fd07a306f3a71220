"""GPU tests of the drivers above the hot path: the schedule runner (CUDA graphs
per regime) and the Ulysses sequence<->head path on a single-rank NCCL group."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fpsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_04648_b200 as m

    return m


def _small_schedule(fpsa, D=10):
    T, W, R = fpsa.TileScheme, fpsa.WindowSpec, fpsa.RegimeParams
    # grid 6x10x32: tiles (6,10,16) tv 960 > (3,10,8) tv 240 > (3,5,16) tv 240? -> use (3,10,16) tv 480
    return fpsa.ScheduleConfig(alpha1=0.2, alpha2=0.6, early=R(T(6, 10, 16), W(1, 1, 1)),
                               mid=R(T(3, 5, 16), W(3, 3, 3)), late=R(T(3, 10, 16), W(2, 1, 2)), total_steps=D)


def test_schedule_runner_graphs_match_eager(fpsa):
    grid, H, d = (6, 10, 32), 2, 128
    sc = _small_schedule(fpsa)
    assert fpsa.validate(sc) == []
    L = grid[0] * grid[1] * grid[2]
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn((L, H, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    eager = fpsa.ScheduleRunner(grid, sc, H, d, use_graphs=False)
    graph = fpsa.ScheduleRunner(grid, sc, H, d, use_graphs=True)
    for t in range(1, sc.total_steps + 1):
        a, b = torch.empty_like(q), torch.empty_like(q)
        ra = eager.step(t, q, k, v, a)
        rb = graph.step(t, q, k, v, b)
        assert ra == rb == sc.regime_of(t)
        ref = fpsa.fps_attention(q, k, v, grid, fpsa.params_at(t, sc).tile.dims, fpsa.params_at(t, sc).window,
                                 layout="lhd")
        assert torch.equal(a, ref) and torch.equal(b, ref)
    rows = graph.run(q, k, v, torch.empty_like(q))
    assert [r.regime for r in rows] == [sc.regime_of(t) for t in range(1, 11)]
    csv = fpsa.rows_to_csv(rows)
    assert csv.splitlines()[0].startswith("step,regime,tile_t,tile_h,tile_w,win_t,win_h,win_w,density")
    assert len(csv.splitlines()) == 11


def test_ulysses_single_rank_matches_plan(fpsa):
    import torch.distributed as dist

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 4, 128
    L = grid[0] * grid[1] * grid[2]
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, v = (torch.randn((L, H, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    uly = fpsa.UlyssesAttention(grid, tile, win, H, d, device="cuda")
    out = uly(q, k, v)
    ref = fpsa.fps_attention(q, k, v, grid, tile, win, layout="lhd")
    assert torch.equal(out, ref)
    # per-head-chunk pipeline: async NCCL all-to-alls around each chunk's kernels
    uly3 = fpsa.UlyssesAttention(grid, tile, win, H, d, device="cuda", chunk_heads=3)
    assert torch.equal(uly3(q, k, v), ref)
    dist.destroy_process_group()


def test_host_streamer_matches_plan(fpsa):
    """Pinned-host streamed path (head chunks, overlapped transfers) == the device plan, bitwise,
    with a chunk size that does not divide the head count."""
    grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 7, 128
    L = grid[0] * grid[1] * grid[2]
    gen = torch.Generator(device="cuda").manual_seed(9)
    q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
    ref = fpsa.FpsaPlan(grid, tile, win, H, d)(q, k, v, "lhd")
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    oh = torch.empty((L, H, d), dtype=torch.bfloat16).pin_memory()
    streamer = fpsa.HostStreamer(grid, tile, win, H, d, chunk_heads=3)
    for _ in range(2):  # the second call reuses the staging buffers
        oh.zero_()
        streamer(qh, kh, vh, oh)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(oh, ref.cpu())
    with pytest.raises(ValueError):
        streamer(q, k, v, oh)  # device tensors are rejected


def _oracle_head(fpsa, grid, tile, win, x_nat, h):
    """Oracle output of head h, natural-order [L, H, d] bf16 inputs -> natural order f32."""
    import oracle as O

    perm = O.tile_perm(grid, tile)
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = (x[:, h, :].float().cpu().numpy()[perm] for x in x_nat)
    offs, ids = O.window_lists(O.tile_grid_dims(grid, tile), win)
    ref, _ = O.fp8_sparse_forward(q, k, v, tv, offs, ids)
    out = np.empty_like(ref)
    out[perm] = ref
    return out


@pytest.mark.parametrize("which", ["c4", "default"])
def test_schedule_runner_regimes_vs_oracle(fpsa, which):
    """One step of every regime through ScheduleRunner (CUDA graphs) against the oracle of that step's
    (tile, window) (experiment.py:178-201, schedule.py:71-73): the BASELINE C4 schedule at the 14B 720p grid,
    and the reference's own default_schedule (schedule.py:58-64: 24576-, 384- and 3072-token tiles) on a grid
    its tiles divide."""
    import oracle as O

    if which == "c4":
        grid, d, sc = (21, 45, 80), 128, fpsa.c4_schedule(50)
    else:
        grid, d, sc = (24, 32, 32), 64, fpsa.default_schedule(50)
    H = 1
    L = grid[0] * grid[1] * grid[2]
    g = torch.Generator(device="cuda").manual_seed(4)
    x = [torch.randn((L, H, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3)]
    runner = fpsa.ScheduleRunner(grid, sc, H, d, use_graphs=True)
    seen = set()
    for t in range(1, sc.total_steps + 1):
        regime = sc.regime_of(t)
        if regime in seen:
            continue
        seen.add(regime)
        out = torch.empty_like(x[0])
        assert runner.step(t, *x, out) == regime
        torch.cuda.synchronize()
        rp = fpsa.params_at(t, sc)
        ref = _oracle_head(fpsa, grid, rp.tile.dims, rp.window.dims, x, 0)
        got = out[:, 0].float().cpu().numpy()
        cos, mabs = O.cosine(got, ref), O.max_abs(got, ref)
        print(f"{which} t={t} {regime} tile {rp.tile.dims} window {rp.window.dims}: cos={cos:.6f} max-abs={mabs:.3e}")
        assert cos >= 0.999 and mabs <= 2e-2
    assert seen == {"early", "mid", "late"}
