"""CPU tests of libfpsa's C ABI and the host-side mirror of the reference API.

No GPU needed: the library loads, exports every symbol include/fpsa.h
declares, and its host entry points (tile grid, permutation, window CSR,
regime, work list) are checked bit-exactly against the reference's golden
vectors and the oracle, including the reference's brute-force acceptance
sweep (test_acceptance.py:104-125: every tile grid <= 64 tiles x 343 windows).
Device entry points are only probed for argument validation (they must fail
with FPSA_EINVAL before touching CUDA).
"""

import ctypes
import itertools
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fpsa.h")


@pytest.fixture(scope="module")
def fpsa():
    from paper_2506_04648_b200 import _lib, build

    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    import paper_2506_04648_b200 as m

    return m


@pytest.fixture(scope="module")
def lib(fpsa):
    from paper_2506_04648_b200 import _lib

    return _lib.lib()


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fpsa_[a-z0-9_]+)\s*\(", text)))


def test_every_header_symbol_exported(lib):
    from paper_2506_04648_b200 import _lib

    syms = header_symbols()
    assert len(syms) >= 12
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), f"{s} declared in include/fpsa.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(syms)


def test_library_is_sm100a(fpsa):
    """The shipped .so carries sm_100a SASS (cuobjdump, when available)."""
    import shutil
    import subprocess

    from paper_2506_04648_b200 import _lib

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_errors(lib):
    assert lib.fpsa_version() >= 10000
    from paper_2506_04648_b200 import _lib

    out = _lib.Dims3()
    st = lib.fpsa_tile_grid(_lib.dims3((21, 30, 52)), _lib.dims3((3, 4, 4)), ctypes.byref(out))
    assert st == _lib.FPSA_EINDIVISIBLE
    assert lib.fpsa_last_error().decode() == \
        "indivisible grid: axis h has 30 tokens, not divisible by tile extent 4"


# ----------------------------------------------------------------- layout
@pytest.mark.parametrize("key", ["perm_4_8_8_2_4_4", "perm_6_8_8_3_4_4", "perm_6_10_16_3_10_4",
                                 "perm_7_9_16_7_9_8", "perm_4_6_10_2_3_5"])
def test_tile_perm_vs_reference(fpsa, codec_golden, key):
    v = [int(x) for x in key.split("_")[1:]]
    tmap = fpsa.build_tile_map(fpsa.GridShape(*v[:3], 8), fpsa.TileScheme(*v[3:]))
    perm = fpsa.tile_contiguous_order(tmap)
    assert np.array_equal(perm, codec_golden[key])
    inv = fpsa.invert_permutation(perm)
    assert np.array_equal(perm[inv], np.arange(perm.size))


def test_full_size_perm_vs_oracle(fpsa):
    for grid, tile in [((21, 30, 52), (3, 10, 4)), ((21, 45, 80), (3, 5, 16)), ((33, 45, 80), (3, 5, 16)),
                       ((21, 45, 80), (7, 15, 16)), ((21, 45, 80), (7, 9, 8))]:
        tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, 128), fpsa.TileScheme(*tile))
        assert np.array_equal(fpsa.tile_contiguous_order(tmap), O.tile_perm(grid, tile))


def test_grid_api_errors(fpsa):
    with pytest.raises(ValueError, match="GridShape.height must be >= 1"):
        fpsa.GridShape(1, 0, 1, 8)
    with pytest.raises(ValueError, match="TileScheme.tile_w must be >= 1"):
        fpsa.TileScheme(1, 1, 0)
    with pytest.raises(ValueError, match="indivisible grid: axis w has 52 tokens, not divisible by tile extent 5"):
        fpsa.build_tile_map(fpsa.GridShape(21, 30, 52, 128), fpsa.TileScheme(3, 10, 5))
    tmap = fpsa.build_tile_map(fpsa.GridShape(4, 8, 8, 64), fpsa.TileScheme(2, 4, 4))
    assert tmap.tile_grid_dims == (2, 2, 2) and tmap.tiles_total == 8 and tmap.tile_volume == 32
    assert fpsa.tile_of_token(tmap, 255) == (1, 1, 1)
    assert fpsa.flat_tile_index(tmap, (1, 0, 1)) == 5
    assert fpsa.token_rows_of_tile(tmap, 3) == slice(96, 128)
    with pytest.raises(IndexError):
        fpsa.tile_of_token(tmap, 256)
    with pytest.raises(IndexError):
        fpsa.flat_tile_index(tmap, (2, 0, 0))


# ----------------------------------------------------------------- windows
MASK_KEYS = ["2_2_2_2_2_2", "7_3_13_3_3_5", "7_9_5_3_3_3", "7_9_5_5_5_3", "4_4_4_6_6_6", "3_5_2_1_4_2",
             "11_9_5_5_5_3", "3_3_5_3_3_1", "3_5_10_3_3_3"]


@pytest.mark.parametrize("key", MASK_KEYS)
def test_window_csr_vs_reference(fpsa, codec_golden, key):
    v = [int(x) for x in key.split("_")]
    m = fpsa.build_block_mask(fpsa.WindowSpec(*v[3:]), tuple(v[:3]))
    assert np.array_equal(m.offsets.astype(np.int64), codec_golden[f"mask_offs_{key}"])
    assert np.array_equal(m.allowed_flat, codec_golden[f"mask_ids_{key}"])
    assert fpsa.density(m) == float(codec_golden[f"mask_density_{key}"])


def test_window_csr_bruteforce_sweep(fpsa):
    """Every tile grid with <= 64 tiles (each axis <= 4) x every window in 1..7^3 (test_acceptance.py:104-125)."""
    dims_list = [d for d in itertools.product(range(1, 5), repeat=3) if d[0] * d[1] * d[2] <= 64]
    wins = list(itertools.product(range(1, 8), repeat=3))
    for dims in dims_list:
        coords = np.array(list(itertools.product(*(range(x) for x in dims))))
        for win in wins:
            m = fpsa.build_block_mask(fpsa.WindowSpec(*win), dims)
            back = np.array([(w - 1) // 2 for w in win])
            fwd = np.array([w // 2 for w in win])
            diff = coords[None, :, :] - coords[:, None, :]  # key - query
            brute = np.all((diff >= -back) & (diff <= fwd), axis=2)
            assert np.array_equal(m.admissible, brute), (dims, win)


def test_window_api(fpsa):
    assert fpsa.neighborhood((0, 0, 0), fpsa.WindowSpec(1, 1, 2), (1, 1, 3)) == [(0, 0, 0), (0, 0, 1)]
    m = fpsa.build_block_mask(fpsa.WindowSpec(1, 1, 3), (1, 1, 4))
    assert m.allowed_counts().tolist() == [2, 3, 3, 2] and fpsa.density(m) == 0.625
    assert fpsa.format_mask_dump(m).splitlines()[1] == "0,0,1 : 0 1 2"
    full = fpsa.full_block_mask((2, 3, 4))
    assert fpsa.density(full) == 1.0
    with pytest.raises(ValueError, match="WindowSpec.win_h must be >= 1"):
        fpsa.WindowSpec(1, 0, 1)
    with pytest.raises(IndexError):
        m.allowed(4)
    tmap = fpsa.build_tile_map(fpsa.GridShape(1, 1, 8, 4), fpsa.TileScheme(1, 1, 2))
    tok = fpsa.expand_token_mask(m, tmap)
    assert tok.shape == (8, 8) and tok[0, 3] and not tok[0, 4]


# ----------------------------------------------------------------- schedule
def test_regimes_vs_reference(fpsa, codec_golden):
    sc = fpsa.default_schedule(50)
    assert [["early", "mid", "late"].index(sc.regime_of(t)) for t in range(1, 51)] == \
        codec_golden["sched_regimes_50"].tolist()
    for D, a1, a2 in [(7, 0.3, 0.6), (1000, 0.2, 0.7), (13, 0.5, 0.9)]:
        s2 = fpsa.ScheduleConfig(alpha1=a1, alpha2=a2, early=sc.early, mid=sc.mid, late=sc.late, total_steps=D)
        got = [["early", "mid", "late"].index(s2.regime_of(t)) for t in range(1, D + 1)]
        assert got == codec_golden[f"sched_regimes_{D}_{a1}_{a2}"].tolist()
    assert fpsa.validate(sc) == []
    assert fpsa.regime_counts(sc) == {"early": 10, "mid": 25, "late": 15}
    with pytest.raises(ValueError):
        sc.regime_of(51)


def test_schedule_validate_violations(fpsa):
    T, W, R = fpsa.TileScheme, fpsa.WindowSpec, fpsa.RegimeParams
    bad = fpsa.ScheduleConfig(alpha1=0.7, alpha2=0.2, early=R(T(1, 1, 1), W(6, 6, 6)), mid=R(T(8, 8, 8), W(1, 1, 1)),
                              late=R(T(2, 2, 2), W(2, 2, 2)), total_steps=0)
    probs = fpsa.validate(bad)
    assert len(probs) == 4
    assert probs[0].startswith("alpha ordering") and probs[2].startswith("granularity ordering")


def test_c4_schedule_is_valid(fpsa):
    """The BASELINE config-5 sweep at the C2 shape passes validate()."""
    T, W, R = fpsa.TileScheme, fpsa.WindowSpec, fpsa.RegimeParams
    sc = fpsa.ScheduleConfig(alpha1=0.2, alpha2=0.7, early=R(T(7, 15, 16), W(3, 3, 1)),
                             mid=R(T(3, 5, 16), W(5, 5, 3)), late=R(T(7, 9, 8), W(3, 3, 3)), total_steps=50)
    assert fpsa.validate(sc) == []
    for t in (1, 10, 11, 35, 36, 50):
        p = fpsa.params_at(t, sc)
        fpsa.build_tile_map(fpsa.GridShape(21, 45, 80, 128), p.tile)


# ----------------------------------------------------------------- work list + accounting
def test_worklist_covers_every_query_block(fpsa):
    from paper_2506_04648_b200.ops import worklist

    for dims, win, tv in [((7, 9, 5), (5, 5, 3), 240), ((7, 3, 13), (3, 3, 5), 120), ((3, 3, 5), (3, 3, 1), 1680),
                          ((3, 5, 10), (3, 3, 3), 504)]:
        m = fpsa.build_block_mask(fpsa.WindowSpec(*win), dims)
        H = 3
        items = worklist(H, m, tv).reshape(-1, 3)
        nqb = -(-tv // 128)
        seen = {(h, u, b) for h, u, b in items.tolist()}
        assert len(seen) == len(items) == H * m.tiles_total * nqb
        counts = np.diff(m.offsets)
        # longest first within each head
        for h in range(H):
            c = counts[items[items[:, 0] == h][:, 1]]
            assert np.all(c[:-1] >= c[1:])


def test_attn_workspace_size(lib):
    n = ctypes.c_int64(0)
    assert lib.fpsa_attn_workspace_bytes(25200, ctypes.byref(n)) == 0
    assert n.value >= 4 * (3 * 25200 + 1)


def test_flops_accounting(fpsa):
    m = fpsa.build_block_mask(fpsa.WindowSpec(5, 5, 3), (7, 9, 5))
    L, d, tv = 75600, 128, 240
    assert fpsa.flops_sparse(L, d, fpsa.density(m)) == m.nnz * 4 * tv * tv * d
    assert fpsa.flops_dense(L, d) == 4 * L * L * d
    with pytest.raises(ValueError):
        fpsa.flops_sparse(L, d, 0.0)


# ----------------------------------------------------------------- device entry points: argument checks only
def test_device_calls_reject_bad_arguments_before_cuda(lib):
    from paper_2506_04648_b200 import _lib

    g, t = _lib.dims3((4, 8, 8)), _lib.dims3((2, 4, 4))
    # d = 48 is unsupported; NULL pointers are invalid
    st = lib.fpsa_quantize_qk(None, _lib.BF16, 48, 0, 1, g, t, 48, 32, _lib.ORDER_TILE, 0, None, None, None, None)
    assert st in (_lib.FPSA_EINVAL, _lib.FPSA_EUNSUPPORTED)
    st = lib.fpsa_quantize_qk(None, _lib.BF16, 64, 0, 1, _lib.dims3((4, 8, 9)), t, 64, 32, _lib.ORDER_TILE, 0,
                              None, None, None, None)
    assert st in (_lib.FPSA_EINVAL, _lib.FPSA_EINDIVISIBLE)
    st = lib.fpsa_attn_fwd(None, None, None, None, None, None, 1, g, t, 64, 128, None, None, None, 1, 0.125, 0, 8.0,
                           _lib.P_ONEPASS, None, _lib.F32, 64, 0, _lib.ORDER_TILE, None, 0, None)
    assert st == _lib.FPSA_EINVAL
    assert lib.fpsa_last_error()
    st = lib.fpsa_attn_fwd(None, None, None, None, None, None, 1, g, t, 64, 128, None, None, None, 1, 0.125, 0, 8.0,
                           7, None, _lib.F32, 64, 0, _lib.ORDER_TILE, None, 0, None)
    assert st == _lib.FPSA_EINVAL and b"p_mode" in lib.fpsa_last_error()
    # the normalised-P mode writes f32 only
    st = lib.fpsa_attn_fwd(None, None, None, None, None, None, 1, g, t, 64, 128, None, None, None, 1, 0.125, 0, 8.0,
                           _lib.P_NORMALIZED, None, _lib.BF16, 64, 0, _lib.ORDER_TILE, None, 0, None)
    assert st == _lib.FPSA_EUNSUPPORTED
    # passthrough entry points
    st = lib.fpsa_tile_gather_bf16(None, _lib.F32, 64, 0, 1, g, t, 64, 128, _lib.ORDER_TILE, None, None)
    assert st == _lib.FPSA_EINVAL
    st = lib.fpsa_tile_gather_bf16(None, _lib.F32, 48, 0, 1, g, t, 48, 128, _lib.ORDER_TILE, None, None)
    assert st == _lib.FPSA_EINVAL  # NULL checked first
    st = lib.fpsa_attn_bf16_fwd(None, None, None, 1, g, t, 64, 128, None, None, None, 1, 0.125, None, _lib.F32, 64,
                                0, _lib.ORDER_TILE, None, 0, None)
    assert st == _lib.FPSA_EINVAL
    st = lib.fpsa_fidelity(None, _lib.F32, None, _lib.F32, 10, 1, 64, 64, 0, None, None)
    assert st == _lib.FPSA_EINVAL


def test_fidelity_from_sums_matches_reference_metrics(fpsa):
    """Host finish of the device fidelity sums == fp8sta/metrics.py:41-88 conventions."""
    import math

    import oracle as O

    rng = np.random.default_rng(3)
    x = rng.standard_normal(4096)
    y = x + 1e-2 * rng.standard_normal(4096)
    sums = (float(x @ y), float(x @ x), float(y @ y), float((x - y) @ (x - y)), float(abs(x).max()),
            float(abs(y).max()))
    cos, mse, snr = fpsa.fidelity_from_sums(*sums, n=x.size)
    assert abs(cos - O.cosine(x, y)) < 1e-12
    assert abs(mse - float(((x - y) ** 2).mean())) < 1e-15
    assert abs(snr - 10 * math.log10((x @ x) / ((x - y) @ (x - y)))) < 1e-9
    with pytest.raises(ValueError):  # all-zero reference: SNR undefined (metrics.py:77-78)
        fpsa.fidelity_from_sums(0, 0, 0, 0, 0.0, 0.0, n=4)
    assert fpsa.fidelity_from_sums(0, 1, 0, 1, 1.0, 0.0, n=4)[0] == 0.0  # one zero vector: cosine 0
    assert fpsa.fidelity_from_sums(*sums[:3], 0.0, *sums[4:], n=x.size)[2] == math.inf


def test_plan_cache_is_lru_bounded():
    from paper_2506_04648_b200.ops import cache_get

    cache, made = {}, []
    for k in [1, 2, 3, 1, 4, 5]:
        cache_get(cache, k, lambda k=k: made.append(k) or k, limit=3)
    assert made == [1, 2, 3, 4, 5]          # 1 was a hit the second time
    assert list(cache) == [1, 4, 5]         # least recently used (2, then 3) dropped
    assert len(cache) == 3 and 5 in cache and 2 not in cache
