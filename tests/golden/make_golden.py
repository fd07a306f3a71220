"""Freeze golden vectors from the reference package ``fp8sta`` (build container only).

Run from the repo root:  python tests/golden/make_golden.py
It imports the reference from /root/reference/pkg/src (read-only, not present
on the GPU box) and writes small .npz fixtures next to this script.  The
fixtures pin the CPU oracle (oracle/fpsa_oracle.py) and, through it, the CUDA
path: codes, scales, permutations and window lists are bit-pinned; attention
outputs are float32 results of the reference's numpy/BLAS engine, compared
with a tolerance (BLAS summation order is platform dependent).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import fp8sta  # noqa: E402
from fp8sta import experiment, fp8, grid, quantize, schedule, sparsity  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def adversarial_quotients(rng, fmt, n_peaks=96):
    """x values whose quotient x/scale sits on / next to every fp8 midpoint."""
    vals = fp8.code_table(fmt)[:128]
    finite = vals[np.isfinite(vals)]
    mids = (finite[:-1] + finite[1:]) / 2.0
    xs = []
    for _ in range(n_peaks):
        peak = np.float32(np.exp2(rng.uniform(-20, 20)) * rng.uniform(1, 2))
        scale = float(peak) / fmt.max_value
        base = (mids * scale).astype(np.float32)
        up = np.nextafter(base, np.float32(np.inf))
        dn = np.nextafter(base, np.float32(-np.inf))
        block = np.concatenate([base, up, dn, -base, -up, -dn, [peak, -peak, 0.0, -0.0]]).astype(np.float32)
        xs.append(block)
    return xs


def main():
    rng = np.random.default_rng(20250604)
    out = {}

    # ---- FP8 codec
    for fmt in (fp8.E4M3, fp8.E5M2):
        out[f"table_{fmt.name}"] = fp8.code_table(fmt)
        x = np.concatenate([
            rng.standard_normal(20000) * np.exp2(rng.uniform(-12, 12, 20000)),
            rng.uniform(-fmt.max_value * 1.2, fmt.max_value * 1.2, 20000),
            np.array([0.0, -0.0, 2.0**-9, -(2.0**-9), 2.0**-10, 1.0625, 1.1875, fmt.max_value,
                      fmt.max_value * 1.01, 1e30, -1e30, 5e-324]),
        ])
        out[f"enc_x_{fmt.name}"] = x
        out[f"enc_c_{fmt.name}"] = fp8.encode(x, fmt)
        x32 = x.astype(np.float32)
        out[f"enc32_x_{fmt.name}"] = x32
        out[f"enc32_c_{fmt.name}"] = fp8.encode(x32, fmt)

    # ---- adversarial tile quantisation (near-tie quotients), one tile per peak
    adv = adversarial_quotients(rng, fp8.E4M3)
    width = max(len(a) for a in adv)
    tiles = np.zeros((len(adv), width), dtype=np.float32)
    for i, a in enumerate(adv):
        tiles[i, : len(a)] = a
    # as a (tiles*rows, 64) matrix with tv rows per tile: pad width to multiple of 64
    d = 64
    rows_per_tile = -(-width // d)
    mat = np.zeros((len(adv), rows_per_tile * d), dtype=np.float32)
    mat[:, :width] = tiles
    mat = mat.reshape(len(adv) * rows_per_tile, d)
    g = grid.GridShape(len(adv), 1, rows_per_tile, d)
    tm = grid.build_tile_map(g, grid.TileScheme(1, 1, rows_per_tile))
    qt = quantize.quantize_qk_tilewise(mat, tm, fp8.E4M3)
    out["adv_x"] = mat
    out["adv_tile_rows"] = np.int64(rows_per_tile)
    out["adv_codes"] = qt.codes
    out["adv_scales"] = qt.scales

    # ---- layouts / masks
    perms = {}
    for gd, td in [((4, 8, 8), (2, 4, 4)), ((6, 8, 8), (3, 4, 4)), ((6, 10, 16), (3, 10, 4)),
                   ((7, 9, 16), (7, 9, 8)), ((4, 6, 10), (2, 3, 5))]:
        tmap = grid.build_tile_map(grid.GridShape(*gd, 8), grid.TileScheme(*td))
        key = "perm_" + "_".join(map(str, gd + td))
        perms[key] = grid.tile_contiguous_order(tmap)
    out.update(perms)

    masks = {}
    for dims, win in [((2, 2, 2), (2, 2, 2)), ((7, 3, 13), (3, 3, 5)), ((7, 9, 5), (3, 3, 3)),
                      ((7, 9, 5), (5, 5, 3)), ((4, 4, 4), (6, 6, 6)), ((3, 5, 2), (1, 4, 2)),
                      ((11, 9, 5), (5, 5, 3)), ((3, 3, 5), (3, 3, 1)), ((3, 5, 10), (3, 3, 3))]:
        m = sparsity.build_block_mask(sparsity.WindowSpec(*win), dims)
        key = "_".join(map(str, dims + win))
        counts = m.allowed_counts()
        masks[f"mask_offs_{key}"] = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        masks[f"mask_ids_{key}"] = m.allowed_flat.astype(np.int64)
        masks[f"mask_density_{key}"] = np.float64(sparsity.density(m))
    out.update(masks)

    # ---- schedule
    sc = schedule.default_schedule(50)
    out["sched_regimes_50"] = np.array([["early", "mid", "late"].index(sc.regime_of(t)) for t in range(1, 51)])
    for D, a1, a2 in [(7, 0.3, 0.6), (1000, 0.2, 0.7), (13, 0.5, 0.9)]:
        sc2 = schedule.ScheduleConfig(alpha1=a1, alpha2=a2, early=sc.early, mid=sc.mid, late=sc.late, total_steps=D)
        out[f"sched_regimes_{D}_{a1}_{a2}"] = np.array(
            [["early", "mid", "late"].index(sc2.regime_of(t)) for t in range(1, D + 1)])

    np.savez_compressed(os.path.join(OUT, "codec_layout.npz"), **out)

    # ---- attention cases (single head, tile-contiguous rows, reference inputs)
    cases = [
        # name, grid, d, tile, window, fmt, seed, dist
        ("c0_toy", (4, 8, 8), 64, (2, 4, 4), (2, 2, 2), "e4m3", 7, "gaussian"),
        ("c0_toy_full", (4, 8, 8), 64, (2, 4, 4), (4, 4, 4), "e4m3", 8, "gaussian"),
        ("small_d128", (4, 16, 16), 128, (2, 4, 16), (3, 3, 3), "e4m3", 11, "gaussian"),
        ("tv120_d128", (6, 10, 16), 128, (3, 10, 4), (3, 3, 5), "e4m3", 12, "gaussian"),
        ("tv240_d128", (6, 10, 32), 128, (3, 5, 16), (3, 3, 3), "e4m3", 13, "gaussian"),
        ("tv240_heavy", (6, 10, 32), 128, (3, 5, 16), (5, 5, 3), "e4m3", 14, "heavy"),
        ("tv240_e5m2", (6, 10, 32), 128, (3, 5, 16), (3, 3, 3), "e5m2", 15, "gaussian"),
        ("tv504_d128", (7, 9, 16), 128, (7, 9, 8), (3, 3, 3), "e4m3", 16, "gaussian"),
        ("tv256_d64", (4, 16, 32), 64, (2, 8, 16), (3, 3, 3), "e4m3", 17, "uniform"),
    ]
    att = {}
    for name, gd, d, td, win, fmtname, seed, dist in cases:
        gshape = grid.GridShape(*gd, d)
        tmap = grid.build_tile_map(gshape, grid.TileScheme(*td))
        sched = schedule.ScheduleConfig(
            alpha1=0.2, alpha2=0.7,
            early=schedule.RegimeParams(grid.TileScheme(*td), sparsity.WindowSpec(*win)),
            mid=schedule.RegimeParams(grid.TileScheme(*td), sparsity.WindowSpec(*win)),
            late=schedule.RegimeParams(grid.TileScheme(*td), sparsity.WindowSpec(*win)),
            total_steps=1)
        cfg = experiment.ExperimentConfig(grid=gshape, schedule=sched, seed=seed, heads=1, fmt_name=fmtname,
                                          distribution=experiment.InputDistribution(dist))
        inp = experiment.gen_inputs(cfg, tmap, 1, 0)
        fmt = fp8.FORMATS[fmtname]
        fc = fp8sta.ForwardConfig(window=sparsity.WindowSpec(*win), fmt=fmt)
        o = fp8sta.fp8_sparse_forward(inp, fc)
        mask = sparsity.build_block_mask(sparsity.WindowSpec(*win), tmap.tile_grid_dims)
        ref = fp8sta.sparse_reference(inp, mask)
        qq = quantize.quantize_qk_tilewise(inp.q, tmap, fmt)
        qk = quantize.quantize_qk_tilewise(inp.k, tmap, fmt)
        qv = quantize.quantize_v_channelwise(inp.v, fmt)
        att[f"{name}__meta"] = np.array(list(gd) + [d] + list(td) + list(win) + [0 if fmtname == "e4m3" else 1]
                                        + [seed, ["gaussian", "uniform", "heavy"].index(dist)])
        # inputs are not stored: oracle.gen_inputs restates the reference's Philox
        # generator (experiment.py:90-115); a checksum pins that restatement
        att[f"{name}__in_sum"] = np.array([inp.q.astype(np.float64).sum(), inp.k.astype(np.float64).sum(),
                                           inp.v.astype(np.float64).sum(), float(inp.q[0, 0]), float(inp.v[-1, -1])])
        rows = np.unique(np.concatenate([np.arange(min(128, gshape.tokens)),
                                         np.arange(gshape.tokens - min(64, gshape.tokens), gshape.tokens)]))
        att[f"{name}__rows"] = rows
        att[f"{name}__out"] = o[rows]
        att[f"{name}__sparse_ref"] = ref[rows]  # passthrough golden (attention.py:192-194)
        att[f"{name}__q_scales"] = qq.scales
        att[f"{name}__k_scales"] = qk.scales
        att[f"{name}__v_scales"] = qv.scales
        small = gshape.tokens <= 256
        for nm, qt in (("q", qq), ("k", qk), ("v", qv)):
            att[f"{name}__{nm}_codes_rows"] = qt.codes[rows] if not small else qt.codes
        print(f"{name}: L={gshape.tokens} out max {np.abs(o).max():.3f}")
    np.savez_compressed(os.path.join(OUT, "attention_cases.npz"), **att)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
