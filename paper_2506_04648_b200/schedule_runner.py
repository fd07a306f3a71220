"""Denoising-step driver: per-step (tile, window) from the schedule, one device plan per regime.

Mirrors the reference's per-step loop (fp8sta/experiment.py:178-201: for t
in 1..D, ``params_at(t)`` picks the regime's tile and window, schedule.py:71-73)
for the GPU hot path.  Each regime gets one ``FpsaPlan`` (window CSR, work
list and FP8 buffers built once) and, optionally, one CUDA graph of its
quantise + attention launches, so a step is a single graph replay.  Rows
follow the reference CSV schema (experiment.py:25-28) plus timing columns.
With ``fidelity=True`` every step also runs the full-precision passthrough
kernel (PassthroughPlan, outside the timed region) and fills the cosine /
mse / snr columns the way experiment._evaluate / _row do
(experiment.py:118-160): per head against the sparse full-precision
attention, then the mean over heads.  Otherwise they are nan.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .fp8 import E4M3, Fp8Format
from .grid import GridShape, build_tile_map
from .metrics import flops_dense, flops_sparse
from .ops import FpsaPlan, PassthroughPlan, device_fidelity
from .schedule import ScheduleConfig, params_at, validate
from .sparsity import build_block_mask, density

CSV_HEADER = (
    "step,regime,tile_t,tile_h,tile_w,win_t,win_h,win_w,"
    "density,flops_dense,flops_sparse,cosine_sim,mse,snr_db,ms,eff_tflops"
)


@dataclass(frozen=True)
class StepRow:
    step: int
    regime: str
    tile: tuple[int, int, int]
    window: tuple[int, int, int]
    density: float
    flops_dense: int  # per head, as the reference reports it
    flops_sparse: int
    ms: float  # all heads, quantise + attention
    eff_tflops: float  # flops_sparse * heads / ms
    cosine_sim: float = math.nan
    mse: float = math.nan
    snr_db: float = math.nan


def _mean(values: list[float]) -> float:
    """experiment.py:_mean: fsum / n, or inf if any value is inf."""
    return math.fsum(values) / len(values) if math.inf not in values else math.inf


class ScheduleRunner:
    """Runs the hot path for every sampling step of a schedule on [L, H, d] bf16 inputs."""

    def __init__(self, grid: tuple[int, int, int], schedule: ScheduleConfig, heads: int, d: int,
                 fmt: Fp8Format = E4M3, device="cuda", use_graphs: bool = True, tau: float = 8.0,
                 fidelity: bool = False, p_mode: str = "onepass"):
        problems = validate(schedule)
        if problems:
            raise ValueError("invalid schedule: " + "; ".join(problems))
        self.grid = tuple(int(x) for x in grid)
        self.schedule, self.heads, self.d = schedule, int(heads), int(d)
        self.fmt, self.device, self.use_graphs, self.tau = fmt, device, use_graphs, tau
        self.fidelity, self.p_mode = fidelity, p_mode
        self._plans: dict = {}
        self._ref_plans: dict = {}
        self._ref_out = None
        self._graphs: dict = {}
        gshape = GridShape(*self.grid, self.d)
        for regime in ("early", "mid", "late"):  # reject indivisible tiles up front (grid.py:95-99)
            build_tile_map(gshape, schedule.params(regime).tile)

    def plan(self, regime: str) -> FpsaPlan:
        p = self._plans.get(regime)
        if p is None:
            rp = self.schedule.params(regime)
            p = FpsaPlan(self.grid, rp.tile.dims, rp.window, self.heads, self.d, self.fmt, device=self.device,
                         tau=self.tau, p_mode=self.p_mode)
            self._plans[regime] = p
        return p

    def reference(self, regime: str, q, k, v):
        """Full-precision sparse attention of the regime's (tile, window) into a reused f32 buffer."""
        import torch

        p = self._ref_plans.get(regime)
        if p is None:
            rp = self.schedule.params(regime)
            p = PassthroughPlan(self.grid, rp.tile.dims, rp.window, self.heads, self.d, device=self.device)
            self._ref_plans[regime] = p
        if self._ref_out is None or self._ref_out.shape != q.shape:
            self._ref_out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        p(q, k, v, "lhd", out=self._ref_out)
        return self._ref_out

    def step(self, t: int, q, k, v, out) -> str:
        """Quantise + attend for sampling step t (1-based); returns the regime."""
        regime = self.schedule.regime_of(t)
        plan = self.plan(regime)
        if not self.use_graphs:
            plan.quantize(q, k, v, "lhd")
            plan.attention(out, "lhd")
            return regime
        import torch

        key = (regime, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr())
        g = self._graphs.get(key)
        if g is None:
            # warm the launch configuration outside the capture, then capture both launches
            plan.quantize(q, k, v, "lhd")
            plan.attention(out, "lhd")
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                plan.quantize(q, k, v, "lhd")
                plan.attention(out, "lhd")
            self._graphs[key] = g
        g.replay()
        return regime

    def run(self, q, k, v, out, steps: int | None = None) -> list[StepRow]:
        """All (or the first `steps`) sampling steps, each timed with CUDA events."""
        import torch

        D = self.schedule.total_steps if steps is None else min(steps, self.schedule.total_steps)
        L = self.grid[0] * self.grid[1] * self.grid[2]
        stream = torch.cuda.current_stream()
        rows = []
        for t in range(1, D + 1):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            regime = self.step(t, q, k, v, out)
            e.record(stream)
            e.synchronize()
            ms = s.elapsed_time(e)
            rp = self.schedule.params(regime)
            plan = self._plans[regime]
            dens = plan.density
            fid = {}
            if self.fidelity:
                per_head = device_fidelity(self.reference(regime, q, k, v), out, "lhd")
                fid = dict(cosine_sim=_mean([m[0] for m in per_head]), mse=_mean([m[1] for m in per_head]),
                           snr_db=_mean([m[2] for m in per_head]))
            rows.append(StepRow(step=t, regime=regime, tile=rp.tile.dims, window=rp.window.dims, density=dens,
                                flops_dense=flops_dense(L, self.d), flops_sparse=flops_sparse(L, self.d, dens),
                                ms=ms, eff_tflops=plan.flops / (ms * 1e-3) / 1e12, **fid))
        return rows


def rows_to_csv(rows: list[StepRow]) -> str:
    """Reference CSV schema (experiment.py:249-260) + ms and effective TFLOPS (fidelity nan unless measured)."""
    lines = [CSV_HEADER]
    for r in rows:
        lines.append(
            f"{r.step},{r.regime},{r.tile[0]},{r.tile[1]},{r.tile[2]},{r.window[0]},{r.window[1]},{r.window[2]},"
            f"{r.density!r},{r.flops_dense},{r.flops_sparse},{r.cosine_sim!r},{r.mse!r},{r.snr_db!r},"
            f"{r.ms!r},{r.eff_tflops!r}")
    return "\n".join(lines) + "\n"


def c4_schedule(total_steps: int = 50) -> ScheduleConfig:
    """BASELINE config 5 at the Wan2.1-14B 720p shape: a schedule validate() accepts."""
    from .grid import TileScheme
    from .schedule import RegimeParams
    from .sparsity import WindowSpec

    return ScheduleConfig(alpha1=0.2, alpha2=0.7,
                          early=RegimeParams(TileScheme(7, 15, 16), WindowSpec(3, 3, 1)),
                          mid=RegimeParams(TileScheme(3, 5, 16), WindowSpec(5, 5, 3)),
                          late=RegimeParams(TileScheme(7, 9, 8), WindowSpec(3, 3, 3)),
                          total_steps=total_steps)


def schedule_density(grid, schedule: ScheduleConfig, t: int) -> float:
    """Density of step t's window (host only; sparsity.py:141-144)."""
    rp = params_at(t, schedule)
    tmap = build_tile_map(GridShape(*grid, 1), rp.tile)
    return density(build_block_mask(rp.window, tmap.tile_grid_dims))
