"""Benchmark: sliding-tile sparse FP8 attention forward at the Wan2.1-14B 720p shape.

One step = the hot path over one batch element: per-tile Q/K and per-channel
V FP8 quantisation of bf16 [L, H, d] inputs in natural (t,h,w) order, then
the sparse FP8 attention forward writing bf16 [L, H, d] (libfpsa kernels).
N GPUs: one process per GPU (torchrun), heads split across ranks
(head-parallel, strong scaling: the same 40-head problem on 1..8 GPUs, no
data-path collective); timing = max over ranks.  ``--ulysses`` instead
feeds sequence-sharded inputs and adds the NCCL sequence<->head all-to-all
(BASELINE config C3, HunyuanVideo 720p).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME] [--ulysses]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse FP8 attn fwd ms + eff. TFLOPS (% FP8 peak) @Wan2.1-14B 720p, 1/2/4/8 GPU"
FP8_SPEC_TFLOPS = 4500.0

CONFIGS = {
    # name: grid, heads, d, tile, window
    "wan14b_720p": ((21, 45, 80), 40, 128, (3, 5, 16), (5, 5, 3)),
    "wan14b_720p_w333": ((21, 45, 80), 40, 128, (3, 5, 16), (3, 3, 3)),
    "wan13b_480p": ((21, 30, 52), 12, 128, (3, 10, 4), (3, 3, 5)),
    "hunyuan_720p": ((33, 45, 80), 24, 128, (3, 5, 16), (5, 5, 3)),
    # the C4 schedule's early and late regimes (schedule_runner.c4_schedule) at the 14B 720p grid
    "c4_early": ((21, 45, 80), 40, 128, (7, 15, 16), (3, 3, 1)),
    "c4_late": ((21, 45, 80), 40, 128, (7, 9, 8), (3, 3, 3)),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="wan14b_720p", choices=sorted(CONFIGS))
    ap.add_argument("--tau", type=float, default=8.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="heads per host-streaming chunk (0: 2, the measured best at C2: 44.8 ms vs 46.6 for 5)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--ulysses", action="store_true", help="sequence-sharded inputs + all-to-all (C3)")
    ap.add_argument("--ulysses-chunk", type=int, default=1,
                    help="heads per pipelined all-to-all chunk (0: one all-to-all per tensor, no overlap)")
    ap.add_argument("--p-mode", default="onepass", choices=["onepass", "normalized"],
                    help="softmax-weight semantics (normalized: the reference's arithmetic, f32 output)")
    ap.add_argument("--dump-out", default=None,
                    help="directory: each rank writes sha256 of its heads' outputs (head-parallel runs)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch(n: int) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks of this script (one process per GPU)
    under torch.distributed.run on 127.0.0.1 and return their exit status (rank 0 prints the line)."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


class Group:
    """Process group for the timing collectives (barrier, max over ranks).  NCCL when every rank has its
    own GPU; gloo when ranks share one (the CPU-side multi-rank test: NCCL refuses two ranks on a device)."""

    def __init__(self, world: int, local: int, torch, dist):
        self.world, self.dist, self.torch = world, dist, torch
        n_dev = torch.cuda.device_count()
        self.device = torch.device("cuda", local % n_dev)
        torch.cuda.set_device(self.device)
        self.backend = None
        if world > 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
            self.backend = "nccl" if n_dev >= local_world else "gloo"
            kw = {"device_id": self.device} if self.backend == "nccl" else {}
            dist.init_process_group(self.backend, **kw)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, values):
        if self.world == 1:
            return list(values)
        dev = self.device if self.backend == "nccl" else "cpu"
        t = self.torch.tensor(list(values), device=dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x4: "sw_power_cap", 0x1: "gpu_idle", 0x2: "applications_clocks_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # pragma: no cover - reported in the JSON
            self.nvml, self.err = None, str(exc)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def summary(self):
        if not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- peaks
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def fp8_gemm_peak(torch):
    """Same-run dense FP8 GEMM throughput (cuBLAS via torch._scaled_mm, 8192^3, best of 10), TF/s."""
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn)
        b = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn).t()
        one = torch.ones((), device="cuda")
        for _ in range(3):
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        return 2 * n ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


def ncu_traffic(config_name: str):
    """dram bytes per attention launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "attn_ncu_summary.json")
    try:
        with open(path) as f:
            data = json.load(f)
        return data.get(config_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------- CPU legs
def _cpu_setup(cfg, seed: int = 0):
    import oracle as O

    grid, H, d, tile, win = cfg
    L = grid[0] * grid[1] * grid[2]
    tv = tile[0] * tile[1] * tile[2]
    q, k, v = O.gen_inputs(seed, 1, 0, L, d)
    dims = O.tile_grid_dims(grid, tile)
    offs, ids = O.window_lists(dims, win)
    return q, k, v, tv, offs, ids, dims[0] * dims[1] * dims[2]


def cpu_passes(cfg, warmup: int, steps: int, budget_s: float):
    """The reference algorithm (oracle port of fp8sta.fp8_sparse_forward: quantise the key tiles, then attend
    every query tile, thread pool over tiles) on the host cores.  A step is one pass over all query tiles of
    head 0 -- the reference's own unit of work -- unless warmup + steps full passes would exceed budget_s, in
    which case each step attends an even sample of the query tiles (and quantises the key tiles they need).
    Both CPU legs of this file use it, so they agree.  Returns (flops, seconds, tiles per step, M)."""
    from oracle.cpu_sample import sample_forward, sample_tiles

    q, k, v, tv, offs, ids, M = _cpu_setup(cfg)
    tiles = sample_tiles(M, M)
    _, _, s_full = sample_forward(q, k, v, tv, offs, ids, tiles)  # also the first warm-up pass
    if (warmup + steps) * s_full > budget_s:
        tiles = sample_tiles(M, max(2, int(M * budget_s / ((warmup + steps) * s_full))))
    for _ in range(max(0, warmup - 1)):
        sample_forward(q, k, v, tv, offs, ids, tiles)
    fl = secs = 0.0
    for _ in range(steps):
        _, f, s = sample_forward(q, k, v, tv, offs, ids, tiles)
        fl, secs = fl + f, secs + s
    return fl, secs, len(tiles), M


def cpu_sample_text(n_tiles: int, M: int, H: int) -> str:
    part = "all" if n_tiles == M else f"an even sample of {n_tiles} of the"
    return (f"per step: {part} {M} query tiles of 1 of {H} heads (oracle port of fp8sta.fp8_sparse_forward, "
            f"numpy, thread pool of {os.cpu_count()} over query tiles; key tiles quantised once per step)")


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port) on the host cores, rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    grid, H, d, tile, win = cfg
    fl, secs, n_tiles, M = cpu_passes(cfg, args.warmup, args.steps, budget_s=150.0)
    tflops = fl / secs / 1e12
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Philox gaussian, reference generator; the GPU arm draws the same N(0,1) with torch)",
        "config": {"workload": args.config, "grid": grid, "heads": H, "d": d, "tile": tile, "window": win},
        "cpu_baseline": {"value": tflops, "unit": "TFLOPS", "cores": cores, "kind": "port",
                         "sample": cpu_sample_text(n_tiles, M, H)},
        "e2e": {"value": tflops, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------- GPU leg
def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args.gpus)
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but the launcher started {world} rank(s)")
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2506_04648_b200 as fpsa

    group = Group(world, local, torch, dist)
    dev = group.device
    grid, H, d, tile, win = CONFIGS[args.config]
    L = grid[0] * grid[1] * grid[2]
    from paper_2506_04648_b200.sharding import UlyssesAttention, head_range

    if args.ulysses:
        if world < 2 or H % world or L % world:
            raise SystemExit("--ulysses needs >= 2 ranks dividing both the heads and the tokens")
        if group.backend != "nccl":
            raise SystemExit("--ulysses needs one GPU per rank (NCCL all-to-all)")
        h0, h1 = 0, H  # every rank holds all heads of its token shard
        Lr, Hr = L // world, H
    else:
        h0, h1 = head_range(rank, world, H)
        Lr, Hr = L, h1 - h0
    gen = torch.Generator(device=dev)
    if args.ulysses:
        gen.manual_seed(1234 + rank)
        q, k, v = (torch.randn((Lr, Hr, d), generator=gen, device=dev).to(torch.bfloat16) for _ in range(3))
    else:
        # per-head seeds: head h gets the same q, k, v whatever the rank count (--dump-out compares them)
        q, k, v = (torch.empty((Lr, Hr, d), dtype=torch.bfloat16, device=dev) for _ in range(3))
        for j in range(Hr):
            gen.manual_seed(1234 + h0 + j)
            for x in (q, k, v):
                x[:, j].copy_(torch.randn((Lr, d), generator=gen, device=dev))
    out = torch.empty_like(q) if args.p_mode == "onepass" else torch.empty(q.shape, dtype=torch.float32, device=dev)
    if args.ulysses:
        uly = UlyssesAttention(grid, tile, win, H, d, device=dev, tau=args.tau,
                               chunk_heads=args.ulysses_chunk or None)
        plan = uly.plan

        def step(q_, k_, v_, out_):
            out_.copy_(uly(q_, k_, v_))
    else:
        plan = fpsa.FpsaPlan(grid, tile, win, Hr, d, tau=args.tau, device=dev, p_mode=args.p_mode)

        def step(q_, k_, v_, out_):
            plan.quantize(q_, k_, v_, "lhd")
            plan.attention(out_, "lhd")
    flops = plan.flops  # this rank's heads
    flops_total = plan.flops // plan.heads * H if not args.ulysses else plan.flops * world

    barrier = group.barrier

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step(q, k, v, out)
    torch.cuda.synchronize()
    plan.check_finite()
    redo = plan.redo_count()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            if args.ulysses:
                step(q, k, v, out)
                ev[i][1].record(stream)
            else:
                plan.quantize(q, k, v, "lhd")
                ev[i][1].record(stream)
                plan.attention(out, "lhd")
            ev[i][2].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = t0.elapsed_time(t1)
    ms_quant = sum(a.elapsed_time(b) for a, b, _ in ev) / args.steps
    ms_attn = sum(b.elapsed_time(c) for _, b, c in ev) / args.steps
    ms_step = ms_total / args.steps
    ms_step, ms_attn, ms_quant = group.max([ms_step, ms_attn, ms_quant])
    total_flops = flops_total
    value = total_flops / (ms_step * 1e-3) / 1e12

    # ---------------- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
        oh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        steps_e2e = max(3, min(args.steps, 10))
        if args.ulysses:
            qd, kd, vd = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

            def e2e_step():
                qd.copy_(qh, non_blocking=True); kd.copy_(kh, non_blocking=True); vd.copy_(vh, non_blocking=True)
                step(qd, kd, vd, out)
                oh.copy_(out, non_blocking=True)
        else:
            # head chunks: the H2D of chunk c+1 and the D2H of chunk c-1 overlap chunk c's kernels
            streamer = fpsa.HostStreamer(grid, tile, win, Hr, d, chunk_heads=args.e2e_chunk or min(Hr, 2),
                                         tau=args.tau, device=dev)

            def e2e_step():
                streamer(qh, kh, vh, oh)
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(steps_e2e):
            e2e_step()
        e.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = s.elapsed_time(e) / steps_e2e
        (ms_e2e,) = group.max([ms_e2e])
        e2e = {"value": total_flops / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOPS", "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": 3 * q.numel() * q.element_size(),
               "d2h_bytes_per_step": out.numel() * out.element_size(),
               "api": ("paper_2506_04648_b200.UlyssesAttention.__call__" if args.ulysses else
                       "paper_2506_04648_b200.HostStreamer.__call__ (FpsaPlan.quantize + .attention per head chunk, "
                       "fpsa_copy2d transfers overlapped)") + " via the C ABI, pinned host"}

    if args.dump_out and not args.ulysses:
        import hashlib

        step(q, k, v, out)
        torch.cuda.synchronize()
        os.makedirs(args.dump_out, exist_ok=True)
        digests = {str(h0 + j): hashlib.sha256(out[:, j].contiguous().view(torch.int16).cpu().numpy().tobytes()).hexdigest()
                   for j in range(Hr)}
        with open(os.path.join(args.dump_out, f"rank{rank}.json"), "w") as f:
            json.dump(digests, f)
    if rank != 0:
        group.close()
        return 0

    peaks = measured_peaks()
    fp8_meas = fp8_gemm_peak(torch)
    if fp8_meas:
        peak, peak_src = fp8_meas, "same-run cuBLAS FP8 e4m3 GEMM 8192^3 (torch._scaled_mm), burst"
    else:
        peak = 2.0 * float(peaks.get("bf16_tflops", 1590.0))
        peak_src = "2 x measured bf16 dense (MEASURED_PEAKS.json)"
    attn_tflops = flops / (ms_attn * 1e-3) / 1e12 if not args.ulysses else None
    # quantiser: algorithmic bytes = bf16 q,k,v read once + e4m3 codes written (9 B per element)
    qbytes = 3 * L * Hr * d * 2 + 3 * L * Hr * d
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "TFLOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "e4m3",
        "data": "synthetic (torch.randn bf16 q/k/v, natural (t,h,w) token order)",
        "config": {
            "workload": args.config, "grid": grid, "heads": H, "d": d, "tile": tile, "window": win,
            "density": plan.density, "global_batch": 1, "heads_per_gpu": Hr if not args.ulysses else H // world,
            "flops_per_step": total_flops, "flops_per_step_rank0": flops, "tau_log2": args.tau,
            "p_mode": args.p_mode,
            "parallelism": (f"ulysses: sequence-sharded inputs, NCCL all-to-all seq<->head, {world} ranks"
                            if args.ulysses else f"head-parallel, {world} rank(s), no collective"),
            "l2": "inputs larger than L2 (bf16 q,k,v = %.2f GB per rank; codes %.2f GB)" % (
                3 * q.numel() * 2 / 1e9, 3 * plan.q_codes.numel() / 1e9),
        },
        "ms_attention": ms_attn,
        "ms_quantize": ms_quant,
        "redo_items": redo,
        "frac_fp8_spec": attn_tflops / FP8_SPEC_TFLOPS if attn_tflops else None,
        "step_frac_fp8_spec": value / world / FP8_SPEC_TFLOPS,
        "roofline": None if args.ulysses else {
            "bound": "tensor", "kernel": "fpsa_attn_kernel", "achieved": attn_tflops, "peak": peak,
            "unit": "TFLOP/s", "frac": attn_tflops / peak, "peak_source": peak_src,
            "traffic": ncu_traffic(args.config),
            "algorithmic": "sum_u |W(u)| * 4 tv^2 d per head (metrics.py:91-102), %d FLOP per launch" % flops,
        },
        "roofline_quantize": {
            "bound": "hbm", "kernels": "chan_amax_kernel + quant_tma_kernel (q,k,v in one launch)",
            "achieved": qbytes / (ms_quant * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": qbytes / (ms_quant * 1e-3) / 1e9 / hbm, "algorithmic_bytes": qbytes,
        },
        "clocks": clocks.summary(),
        "gpu_launches": 4 * args.steps,  # chan_amax + quant_tma + fpsa_attn (main + exact redo) per step
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu:
        fl, secs, n_tiles, M = cpu_passes(CONFIGS[args.config], 1, 2, budget_s=args.cpu_seconds)
        line["cpu_baseline"] = {"value": fl / secs / 1e12, "unit": "TFLOPS", "cores": os.cpu_count(),
                                "kind": "port", "sample": cpu_sample_text(n_tiles, M, H) + f", {secs:.1f} s timed"}
    print(json.dumps(line))
    group.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
