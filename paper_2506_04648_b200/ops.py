"""Device path: quantise + sliding-tile sparse FP8 attention on B200 through libfpsa.

``FpsaPlan`` owns the device state of one problem shape (window CSR, work
list, FP8 code / scale buffers) so repeated calls allocate nothing;
``fps_attention`` is the one-call functional form.  Tensors are torch CUDA
tensors; torch supplies device memory and the current stream, all compute is
in libfpsa's sm_100a kernels.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import _lib
from .fp8 import E4M3, Fp8Format
from .sparsity import BlockMask, WindowSpec, build_block_mask

BLOCK = 128  # rows per query block / keys per key block of the attention kernel


def _torch():
    import torch  # local import: host-only users of the package need no CUDA

    return torch


def _ptr(t) -> int:
    return t.data_ptr()


def _stream(device=None):
    return _torch().cuda.current_stream(device).cuda_stream


P_MODES = {"onepass": _lib.P_ONEPASS, "normalized": _lib.P_NORMALIZED}


def _dtype_id(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return _lib.F32
    if t.dtype == torch.bfloat16:
        return _lib.BF16
    raise NotImplementedError(f"input dtype {t.dtype} not supported (float32 / bfloat16)")


def tile_pitch(tile_volume: int) -> int:
    """Rows per tile slot in the padded code layout (multiple of 128)."""
    return -(-tile_volume // BLOCK) * BLOCK


def worklist(heads: int, mask: BlockMask, tile_volume: int) -> np.ndarray:
    """(head, query tile, query block) items, longest first within each head."""
    L = _lib.lib()
    n = ctypes.c_int64(0)
    td = _lib.dims3(mask.tile_grid_dims)
    offs = np.ascontiguousarray(mask.offsets, dtype=np.int32)
    _lib.check(L.fpsa_attn_worklist(heads, td, tile_volume, offs.ctypes.data_as(_lib._pi32), None, 0,
                                    ctypes.byref(n)))
    items = np.empty(3 * n.value, dtype=np.int32)
    _lib.check(L.fpsa_attn_worklist(heads, td, tile_volume, offs.ctypes.data_as(_lib._pi32),
                                    items.ctypes.data_as(_lib._pi32), n.value, ctypes.byref(n)))
    return items


class _TilePlan:
    """Shape-derived device state shared by the FP8 and passthrough plans:
    tile grid, window CSR, work list and the attention workspace."""

    def __init__(self, grid, tile, window, heads: int, d: int, device, pitch: int | None):
        torch = _torch()
        self.grid = tuple(int(x) for x in grid)
        self.tile = tuple(int(x) for x in tile)
        self.window = window if isinstance(window, WindowSpec) else WindowSpec(*window)
        self.heads, self.d = int(heads), int(d)
        out = _lib.Dims3()
        _lib.check(_lib.lib().fpsa_tile_grid(_lib.dims3(self.grid), _lib.dims3(self.tile), out))
        self.tile_dims = (out.t, out.h, out.w)
        self.M = out.t * out.h * out.w
        self.tv = self.tile[0] * self.tile[1] * self.tile[2]
        self.L = self.grid[0] * self.grid[1] * self.grid[2]
        self.pitch = tile_pitch(self.tv) if pitch is None else int(pitch)
        self.mask = build_block_mask(self.window, self.tile_dims)
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        dev = self.device
        self.offs = torch.from_numpy(self.mask.offsets.astype(np.int32)).to(dev)
        self.ids = torch.from_numpy(np.ascontiguousarray(self.mask.ids, dtype=np.int32)).to(dev)
        items = worklist(self.heads, self.mask, self.tv)
        self.n_items = items.size // 3
        self.items = torch.from_numpy(items).to(dev)
        need = ctypes.c_int64(0)
        _lib.check(_lib.lib().fpsa_attn_workspace_bytes(self.n_items, ctypes.byref(need)))
        self.attn_ws = torch.zeros(-(-need.value // 4), dtype=torch.int32, device=dev)

    def _guard(self):
        """Make the plan's device current for a call: its buffers, TMA maps and streams live there."""
        return _torch().cuda.device(self.device)

    # ------------------------------------------------------------------ accounting
    @property
    def density(self) -> float:
        return self.mask.nnz / (self.M * self.M)

    @property
    def flops(self) -> int:
        """Algorithmic FLOPs of one call: heads * sum_u |W(u)| * 4 tv^2 d (metrics.py:91-102)."""
        return self.heads * self.mask.nnz * 4 * self.tv * self.tv * self.d

    def redo_count(self) -> int:
        """Work items the last attention call recomputed in exact mode (synchronises)."""
        return int(self.attn_ws[0].item())

    # ------------------------------------------------------------------ strides
    def _strides(self, x, layout: str):
        if x.device.type != "cuda":
            raise ValueError("inputs must be CUDA tensors")
        if x.stride(-1) != 1:
            raise ValueError("channel dimension must be contiguous")
        if layout == "lhd":
            if tuple(x.shape) != (self.L, self.heads, self.d):
                raise ValueError(f"expected [L, H, d] = {(self.L, self.heads, self.d)}, got {tuple(x.shape)}")
            return x.stride(0), x.stride(1)
        if layout == "hld":
            if tuple(x.shape) != (self.heads, self.L, self.d):
                raise ValueError(f"expected [H, L, d] = {(self.heads, self.L, self.d)}, got {tuple(x.shape)}")
            return x.stride(1), x.stride(0)
        if layout == "ld":
            if self.heads != 1 or tuple(x.shape) != (self.L, self.d):
                raise ValueError(f"expected [L, d] = {(self.L, self.d)}, got {tuple(x.shape)}")
            return x.stride(0), 0
        raise ValueError(f"unknown layout {layout!r}")

    def _out_args(self, out, layout: str, softmax_scale):
        torch = _torch()
        scale = np.float32(1.0 / math.sqrt(self.d)) if softmax_scale is None else np.float32(softmax_scale)
        if not scale > 0:
            raise ValueError("softmax_scale must be > 0")
        ts, hs = self._strides(out, layout)
        odt = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}.get(out.dtype)
        if odt is None:
            raise NotImplementedError(f"output dtype {out.dtype} not supported")
        return float(scale), odt, ts, hs


class FpsaPlan(_TilePlan):
    """Device buffers + launch parameters for one (grid, tile, window, heads, d, fmt).

    Layouts accepted by :meth:`quantize` / :meth:`__call__`:
      ``"lhd"``  [L, H, d]  (one sample of Wan's [B, L, H, d])
      ``"hld"``  [H, L, d]
      ``"ld"``   [L, d]     single head
    in natural (t, h, w) token order, or with ``tile_order=True`` rows already
    tile-contiguous (the reference's convention, fp8sta/attention.py:36-61).
    """

    def __init__(self, grid, tile, window, heads: int, d: int, fmt: Fp8Format = E4M3, *,
                 device="cuda", tau: float = 8.0, pitch: int | None = None, p_mode: str = "onepass"):
        if p_mode not in P_MODES:
            raise ValueError(f"p_mode must be one of {sorted(P_MODES)}, got {p_mode!r}")
        super().__init__(grid, tile, window, heads, d, device, pitch)
        torch = _torch()
        self.fmt, self.tau, self.p_mode = fmt, float(tau), p_mode
        dev = self.device
        rows = self.heads * self.M * self.pitch
        self.q_codes = torch.empty(rows * self.d, dtype=torch.uint8, device=dev)
        self.k_codes = torch.empty_like(self.q_codes)
        self.v_codes = torch.empty_like(self.q_codes)
        self.q_scales = torch.empty(self.heads * self.M, dtype=torch.float64, device=dev)
        self.k_scales = torch.empty_like(self.q_scales)
        self.v_scales = torch.empty(self.heads * self.d, dtype=torch.float64, device=dev)
        ws = ctypes.c_int64(0)
        _lib.check(_lib.lib().fpsa_quantize_workspace_bytes(self.heads, self.d, ctypes.byref(ws)))
        self.workspace = torch.empty(-(-ws.value // 4), dtype=torch.int32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)

    # ------------------------------------------------------------------ kernels
    def quantize(self, q, k, v, layout: str = "lhd", tile_order: bool = False, stream=None) -> None:
        """K1/K2: per-tile Q/K and per-channel V codes into the plan's buffers."""
        with self._guard():
            self._quantize(q, k, v, layout, tile_order, _stream(self.device) if stream is None else stream)

    def _quantize(self, q, k, v, layout, tile_order, st) -> None:
        L = _lib.lib()
        order = _lib.ORDER_TILE if tile_order else _lib.ORDER_NATURAL
        g, t = _lib.dims3(self.grid), _lib.dims3(self.tile)
        f = self.fmt.abi_id
        strides = [self._strides(x, layout) for x in (q, k, v)]
        if strides[0] == strides[1] == strides[2] and q.dtype == k.dtype == v.dtype:
            ts, hs = strides[0]
            _lib.check(L.fpsa_quantize_qkv(
                _ptr(q), _ptr(k), _ptr(v), _dtype_id(q), ts, hs, self.heads, g, t, self.d, self.pitch, order, f,
                _ptr(self.q_codes), _ptr(self.k_codes), _ptr(self.v_codes), _ptr(self.q_scales),
                _ptr(self.k_scales), _ptr(self.v_scales), _ptr(self.workspace), _ptr(self.err), st))
            return
        for x, codes, scales in ((q, self.q_codes, self.q_scales), (k, self.k_codes, self.k_scales)):
            ts, hs = self._strides(x, layout)
            _lib.check(L.fpsa_quantize_qk(_ptr(x), _dtype_id(x), ts, hs, self.heads, g, t, self.d, self.pitch,
                                          order, f, _ptr(codes), _ptr(scales), _ptr(self.err), st))
        ts, hs = self._strides(v, layout)
        _lib.check(L.fpsa_quantize_v(_ptr(v), _dtype_id(v), ts, hs, self.heads, g, t, self.d, self.pitch, order,
                                     f, _ptr(self.v_codes), _ptr(self.v_scales), _ptr(self.workspace),
                                     _ptr(self.err), st))

    def quantize_with_amax(self, q, k, v, q_tile_amax=None, k_tile_amax=None, v_channel_amax=None,
                           layout: str = "lhd", tile_order: bool = False, stream=None) -> None:
        """The upstream-fusion hook (Alg. 1 steps 2-3): like :meth:`quantize`, with the absolute
        maxima supplied by the producer of q, k, v -- f32 CUDA tensors [H, M] (tile order) for q / k,
        [H, d] for v; any may be None.  They must equal the true maxima; the codes are then identical to
        :meth:`quantize`'s, and a supplied v maximum removes the extra read of v."""
        torch = _torch()
        strides = [self._strides(x, layout) for x in (q, k, v)]
        if not (strides[0] == strides[1] == strides[2] and q.dtype == k.dtype == v.dtype):
            raise ValueError("q, k, v must share dtype and strides")

        def amax_arg(t, shape):
            if t is None:
                return None
            if t.dtype != torch.float32 or t.device != self.device or tuple(t.shape) != shape or not t.is_contiguous():
                raise ValueError(f"amax must be a contiguous float32 {shape} tensor on {self.device}")
            return _ptr(t)

        qa = amax_arg(q_tile_amax, (self.heads, self.M))
        ka = amax_arg(k_tile_amax, (self.heads, self.M))
        va = amax_arg(v_channel_amax, (self.heads, self.d))
        ts, hs = strides[0]
        order = _lib.ORDER_TILE if tile_order else _lib.ORDER_NATURAL
        with self._guard():
            st = _stream(self.device) if stream is None else stream
            _lib.check(_lib.lib().fpsa_quantize_qkv_amax(
                _ptr(q), _ptr(k), _ptr(v), _dtype_id(q), ts, hs, self.heads, _lib.dims3(self.grid),
                _lib.dims3(self.tile), self.d, self.pitch, order, self.fmt.abi_id, qa, ka, va, _ptr(self.q_codes),
                _ptr(self.k_codes), _ptr(self.v_codes), _ptr(self.q_scales), _ptr(self.k_scales),
                _ptr(self.v_scales), _ptr(self.workspace), _ptr(self.err), st))

    def attention(self, out, layout: str = "lhd", tile_order: bool = False, softmax_scale: float | None = None,
                  stream=None) -> None:
        """K4 over the quantised buffers; writes `out` (f32 or bf16; f32 in the normalised-P mode)."""
        scale, odt, ts, hs = self._out_args(out, layout, softmax_scale)
        with self._guard():
            st = _stream(self.device) if stream is None else stream
            _lib.check(_lib.lib().fpsa_attn_fwd(
                _ptr(self.q_codes), _ptr(self.k_codes), _ptr(self.v_codes), _ptr(self.q_scales),
                _ptr(self.k_scales), _ptr(self.v_scales), self.heads, _lib.dims3(self.grid), _lib.dims3(self.tile),
                self.d, self.pitch, _ptr(self.offs), _ptr(self.ids), _ptr(self.items), self.n_items, scale,
                self.fmt.abi_id, self.tau, P_MODES[self.p_mode], _ptr(out), odt, ts, hs,
                _lib.ORDER_TILE if tile_order else _lib.ORDER_NATURAL, _ptr(self.attn_ws), self.attn_ws.numel() * 4,
                st))

    def check_finite(self) -> None:
        """Raise ValueError if a quantised input held a non-finite value (synchronises)."""
        if int(self.err.item()) != 0:
            self.err.zero_()
            raise ValueError("non-finite value in quantization input")

    def __call__(self, q, k, v, layout: str = "lhd", out=None, out_dtype=None, tile_order: bool = False,
                 softmax_scale: float | None = None):
        torch = _torch()
        if out is None:
            dt = out_dtype or (q.dtype if q.dtype in (torch.float32, torch.bfloat16) else torch.float32)
            out = torch.empty(q.shape, dtype=dt, device=q.device)
        self.quantize(q, k, v, layout, tile_order)
        self.attention(out, layout, tile_order, softmax_scale)
        return out

class HostStreamer:
    """Quantise + attention of pinned host [L, H, d] tensors with transfers overlapped.

    Heads are processed in chunks: while chunk c is quantised and attended on
    the compute stream, chunk c+1's q, k, v travel host -> device on a copy
    stream and chunk c-1's output device -> host on another (PCIe is full
    duplex), through double-buffered device staging.  Per-head independence
    (scales, windows and outputs are per head) is what makes
    head chunks exact.  Transfers use fpsa_copy2d (strided rows: a chunk is a
    run of heads of every token).  The call is asynchronous with respect to
    the host and ordered on the caller's current stream: synchronising that
    stream makes ``out_host`` complete.
    """

    def __init__(self, grid, tile, window, heads: int, d: int, fmt: Fp8Format = E4M3, *, chunk_heads: int = 2,
                 device="cuda", tau: float = 8.0):
        torch = _torch()
        self.heads, self.d = int(heads), int(d)
        self.chunk = max(1, min(int(chunk_heads), self.heads))
        self.device = torch.device(device)
        sizes = {min(self.chunk, self.heads - h0) for h0 in range(0, self.heads, self.chunk)}
        self.plans = {hc: FpsaPlan(grid, tile, window, hc, d, fmt, device=self.device, tau=tau) for hc in sizes}
        any_plan = next(iter(self.plans.values()))
        self.L = any_plan.L
        shape = (self.L, self.chunk, self.d)
        self.stage_in = [[torch.empty(shape, dtype=torch.bfloat16, device=self.device) for _ in range(3)]
                         for _ in range(2)]
        self.stage_out = [torch.empty(shape, dtype=torch.bfloat16, device=self.device) for _ in range(2)]
        self.s_in = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)

    @property
    def flops(self) -> int:
        p = next(iter(self.plans.values()))
        return p.flops // p.heads * self.heads

    def __call__(self, q_host, k_host, v_host, out_host) -> None:
        with _torch().cuda.device(self.device):
            self._run(q_host, k_host, v_host, out_host)

    def _run(self, q_host, k_host, v_host, out_host) -> None:
        torch = _torch()
        for x in (q_host, k_host, v_host, out_host):
            if x.device.type != "cpu" or not x.is_pinned() or not x.is_contiguous() or x.dtype != torch.bfloat16:
                raise ValueError("host tensors must be pinned, contiguous bf16")
            if tuple(x.shape) != (self.L, self.heads, self.d):
                raise ValueError(f"expected [L, H, d] = {(self.L, self.heads, self.d)}, got {tuple(x.shape)}")
        L = _lib.lib()
        comp = torch.cuda.current_stream(self.device)
        row = self.heads * self.d * 2  # host pitch (bytes)
        ev_in_ready = [torch.cuda.Event() for _ in range(2)]
        ev_in_free = [torch.cuda.Event() for _ in range(2)]
        ev_out_ready = [torch.cuda.Event() for _ in range(2)]
        ev_out_free = [torch.cuda.Event() for _ in range(2)]
        start = torch.cuda.Event()
        start.record(comp)
        self.s_in.wait_event(start)
        self.s_out.wait_event(start)
        for c, h0 in enumerate(range(0, self.heads, self.chunk)):
            b, hc = c % 2, min(self.chunk, self.heads - h0)
            plan = self.plans[hc]
            width = hc * self.d * 2
            dpitch = self.chunk * self.d * 2
            if c >= 2:
                self.s_in.wait_event(ev_in_free[b])
            for src, dst in zip((q_host, k_host, v_host), self.stage_in[b]):
                _lib.check(L.fpsa_copy2d(_ptr(dst), dpitch, src.data_ptr() + h0 * self.d * 2, row, width, self.L,
                                         self.s_in.cuda_stream))
            ev_in_ready[b].record(self.s_in)
            comp.wait_event(ev_in_ready[b])
            qd, kd, vd = (t[:, :hc] for t in self.stage_in[b])
            plan.quantize(qd, kd, vd, "lhd", stream=comp.cuda_stream)
            ev_in_free[b].record(comp)
            if c >= 2:
                comp.wait_event(ev_out_free[b])
            od = self.stage_out[b][:, :hc]
            plan.attention(od, "lhd", stream=comp.cuda_stream)
            ev_out_ready[b].record(comp)
            self.s_out.wait_event(ev_out_ready[b])
            _lib.check(L.fpsa_copy2d(out_host.data_ptr() + h0 * self.d * 2, row, _ptr(od), dpitch, width, self.L,
                                     self.s_out.cuda_stream))
            ev_out_free[b].record(self.s_out)
        done = torch.cuda.Event()
        done.record(self.s_out)
        comp.wait_event(done)
        # the staging buffers are reused by the next call: make the copy streams wait for this call's compute
        done_c = torch.cuda.Event()
        done_c.record(comp)
        self.s_in.wait_event(done_c)


class PassthroughPlan(_TilePlan):
    """Full-precision sliding-tile sparse attention (the reference's passthrough /
    sparse_reference, fp8sta/attention.py:152-154, :165-176, :192-194) on bf16
    operands: :meth:`gather` lays q, k, v out tile-major in bf16, :meth:`attention`
    runs the tcgen05 kind::f16 kernel.  Same layouts and work list as FpsaPlan."""

    def __init__(self, grid, tile, window, heads: int, d: int, *, device="cuda", pitch: int | None = None):
        super().__init__(grid, tile, window, heads, d, device, pitch)
        torch = _torch()
        rows = self.heads * self.M * self.pitch
        self.q_tiles = torch.empty((rows, self.d), dtype=torch.bfloat16, device=self.device)
        self.k_tiles = torch.empty_like(self.q_tiles)
        self.v_tiles = torch.empty_like(self.q_tiles)

    def gather(self, q, k, v, layout: str = "lhd", tile_order: bool = False, stream=None) -> None:
        """q, k, v -> tile-major padded bf16 (f32 inputs rounded to nearest even)."""
        L = _lib.lib()
        order = _lib.ORDER_TILE if tile_order else _lib.ORDER_NATURAL
        g, t = _lib.dims3(self.grid), _lib.dims3(self.tile)
        with self._guard():
            st = _stream(self.device) if stream is None else stream
            for x, dst in ((q, self.q_tiles), (k, self.k_tiles), (v, self.v_tiles)):
                ts, hs = self._strides(x, layout)
                _lib.check(L.fpsa_tile_gather_bf16(_ptr(x), _dtype_id(x), ts, hs, self.heads, g, t, self.d,
                                                   self.pitch, order, _ptr(dst), st))

    def attention(self, out, layout: str = "lhd", tile_order: bool = False, softmax_scale: float | None = None,
                  stream=None) -> None:
        """Passthrough attention over the gathered tiles; writes `out` (f32 or bf16)."""
        scale, odt, ts, hs = self._out_args(out, layout, softmax_scale)
        with self._guard():
            st = _stream(self.device) if stream is None else stream
            _lib.check(_lib.lib().fpsa_attn_bf16_fwd(
                _ptr(self.q_tiles), _ptr(self.k_tiles), _ptr(self.v_tiles), self.heads, _lib.dims3(self.grid),
                _lib.dims3(self.tile), self.d, self.pitch, _ptr(self.offs), _ptr(self.ids), _ptr(self.items),
                self.n_items, scale, _ptr(out), odt, ts, hs, _lib.ORDER_TILE if tile_order else _lib.ORDER_NATURAL,
                _ptr(self.attn_ws), self.attn_ws.numel() * 4, st))

    def __call__(self, q, k, v, layout: str = "lhd", out=None, out_dtype=None, tile_order: bool = False,
                 softmax_scale: float | None = None):
        torch = _torch()
        if out is None:
            dt = out_dtype or (q.dtype if q.dtype in (torch.float32, torch.bfloat16) else torch.float32)
            out = torch.empty(q.shape, dtype=dt, device=q.device)
        self.gather(q, k, v, layout, tile_order)
        self.attention(out, layout, tile_order, softmax_scale)
        return out


def device_fidelity(ref, approx, layout: str = "lhd", stream=None) -> list[tuple[float, float, float]]:
    """Per-head (cosine, mse, snr_db) of `approx` against `ref`.

    [L, H, d] / [H, L, d] / [L, d] CUDA tensors, f32 or bf16, same shape and
    strides; reduced on the device (fpsa_fidelity) and finished like
    fp8sta/metrics.py:41-88.  Synchronises.
    """
    torch = _torch()
    if tuple(ref.shape) != tuple(approx.shape) or ref.stride() != approx.stride():
        raise ValueError("ref and approx must have the same shape and strides")
    if ref.stride(-1) != 1:
        raise ValueError("channel dimension must be contiguous")
    if layout == "lhd":
        tokens, heads, d = ref.shape
        ts, hs = ref.stride(0), ref.stride(1)
    elif layout == "hld":
        heads, tokens, d = ref.shape
        ts, hs = ref.stride(1), ref.stride(0)
    elif layout == "ld":
        (tokens, d), heads = ref.shape, 1
        ts, hs = ref.stride(0), 0
    else:
        raise ValueError(f"unknown layout {layout!r}")
    sums = torch.empty((heads, 6), dtype=torch.float64, device=ref.device)
    with torch.cuda.device(ref.device):
        st = _stream(ref.device) if stream is None else stream
        _lib.check(_lib.lib().fpsa_fidelity(_ptr(ref), _dtype_id(ref), _ptr(approx), _dtype_id(approx), tokens, heads,
                                            d, ts, hs, _ptr(sums), st))
    from .metrics import fidelity_from_sums

    return [fidelity_from_sums(*row, n=tokens * d) for row in sums.cpu().tolist()]


_PLANS: dict = {}
_PLANS_MAX = 8  # cached plans (each holds the code buffers of its shape); the least recently used is dropped


def cache_get(cache: dict, key, make, limit: int = _PLANS_MAX):
    """LRU lookup shared by the plan caches of fps_attention and fp8_sparse_forward."""
    plan = cache.pop(key, None)
    if plan is None:
        plan = make()
        while len(cache) >= limit:
            cache.pop(next(iter(cache)))
    cache[key] = plan  # most recent last
    return plan


def fps_attention(q, k, v, grid, tile, window, *, fmt: Fp8Format = E4M3, softmax_scale: float | None = None,
                  layout: str = "blhd", out_dtype=None, tau: float = 8.0):
    """Joint tile-wise FP8 quantisation + sliding-tile sparse attention, natural token order.

    q, k, v: [B, L, H, d] (``layout="blhd"``, Wan / HunyuanVideo convention)
    or [L, H, d] (``"lhd"``), bf16 or f32 CUDA tensors.  Returns the same
    shape in ``out_dtype`` (default: input dtype).
    """
    batched = layout == "blhd"
    if batched:
        B, L, H, d = q.shape
    elif layout == "lhd":
        B, (L, H, d) = 1, q.shape
    else:
        raise ValueError(f"unknown layout {layout!r}")
    win = window if isinstance(window, WindowSpec) else WindowSpec(*window)
    torch = _torch()
    # one plan (code buffers + workspace) per device, stream and thread: calls that could overlap never share
    # buffers, calls on one stream are ordered by it
    stream = torch.cuda.current_stream(q.device)
    key = (tuple(grid), tuple(tile), win.dims, H, d, fmt.name, str(q.device), tau, stream.cuda_stream,
           threading.get_ident())
    plan = cache_get(_PLANS, key, lambda: FpsaPlan(grid, tile, win, H, d, fmt, device=q.device, tau=tau))
    out = torch.empty(q.shape, dtype=out_dtype or q.dtype, device=q.device)
    for b in range(B):
        sl = (lambda x: x[b]) if batched else (lambda x: x)
        plan.quantize(sl(q), sl(k), sl(v), "lhd")
        plan.attention(sl(out), "lhd", softmax_scale=softmax_scale)
    return out
