"""Per-tile timeline of the TMA quantiser (CTA 0) from a -DFPSA_QTRACE build: FPSA_LIB=libfpsa_qtrace.so."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04648_b200 as F  # noqa: E402
from paper_2506_04648_b200 import _lib as L  # noqa: E402

grid, tile, H, d = (21, 45, 80), (3, 5, 16), 40, 128
Lt = grid[0] * grid[1] * grid[2]
xs = [torch.randn((Lt, H, d), device="cuda").to(torch.bfloat16) for _ in range(3)]
plan = F.FpsaPlan(grid, tile, (5, 5, 3), H, d)
va = xs[2].float().abs().amax(dim=0).contiguous()
for _ in range(3):
    plan.quantize_with_amax(*xs, None, None, va, layout="lhd") if "--amax" in sys.argv else plan.quantize(*xs, "lhd")
torch.cuda.synchronize()
lib = L.lib()
buf = (ctypes.c_longlong * (128 * 5))()
lib.fpsa_qtrace_timeline.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
lib.fpsa_qtrace_timeline(buf)
cnt = (ctypes.c_ulonglong * 4)()
if hasattr(lib, "fpsa_qtrace_counts"):
    lib.fpsa_qtrace_counts(cnt)
    n_tiles = max(1, cnt[2])
    print(f"fix-up loop: {cnt[0] / n_tiles / 24:.2f} trips per warp-tile, {cnt[1] / n_tiles:.1f} ambiguous bytes per tile "
          f"({cnt[1] / n_tiles / (240 * 128) * 100:.3f} % of elements), over {cnt[2]} tiles")
T = np.array(buf, dtype=np.int64).reshape(128, 5)
T = T[(T > 0).all(1)]
t0 = T[0, 0]
print("tile | issue full(w0) barrier(w0) done(w0) done(w23)   (clk rel. to tile 0 issue)")
for k in range(min(40, len(T))):
    print(f"{k:3d} | " + " ".join(f"{x - t0:8d}" for x in T[k]))
S = T[4:]
print(f"mean over tiles 4..: load latency {np.mean(S[:, 1] - S[:, 0]):.0f}, full->barrier {np.mean(S[:, 2] - S[:, 1]):.0f}, "
      f"barrier->w0 done {np.mean(S[:, 3] - S[:, 2]):.0f}, w23 done - w0 done {np.mean(S[:, 4] - S[:, 3]):.0f}, "
      f"issue spacing {np.mean(np.diff(T[:, 0])):.0f}, full spacing {np.mean(np.diff(T[:, 1])):.0f}")
