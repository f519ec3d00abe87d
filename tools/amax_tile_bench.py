"""Microbenchmark of the per-row / per-column amax pass (rowwise recipe) on C2/C3-sized tensors:
multi-tensor warp-specialised kernel (default, knob amax_rc = 1), the TMA-ring strip kernel (amax_rc = 0) and
the register-only kernel (amax_rc = 0, amax_tile_tma = 0).  GB/s = 2 B read per
element / time, a 512 MiB buffer rewritten between calls (context for tuning)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import _lib as L  # noqa: E402
from paper_2507_16099_b200 import ops  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


IMPLS = {"rc": {"amax_rc": 1}, "tma": {"amax_rc": 0}, "regs": {"amax_rc": 0, "amax_tile_tma": 0}}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
t_flush = timeit(lambda: flush.zero_())
for R, C in ((16384, 14336), (16384, 4096), (14336, 4096)):
    x = torch.randn((R, C), device="cuda", dtype=torch.bfloat16)
    h = ops.hp(x)
    out = torch.empty(R + C, dtype=torch.float32, device="cuda")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    row = {"R": R, "C": C}
    for gran, gi in (("row", L.GRAN_ROW), ("col", L.GRAN_COL), ("row_col", L.GRAN_ROW_COL)):
        if gran == "row_col":   # the rowwise recipe's dual amax through the cast entry (amax only timed via cast)
            continue
        for impl, kn in IMPLS.items():
            ops.reset_knobs()
            for k, v in kn.items():
                ops.set_knob(k, v)

            def f():
                flush.zero_()
                L.check(L.lib.fp8_amax(h, gi, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                       ws.numel(), ops._stream()), "amax")
            ms = timeit(f) - t_flush
            row[f"{gran}_{impl}_GBps"] = round(R * C * 2 / ms / 1e6)
    ops.reset_knobs()
    # dual row+col amax + dual cast (the rowwise recipe's X pass), end to end through fp8_cast_scaled
    for impl, kn in IMPLS.items():
        ops.reset_knobs()
        for k, v in kn.items():
            ops.set_knob(k, v)
        ms = timeit(lambda: (flush.zero_(), ops.cast(x, "e4m3", "row_col", want_q=True, want_qt=True))) - t_flush
        row[f"rowcol_amax+cast_{impl}_GBps"] = round(R * C * 6 / ms / 1e6)
    ops.reset_knobs()
    print(json.dumps(row), flush=True)
