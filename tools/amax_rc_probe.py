"""A/B probe of the row / column amax kernel (amax_rc_kernel) on one large bf16 tensor (larger than L2, no
flush): read rate with the consumers skipping the tile (knob amax_rc_debug bit 0: TMA stream alone, results
invalid), with interleaved tile order (bit 1), both, and the product kernel; the tensorwise bulk amax and a
torch read+write copy for scale.  Tuning context only.

    python tools/amax_rc_probe.py [R] [C]
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import _lib as L  # noqa: E402
from paper_2507_16099_b200 import ops  # noqa: E402


def timeit(fn, iters=30):
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


R = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
C = int(sys.argv[2]) if len(sys.argv) > 2 else 14336
x = torch.randn((R, C), device="cuda", dtype=torch.bfloat16)
h = ops.hp(x)
out = torch.empty(R + C, dtype=torch.float32, device="cuda")
ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
nb = R * C * 2
res = {"R": R, "C": C}
for gran, gi in (("row", L.GRAN_ROW), ("col", L.GRAN_COL), ("tensor", L.GRAN_TENSOR)):
    for dbg in ((0, 1, 4) if gran != "tensor" else (0,)):
        ops.reset_knobs()
        if dbg == 4:   # the product kernel with sleeping barrier waits (knob wait_sleep bit 0)
            ops.set_knob("wait_sleep", 1)
        else:
            ops.set_knob("amax_rc_debug", dbg)

        def f():
            L.check(L.lib.fp8_amax(h, gi, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                   ws.numel(), ops._stream()), "amax")
        res[f"{gran}_dbg{dbg}_TBps"] = round(nb / timeit(f) / 1e9, 3)
ops.reset_knobs()
y = torch.empty_like(x)
res["torch_copy_rw_TBps"] = round(2 * nb / timeit(lambda: y.copy_(x)) / 1e9, 3)
print(json.dumps(res), flush=True)
