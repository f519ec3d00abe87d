"""A/B probe of the MXFP8 dim0 + dim1 TMA cast on the c4 dY shape (larger than L2, no flush): the product
kernel (the TMA ring), the warp-specialised kernel (mx_cast_ws = 1), the ring kernel without its code stores
(knob mx_cast_debug = 1: results invalid), the occupancy-3 variant, dim0 only and dim1 only.  Rate = algorithmic bytes (2 read + 1 + 1 written + 2/32 scales per element for dim0 +
dim1) / time.  Tuning context only.

    python tools/mx_cast_probe.py [R] [C]
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
C = int(sys.argv[2]) if len(sys.argv) > 2 else 28672
x = torch.randn((R, C), device="cuda", dtype=torch.bfloat16)
q0 = torch.empty((R, C), dtype=torch.uint8, device="cuda")
q1 = torch.empty((R, C), dtype=torch.uint8, device="cuda")
s0 = torch.empty(R * C // 32, dtype=torch.uint8, device="cuda")
s1 = torch.empty(R * C // 32, dtype=torch.uint8, device="cuda")
h = ops.hp(x)
res = {"R": R, "C": C}
for name, kn, a0, a1 in (("default", {}, True, True), ("sleep", {"wait_sleep": 1}, True, True),
                         ("ws", {"mx_cast_ws": 1}, True, True),
                         ("tstore", {"mx_cast_tstore": 1}, True, True),
                         ("ring_nostores", {"mx_cast_debug": 1}, True, True),
                         ("occ3", {"mx_cast_occ3": 1}, True, True), ("dim0_only", {}, True, False),
                         ("dim1_only", {}, False, True)):
    ops.reset_knobs()
    for k, v in kn.items():
        ops.set_knob(k, v)
    t8 = L.Tensor8(q0.data_ptr() if a0 else None, q1.data_ptr() if a1 else None, s0.data_ptr() if a0 else None,
                   s1.data_ptr() if a1 else None, None, None, L.E5M2, ops.GRANS["mx32_rm"], R, C)

    def f():
        L.check(L.lib.fp8_cast_scaled(h, L.MX_FLOOR, None, ctypes.byref(t8), None, 0, ops._stream()), "cast")
    ms = timeit(f)
    alg = R * C * (2 + (1 + 1 / 32) * (int(a0) + int(a1)))
    res[name + "_TBps"] = round(alg / ms / 1e9, 3)
ops.reset_knobs()
print(json.dumps(res), flush=True)
