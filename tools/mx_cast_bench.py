"""Microbenchmark of the MXFP8 dim0+dim1 cast on the C4 operand shapes (context for tuning).

Compares the TMA-pipelined persistent kernel (default) with the register-only kernel
(knob mx_cast_tma = 0), for the row-major dim1 layout (MX32_RM, the linear's default) and the
transposed one (MX32).  GB/s = algorithmic bytes (2 read + 1 + 1 written + 2/32 scales per
element) / time; inputs are larger than L2 and a 512 MiB buffer is rewritten between calls.
"""
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


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    t_flush = timeit(lambda: flush.zero_())
    res = []
    for R, C in ((16384, 28672), (16384, 8192), (28672, 8192)):
        x = torch.randn((R, C), device="cuda", dtype=torch.bfloat16)
        q0 = torch.empty((R, C), dtype=torch.uint8, device="cuda")
        q1 = torch.empty((R, C), dtype=torch.uint8, device="cuda")
        s0 = torch.empty(R * C // 32, dtype=torch.uint8, device="cuda")
        s1 = torch.empty(R * C // 32, dtype=torch.uint8, device="cuda")
        alg = R * C * (4 + 2 / 32)
        for gran in ("mx32_rm", "mx32"):
            t8 = L.Tensor8(q0.data_ptr(), q1.data_ptr(), s0.data_ptr(), s1.data_ptr(), None, None,
                           L.E5M2, ops.GRANS[gran], R, C)
            h = ops.hp(x)

            def f():
                flush.zero_()
                L.check(L.lib.fp8_cast_scaled(h, L.MX_FLOOR, None, ctypes.byref(t8), None, 0,
                                              ops._stream()), "cast")
            row = {"R": R, "C": C, "gran": gran}
            for impl in ("1", "0"):
                ops.set_knob("mx_cast_tma", int(impl))
                ms = timeit(f) - t_flush
                row["tma" if impl == "1" else "regs"] = {"ms": round(ms, 4), "GBps": round(alg / ms / 1e6)}
            ops.reset_knobs()
            res.append(row)
            print(json.dumps(row), flush=True)
        del x, q0, q1, s0, s1
    return res


if __name__ == "__main__":
    main()
