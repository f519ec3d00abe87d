"""Which resource bounds the tcgen05 GEMM?  Times the plain-FP8 and MXFP8 kernels on C2/C4 shapes with
pipeline-isolation knobs (gemm_debug: 0 normal, 1 no epilogue stores, 256 no operand loads -- stages
complete on arrivals, MMAs read stale smem -- 257 both; results invalid for the debug modes) and samples
the SM clock during each run, reporting flop per clock per SM.  If removing the operand loads raises
flop/clk/SM a lot, the mainloop is bound by L2 -> SMEM operand bandwidth, not by the tensor pipe.
    python tools/gemm_bound_probe.py"""

import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops  # noqa: E402

SHAPES = [tuple(int(v) for v in s.split("x")) for s in
          os.environ.get("PROBE_SHAPES", "16384x14336x4096,16384x4096x14336,16384x28672x8192").split(",")]
MODES = [int(m) for m in os.environ.get("PROBE_MODES", "0,1,256,257").split(",")]
KNOBS = [kv.split("=") for kv in os.environ.get("PROBE_KNOBS", "").split(",") if kv]   # e.g. gemm_n512=1
KINDS = os.environ.get("PROBE_KINDS", "fp8,mx").split(",")


class Clock:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.s, self.stop = [], threading.Event()

    def run(self):
        while not self.stop.is_set():
            self.s.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            time.sleep(0.002)

    def __enter__(self):
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *e):
        self.stop.set()
        self.t.join()

    def median(self):
        s = sorted(self.s)
        return s[len(s) // 2] if s else float("nan")


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clock() as c:
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
    return a.elapsed_time(b) / iters, c.median()


def main():
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for M, N, K in SHAPES:
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.randint(0, 0x70, (M, K), dtype=torch.uint8, device="cuda", generator=g)
        B = torch.randint(0, 0x70, (N, K), dtype=torch.uint8, device="cuda", generator=g)
        s = torch.ones(1, device="cuda")
        sfa = torch.full((M * K // 32,), 127, dtype=torch.uint8, device="cuda")
        sfb = torch.full((N * K // 32,), 127, dtype=torch.uint8, device="cuda")
        flops = 2.0 * M * N * K
        iters = max(5, int(2e13 / flops))
        for kind in KINDS:
            for mode in MODES:
                for k, v in KNOBS:
                    ops.set_knob(k, int(v))
                ops.set_knob("gemm_debug", mode)
                if kind == "fp8":
                    fn = lambda: ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor")  # noqa: E731
                else:
                    fn = lambda: ops.gemm(A, "e4m3", sfa, B, "e4m3", sfb, "mx32")  # noqa: E731
                ms, mhz = timeit(fn, iters)
                ops.reset_knobs()
                tf = flops / ms / 1e9
                print(json.dumps({"shape": [M, N, K], "kind": kind, "debug": mode, "ms": round(ms, 4),
                                  "tflops": round(tf), "sm_mhz": mhz,
                                  "flop_per_clk_sm": round(tf * 1e12 / (mhz * 1e6) / nsm)}), flush=True)
        del A, B, sfa, sfb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
