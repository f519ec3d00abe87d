"""Energy per flop of the GEMM under the 1 kW cap: each variant runs back to back for ~2 s while NVML samples
SM clock and board power; reports sustained TFLOP/s, median clock, median power and pJ per flop.  The
gemm_debug variants (results invalid) remove the operand loads (256) or the epilogue stores (1), which
shows how much of the power budget data movement takes.
    ENERGY_SHAPE=16384x28672x8192 ENERGY_KIND=mx python tools/energy_probe.py"""
import json
import os
import sys
import threading
import time

import torch
import pynvml

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops  # noqa: E402

M, N, K = (int(v) for v in os.environ.get("ENERGY_SHAPE", "16384x28672x8192").split("x"))
KIND = os.environ.get("ENERGY_KIND", "mx")
MODES = [int(m) for m in os.environ.get("ENERGY_MODES", "0,256,1,257").split(",")]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randint(0, 0x70, (M, K), dtype=torch.uint8, device="cuda", generator=g)
B = torch.randint(0, 0x70, (N, K), dtype=torch.uint8, device="cuda", generator=g)
s = torch.ones(1, device="cuda")
sfa = torch.full((M * K // 32,), 127, dtype=torch.uint8, device="cuda")
sfb = torch.full((N * K // 32,), 127, dtype=torch.uint8, device="cuda")
fn = (lambda: ops.gemm(A, "e4m3", sfa, B, "e4m3", sfb, "mx32")) if KIND == "mx" else \
    (lambda: ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor"))
flops = 2.0 * M * N * K
for mode in MODES:
    ops.set_knob("gemm_debug", mode)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.time()
    while time.time() - t0 < 0.5:   # reach the power-capped steady state first
        fn()
        torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.005)

    th = threading.Thread(target=sample)
    th.start()
    n = max(20, int(2.0 / (flops / 2.5e15)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    clk = sorted(c for c, _ in samples)[len(samples) // 2]
    pw = sorted(p for _, p in samples)[len(samples) // 2]
    tf = flops / ms / 1e9
    print(json.dumps({"shape": [M, N, K], "kind": KIND, "debug": mode, "ms": round(ms, 4), "tflops": round(tf),
                      "sm_mhz": clk, "power_w": round(pw), "pj_per_flop": round(pw / (tf * 1e12) * 1e12, 4),
                      "flop_per_clk_sm": round(tf * 1e12 / (clk * 1e6) / 148)}), flush=True)
ops.reset_knobs()
