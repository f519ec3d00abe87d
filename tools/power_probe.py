"""Run the C2 forward GEMM back to back for ~2 s while sampling NVML SM clock / power / throttle
reasons every 5 ms: tells whether the GEMM is power-capped."""
import json, os, sys, threading, time
import torch
import pynvml
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
M, N, K = 16384, 14336, 4096
A = torch.randint(0, 0x70, (M, K), dtype=torch.uint8, device="cuda")
B = torch.randint(0, 0x70, (N, K), dtype=torch.uint8, device="cuda")
s = torch.ones(1, device="cuda")
for _ in range(5):
    ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor")
torch.cuda.synchronize()
samples = []
stop = threading.Event()


def sample():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.005)


t = threading.Thread(target=sample)
t.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 3000
e0.record()
for _ in range(n):
    ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor")
e1.record()
torch.cuda.synchronize()
stop.set()
t.join()
ms = e0.elapsed_time(e1) / n
clk = sorted(x[0] for x in samples)
pw = sorted(x[1] for x in samples)
reasons = 0
for x in samples:
    reasons |= x[2]
print(json.dumps({"tflops": 2 * M * N * K / ms / 1e9, "ms": ms, "n_samples": len(samples),
                  "sm_mhz_p10_p50_p90": [clk[len(clk) // 10], clk[len(clk) // 2], clk[9 * len(clk) // 10]],
                  "power_w_p10_p50_p90": [pw[len(pw) // 10], pw[len(pw) // 2], pw[9 * len(pw) // 10]],
                  "throttle_reasons_or": hex(reasons)}))
