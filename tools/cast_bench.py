"""Microbenchmark of the memory-bound kernels on C2-sized tensors (context for tuning)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops


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


dy = torch.randn((16384, 14336), device="cuda", dtype=torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for cfg in ("44", "48", "4C", "4G", "84", "88", "8C", "28", "2G"):
    ops.set_knob("amax_blocks_per_sm", int(cfg[0]))
    ops.set_knob("amax_loads", {"4": 4, "8": 8, "C": 12, "G": 16}[cfg[1]])
    def f():
        flush.zero_()
        ops.amax(dy)
    t_flush = timeit(lambda: flush.zero_())
    ms = timeit(f) - t_flush
    res[cfg] = round(dy.numel() * 2 / ms / 1e6)
print(json.dumps({"amax_flat_GBps": res}))
ops.reset_knobs()
ms = timeit(lambda: (flush.zero_(), ops.cast(dy, "e5m2", "tensor"))) - timeit(lambda: flush.zero_())
print(json.dumps({"amax+cast tensorwise GB/s (alg 5 B/elem)": round(dy.numel() * 5 / ms / 1e6)}))
# reference read bandwidth: torch reductions / copy on the same tensor
ms = timeit(lambda: (flush.zero_(), torch.amax(dy))) - timeit(lambda: flush.zero_())
print(json.dumps({"torch.amax GB/s": round(dy.numel() * 2 / ms / 1e6)}))
ms = timeit(lambda: (flush.zero_(), dy.float().sum() if False else dy.sum())) - timeit(lambda: flush.zero_())
print(json.dumps({"torch.sum GB/s": round(dy.numel() * 2 / ms / 1e6)}))
out = torch.empty_like(dy)
ms = timeit(lambda: (flush.zero_(), out.copy_(dy))) - timeit(lambda: flush.zero_())
print(json.dumps({"copy GB/s (r+w)": round(dy.numel() * 4 / ms / 1e6)}))
