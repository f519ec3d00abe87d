"""How much of a bench step is launch overhead: the same step timed eagerly (with and without the
per-launch profiling events) and as a CUDA-graph replay.  Context for tuning; not part of the contract.

    python tools/graph_probe.py c3 [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_16099_b200 import _lib as L, ops  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    M = cfg["M"]
    lin = cfg.get("linears") or [("w", cfg["N"], cfg["K"])]
    units = []
    for i, (nm, N, K) in enumerate(lin):
        x, w, dy = bench.make_inputs(dict(cfg, N=N, K=K), M, N, K, 0, 1, dev, seed=i)
        plan = ops.LinearPlan(M, N, K, recipe=cfg["recipe"], out_dtype=torch.bfloat16, device=dev)
        units.append(dict(x=x, w=w, dy=dy, plan=plan, saved=plan.new_saved(dev),
                          y=torch.empty((M, N), dtype=torch.bfloat16, device=dev),
                          dx=torch.empty((M, K), dtype=torch.bfloat16, device=dev),
                          dw=torch.empty((N, K), dtype=torch.bfloat16, device=dev)))

    def step():
        for u in units:
            u["plan"].forward(u["x"], u["w"], u["saved"], y=u["y"])
            u["plan"].backward(u["dy"], u["saved"], dx=u["dx"], dw=u["dw"], x=u["x"])

    def timed(fn, n):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    res = {"eager_ms": [], "eager_profiled_ms": [], "graph_ms": []}
    for _ in range(4):   # alternate, so clock / power drift does not bias any variant
        L.lib.fp8_profile_enable(1)
        res["eager_profiled_ms"].append(round(timed(step, steps), 4))
        L.lib.fp8_profile_enable(0)
        L.lib.fp8_profile_collect(None, None, 0)
        res["eager_ms"].append(round(timed(step, steps), 4))
        res["graph_ms"].append(round(timed(g.replay, steps), 4))
    print({"config": name, **res})


if __name__ == "__main__":
    main()
