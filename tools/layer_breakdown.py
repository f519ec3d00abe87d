"""Per-launch device times of one c3 (7-linear layer) step, in-step (not serialised like ncu): which
amax / cast / GEMM launches lose time against their algorithmic bytes or flops.  Tuning context only.

    python tools/layer_breakdown.py [config] [steps]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_16099_b200 import _lib as L, ops  # noqa: E402

KIND = {0: "amax", 1: "cast", 2: "mx_cast", 3: "transpose", 4: "gemm_fp8", 5: "gemm_mx", 6: "gemm_bf16", 7: "p2p"}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cfg = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    M = cfg["M"]
    units = []
    for i, (nm, N, K) in enumerate(cfg["linears"]):
        x, w, dy = bench.make_inputs(dict(cfg, N=N, K=K), M, N, K, 0, 1, dev, seed=i)
        plan = ops.LinearPlan(M, N, K, recipe=cfg["recipe"], out_dtype=torch.bfloat16, device=dev)
        units.append(dict(name=nm, N=N, K=K, x=x, w=w, dy=dy, plan=plan, saved=plan.new_saved(dev),
                          y=torch.empty((M, N), dtype=torch.bfloat16, device=dev),
                          dx=torch.empty((M, K), dtype=torch.bfloat16, device=dev),
                          dw=torch.empty((N, K), dtype=torch.bfloat16, device=dev)))

    def step():
        for u in units:
            u["plan"].forward(u["x"], u["w"], u["saved"], y=u["y"])
            u["plan"].backward(u["dy"], u["saved"], dx=u["dx"], dw=u["dw"], x=u["x"])

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    L.lib.fp8_profile_collect(None, None, 0)
    L.lib.fp8_profile_enable(1)
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    L.lib.fp8_profile_enable(0)
    cap = 4096
    kinds, durs = (ctypes.c_int * cap)(), (ctypes.c_float * cap)()
    n = L.lib.fp8_profile_collect(kinds, durs, cap)
    per = n // steps
    acc = [0.0] * per
    for i in range(n):
        acc[i % per] += durs[i] / steps
    print(f"{name}: {per} launches per step, sum {sum(acc):.3f} ms")
    # algorithmic bytes / flops per launch (rowwise: fwd amax X+W, fwd cast X+W (read 2 + two 1-B copies),
    # GEMM, bwd amax dY, bwd cast dY, GEMM (dX + dW))
    work = []
    for u in units:
        N, K = u["N"], u["K"]
        xw = M * K + N * K
        work += [("amax X,W", 2 * xw, "B"), ("cast X,W", 4 * xw, "B"), ("gemm fwd", 2 * M * N * K, "F"),
                 ("amax dY", 2 * M * N, "B"), ("cast dY", 4 * M * N, "B"), ("gemm bwd", 4 * M * N * K, "F")]
    for i in range(per):
        lab, w, kind = work[i] if per == len(work) else ("", 0, "B")
        rate = (f"{w / (acc[i] * 1e-3) / 1e9:8.0f} GB/s" if kind == "B" else f"{w / (acc[i] * 1e-3) / 1e12:8.0f} TF/s") \
            if w else ""
        print(f"  {i:3d} {KIND.get(kinds[i], kinds[i]):10s} {acc[i] * 1e3:9.1f} us  {units[i // 6]['name'] if per == len(work) else '':4s}"
              f" {lab:9s} {rate}")


if __name__ == "__main__":
    main()
