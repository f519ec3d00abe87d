"""Per-launch device times of one c3 (7-linear layer) step, in-step (not serialised like ncu): which
amax / cast / GEMM launches lose time against their algorithmic bytes or flops.  Tuning context only.

    python tools/layer_breakdown.py [config] [steps] [--separate] [--knob=name=value ...]
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
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "c3"
    steps = int(args[1]) if len(args) > 1 else 10
    cfg = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    M = cfg["M"]
    shared = "--separate" not in sys.argv
    for a in sys.argv[1:]:
        if a.startswith("--knob="):
            k, v = a[len("--knob="):].split("=")
            ops.set_knob(k, int(v))
    units = []
    for i, (nm, N, K) in enumerate(cfg["linears"]):
        x, w, dy = bench.make_inputs(dict(cfg, N=N, K=K), M, N, K, 0, 1, dev, seed=i)
        units.append(dict(name=nm, N=N, K=K, x=x, w=w, dy=dy,
                          y=torch.empty((M, N), dtype=torch.bfloat16, device=dev),
                          dx=torch.empty((M, K), dtype=torch.bfloat16, device=dev),
                          dw=torch.empty((N, K), dtype=torch.bfloat16, device=dev)))
    # shared-input groups as in bench.run_layer (--separate: every linear on its own)
    byname = {u["name"]: u for u in units}
    groups = [[byname[n] for n in g] for g in cfg.get("shared", [])] if shared else []
    grouped = {id(u) for g in groups for u in g}
    groups += [[u] for u in units if id(u) not in grouped]
    groups.sort(key=lambda g: units.index(g[0]))
    batched = cfg["recipe"] == "rowwise" and ops.get_knob("group_batch") == 1
    work = []   # (label, algorithmic bytes or flops, "B" / "F") per launch, in launch order
    for g in groups:
        K = g[0]["K"]
        for u in g[1:]:
            u["x"] = g[0]["x"]
        names = "/".join(u["name"] for u in g)
        if len(g) == 1:
            u = g[0]
            u["plan"] = ops.LinearPlan(M, u["N"], K, recipe=cfg["recipe"], out_dtype=torch.bfloat16, device=dev)
            u["saved"] = u["plan"].new_saved(dev)
        else:
            sp = ops.SharedInputPlan(M, [u["N"] for u in g], K, recipe=cfg["recipe"], out_dtype=torch.bfloat16,
                                     device=dev)
            for u, t in zip(g, sp.new_saved(dev)):
                u["saved"] = t
            g[0]["group_plan"] = sp
        # amax: read 2 B / element; cast: read 2 + two 1-B copies
        if batched and len(g) > 1:   # rowwise group: one amax + one cast launch over X and every W_i / dY_i
            xw = M * K + sum(u["N"] * K for u in g)
            work += [("amax X,W " + names, 2 * xw, "B"), ("cast X,W " + names, 4 * xw, "B")]
            work += [("gemm fwd " + names, sum(2 * M * u["N"] * K for u in g), "F")]
            gy = sum(M * u["N"] for u in g)
            work += [("amax dY " + names, 2 * gy, "B"), ("cast dY " + names, 4 * gy, "B")]
            work += [("gemm bwd " + names, sum(4 * M * u["N"] * K for u in g), "F")]
            continue
        for j, u in enumerate(g):
            xw = (M * K if j == 0 else 0) + u["N"] * K
            lab = ("X," if j == 0 else "") + "W " + u["name"]
            work += [("amax " + lab, 2 * xw, "B"), ("cast " + lab, 4 * xw, "B")]
        work += [("gemm fwd " + names, sum(2 * M * u["N"] * K for u in g), "F")]
        for u in g:
            work += [("amax dY " + u["name"], 2 * M * u["N"], "B"), ("cast dY " + u["name"], 4 * M * u["N"], "B")]
        work += [("gemm bwd " + names, sum(4 * M * u["N"] * K for u in g), "F")]

    def step():
        for g in groups:
            if len(g) == 1:
                u = g[0]
                u["plan"].forward(u["x"], u["w"], u["saved"], y=u["y"])
                u["plan"].backward(u["dy"], u["saved"], dx=u["dx"], dw=u["dw"], x=u["x"])
            else:
                sp, sv = g[0]["group_plan"], [u["saved"] for u in g]
                sp.forward(g[0]["x"], [u["w"] for u in g], sv, ys=[u["y"] for u in g])
                sp.backward([u["dy"] for u in g], sv, dxs=[u["dx"] for u in g], dws=[u["dw"] for u in g], x=g[0]["x"])

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
    for i in range(per):
        lab, w, kind = work[i] if per == len(work) else ("", 0, "B")
        rate = (f"{w / (acc[i] * 1e-3) / 1e9:8.0f} GB/s" if kind == "B" else f"{w / (acc[i] * 1e-3) / 1e12:8.0f} TF/s") \
            if w else ""
        print(f"  {i:3d} {KIND.get(kinds[i], kinds[i]):10s} {acc[i] * 1e3:9.1f} us  {lab:22s} {rate}")

if __name__ == "__main__":
    main()
