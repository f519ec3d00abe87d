"""GEMM efficiency probe normalised by the SM clock: runs each variant back to back for ~1.5 s while
sampling NVML (SM clock, power) and reports TFLOP/s, median SM MHz and flop/cycle/SM
(= TFLOP/s / (MHz x SMs)), which separates kernel design from the power-capped clock.
Variants: our tensorwise FP8 GEMM, our MXFP8 GEMM (+ knob experiments, MX_PROBE_KNOBS="gemm_raster=0;mx_sf_split=2"), cuBLASLt FP8 / MXFP8.
Context for tuning only; not part of the contract."""
import json
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.environ.get("FP8T_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops  # noqa: E402

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
SMS = torch.cuda.get_device_properties(0).multi_processor_count


def probe(fn, flops, seconds=1.5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    n = max(5, int(seconds / max(time.perf_counter() - t0, 1e-4)))
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(H) / 1000.0))
            time.sleep(0.005)

    th = threading.Thread(target=sample, daemon=True)
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
    finally:
        stop.set()
        th.join()
    ms = a.elapsed_time(b) / n
    clk = sorted(s[0] for s in samples) or [0]
    pw = sorted(s[1] for s in samples) or [0]
    mhz = clk[len(clk) // 2]
    tf = flops / ms / 1e9
    return {"tflops": round(tf), "mhz": mhz, "w": round(pw[len(pw) // 2]),
            "flop_per_clk_sm": round(tf * 1e12 / (mhz * 1e6 * SMS)) if mhz else None}


def main():
    shapes = [tuple(int(v) for v in sh.split("x")) for sh in
              os.environ.get("MX_PROBE_SHAPES", "16384x28672x8192,16384x14336x4096").split(",")]
    variants = os.environ.get("MX_PROBE_VARIANTS", "fp8,mx,cublas_fp8,cublas_mx").split(",")
    envs = [e for e in os.environ.get("MX_PROBE_KNOBS", "").split(";") if e]   # e.g. "gemm_raster=0"
    for M, N, K in shapes:
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.randint(0, 0x70, (M, K), dtype=torch.uint8, device="cuda", generator=g)
        B = torch.randint(0, 0x70, (N, K), dtype=torch.uint8, device="cuda", generator=g)
        sfa = torch.randint(118, 128, (M * K // 32,), dtype=torch.uint8, device="cuda", generator=g)
        sfb = torch.randint(118, 128, (N * K // 32,), dtype=torch.uint8, device="cuda", generator=g)
        s = torch.ones(1, device="cuda")
        flops = 2.0 * M * N * K
        for v in variants:
            runs = [("", None)] + ([(e, e) for e in envs] if v in ("mx", "fp8") else [])
            for tag, env in runs:
                if env:
                    for kv in env.split(","):
                        k, val = kv.split("=")
                        ops.set_knob(k, int(val))
                if v == "fp8":
                    fn = lambda: ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor")  # noqa: E731
                elif v == "mx":
                    fn = lambda: ops.gemm(A, "e4m3", sfa, B, "e4m3", sfb, "mx32")  # noqa: E731
                elif v in ("mx_mn", "fp8_mn"):   # both operands MN-major (the backward's layout)
                    At, Bt = A.t().contiguous(), B.t().contiguous()
                    if v == "mx_mn":
                        fn = lambda: ops.gemm(At, "e4m3", sfa, Bt, "e4m3", sfb, "mx32", a_mn=True, b_mn=True)  # noqa: E731
                    else:
                        fn = lambda: ops.gemm(At, "e4m3", s, Bt, "e4m3", s, "tensor", a_mn=True, b_mn=True)  # noqa: E731
                elif v == "cublas_fp8":
                    a8, b8 = A.view(torch.float8_e4m3fn), B.view(torch.float8_e4m3fn)
                    fn = lambda: torch._scaled_mm(a8, b8.t(), scale_a=s, scale_b=s, out_dtype=torch.bfloat16)  # noqa: E731
                else:
                    a8, b8 = A.view(torch.float8_e4m3fn), B.view(torch.float8_e4m3fn)
                    e8 = torch.float8_e8m0fnu
                    fn = lambda: torch._scaled_mm(a8, b8.t(), scale_a=sfa.view(e8), scale_b=sfb.view(e8),  # noqa: E731
                                                  out_dtype=torch.bfloat16)
                try:
                    r = probe(fn, flops)
                except Exception as e:  # noqa: BLE001
                    r = {"error": str(e)[:100]}
                ops.reset_knobs()
                print(json.dumps({"shape": [M, N, K], "variant": v, "env": tag, **r}), flush=True)
        del A, B, sfa, sfb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
