"""GEMM-only microbenchmark: our tcgen05 kernel (both CTA-group modes) vs cuBLASLt FP8
(torch._scaled_mm) on the C2 GEMM shapes.  Context for tuning; not part of the contract."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops  # noqa: E402

SHAPES = [(16384, 14336, 4096), (16384, 4096, 14336), (14336, 4096, 16384), (8192, 8192, 8192),
          (16384, 28672, 8192)]


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
    out = []
    for M, N, K in SHAPES:
        A = torch.randint(0, 0x70, (M, K), dtype=torch.uint8, device="cuda")
        B = torch.randint(0, 0x70, (N, K), dtype=torch.uint8, device="cuda")
        s = torch.ones(1, device="cuda")
        D = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        flops = 2.0 * M * N * K
        row = {"M": M, "N": N, "K": K}
        for dbg in ("0", "1"):   # 1: epilogue stores skipped (mainloop-only upper bound)
            ops.set_knob("gemm_debug", int(dbg))
            ms = timeit(lambda: ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor"))
            row["ours" if dbg == "0" else "ours_nostore"] = round(flops / ms / 1e9)
        ops.set_knob("gemm_debug", int("0"))
        if M % 128 == 0 and N % 128 == 0 and K % 128 == 0:   # MXFP8 block-scaled kind, codes 127 (=1.0)
            sfa = torch.full((M * K // 32,), 127, dtype=torch.uint8, device="cuda")
            sfb = torch.full((N * K // 32,), 127, dtype=torch.uint8, device="cuda")
            for dbg in os.environ.get("GEMM_BENCH_MX_DBG", "0,2").split(","):
                # 1: no epilogue stores; 2: no tcgen05.cp of scales; 4: no scale TMA loads
                ops.set_knob("gemm_debug", int(dbg))
                ms = timeit(lambda: ops.gemm(A, "e4m3", sfa, B, "e4m3", sfb, "mx32"))
                row["ours_mx" + ("" if dbg == "0" else "_dbg" + dbg)] = round(flops / ms / 1e9)
            ops.set_knob("gemm_debug", int("0"))
            # MN-major operands (the MXFP8 backward's layout): A stored [K,M], B stored [K,N]
            At, Bt = A.t().contiguous(), B.t().contiguous()
            ms = timeit(lambda: ops.gemm(At, "e4m3", sfa, Bt, "e4m3", sfb, "mx32", a_mn=True, b_mn=True))
            row["ours_mx_mnmn"] = round(flops / ms / 1e9)
            del At, Bt
            try:   # cuBLASLt MXFP8 (block-scaled) through torch._scaled_mm with e8m0 scales
                e8 = torch.float8_e8m0fnu
                ms = timeit(lambda: torch._scaled_mm(A.view(torch.float8_e4m3fn), B.view(torch.float8_e4m3fn).t(),
                                                     scale_a=sfa.view(e8), scale_b=sfb.view(e8),
                                                     out_dtype=torch.bfloat16))
                row["cublaslt_mxfp8_tflops"] = round(flops / ms / 1e9)
            except Exception as e:  # noqa: BLE001
                row["cublaslt_mxfp8_tflops"] = f"n/a: {e}"[:120]
        try:
            a8 = A.view(torch.float8_e4m3fn)
            b8 = B.view(torch.float8_e4m3fn)
            ms = timeit(lambda: torch._scaled_mm(a8, b8.t(), scale_a=s, scale_b=s, out_dtype=torch.bfloat16))
            row["cublaslt_fp8_tflops"] = round(flops / ms / 1e9)
        except Exception as e:  # noqa: BLE001
            row["cublaslt_fp8_tflops"] = f"n/a: {e}"[:80]
        Ab = torch.randn((M, K), dtype=torch.bfloat16, device="cuda")
        Bb = torch.randn((N, K), dtype=torch.bfloat16, device="cuda")
        ms = timeit(lambda: torch.matmul(Ab, Bb.t()), iters=10)
        row["cublas_bf16_tflops"] = round(flops / ms / 1e9)
        out.append(row)
        print(json.dumps(row), flush=True)
        del A, B, D, Ab, Bb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
