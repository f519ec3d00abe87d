"""One launch each of our fwd-shape GEMM and cuBLASLt FP8 (for side-by-side ncu captures)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16099_b200 import ops
M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 14336, 4096))]
A = torch.randint(0, 0x70, (M, K), dtype=torch.uint8, device="cuda")
B = torch.randint(0, 0x70, (N, K), dtype=torch.uint8, device="cuda")
s = torch.ones(1, device="cuda")
for _ in range(2):
    ops.gemm(A, "e4m3", s, B, "e4m3", s, "tensor")
    torch._scaled_mm(A.view(torch.float8_e4m3fn), B.view(torch.float8_e4m3fn).t(), scale_a=s, scale_b=s,
                     out_dtype=torch.bfloat16)
torch.cuda.synchronize()
