"""Small invocations of every kernel family for compute-sanitizer runs."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2507_16099_b200 import ops

M, N, K = 256, 384, 512
x, w, dy = synth.linear_inputs("c2", M, N, K, seed=0)
X, W, G = (torch.from_numpy(a).to(torch.bfloat16).cuda() for a in (x, w, dy))
for gran in ("tensor", "row", "col", "row_col"):
    ops.cast(X, "e4m3", gran, want_q=True, want_qt=True)
ops.cast(X, "e4m3", "mx32", want_q=True, want_qt=True)      # TMA-ring MX cast (transposed dim1)
ops.cast(X, "e5m2", "mx32_rm", want_q=True, want_qt=True)   # TMA-ring MX cast (row-major dim1)
ops.amax(X, "row"), ops.amax(X, "col")                      # TMA-ring strip amax
for recipe in ("tensorwise", "rowwise", "rowwise_gw_hp", "mxfp8"):
    plan = ops.LinearPlan(M, N, K, recipe=recipe)
    saved = plan.new_saved()
    plan.forward(X, W, saved)
    plan.backward(G, saved, x=X)
    plan.forward(X, W, None)
# MoE grouped GEMM (M-grouped fwd / dX, K-grouped dW, an empty expert)
sizes = [128, 0, 256, 128]
E, T = len(sizes), sum(sizes)
offs = torch.tensor(np.concatenate([[0], np.cumsum(sizes)]), dtype=torch.int32, device="cuda")
for recipe in ("tensorwise", "rowwise"):
    gp = ops.GroupedPlan(T, E, 256, K, recipe=recipe)
    gs = gp.new_saved()
    Xg = torch.randn((T, K), device="cuda").to(torch.bfloat16)
    Wg = (torch.randn((E * 256, K), device="cuda") * 0.02).to(torch.bfloat16)
    Gg = (torch.randn((T, 256), device="cuda") * 1e-3).to(torch.bfloat16)
    gp.forward(Xg, Wg, offs, gs)
    gp.backward(Gg, offs, gs)
# fused P2P FSDP gather over 2 simulated ranks, and the MX scale re-tiling
from paper_2507_16099_b200.fsdp import P2PWindow
wins = P2PWindow.local_group(2, N * K)
P2PWindow.allgather_local(wins, [W[:N // 2].contiguous(), W[N // 2:].contiguous()])
torch.cuda.synchronize()
for w_ in wins:
    w_.close()
# long-K plain GEMM (4 epilogue warps; the short-K launches above use 8)
A8 = torch.randint(0, 0x70, (256, 2304), dtype=torch.uint8, device="cuda")
B8 = torch.randint(0, 0x70, (256, 2304), dtype=torch.uint8, device="cuda")
one = torch.ones(1, device="cuda")
ops.gemm(A8, "e4m3", one, B8, "e4m3", one, "tensor")
slots = [ops.cast(W[r * 128:(r + 1) * 128].contiguous(), "e4m3", "mx32_rm", want_q=True, want_qt=True) for r in range(3)]
ops.mx_scales_unshard(torch.cat([s["scale_t"] for s in slots]), 3, 128, K)
torch.cuda.synchronize()
# 256 x 512 GEMM tiles: bf16 output through the TMA-store epilogue, fp32 output through direct stores,
# a two-problem launch (linear backward with N, K multiples of 512 and K >= 8192 -> the auto policy)
ops.set_knob("gemm_n512", 1)
A9 = torch.randint(0, 0x70, (512, 1024), dtype=torch.uint8, device="cuda")
B9 = torch.randint(0, 0x70, (1024, 1024), dtype=torch.uint8, device="cuda")
ops.gemm(A9, "e4m3", one, B9, "e4m3", one, "tensor")
ops.gemm(A9, "e4m3", one, B9, "e4m3", one, "tensor", out_dtype=torch.float32)
ops.set_knob("gemm_n512", 2)
X9 = torch.randn((256, 8192), device="cuda").to(torch.bfloat16)
W9 = (torch.randn((512, 8192), device="cuda") * 0.02).to(torch.bfloat16)
G9 = (torch.randn((256, 512), device="cuda") * 1e-3).to(torch.bfloat16)
p9 = ops.LinearPlan(256, 512, 8192, recipe="tensorwise")
s9 = p9.new_saved()
p9.forward(X9, W9, s9)
p9.backward(G9, s9)
ops.reset_knobs()
# shared-input groups: multi-problem GEMM launches (6 problems in the backward), FP8 + BF16 kinds apart
for recipe in ("rowwise", "mxfp8", "rowwise_gw_hp", "tensorwise"):
    Ns = [256, 128, 128]
    sp = ops.SharedInputPlan(256, Ns, 256, recipe=recipe)
    sv = sp.new_saved()
    Xs = torch.randn((256, 256), device="cuda").to(torch.bfloat16)
    Ws = [(torch.randn((n, 256), device="cuda") * 0.02).to(torch.bfloat16) for n in Ns]
    Gs = [(torch.randn((256, n), device="cuda") * 1e-3).to(torch.bfloat16) for n in Ns]
    sp.forward(Xs, Ws, sv)
    sp.backward(Gs, sv, x=Xs)
# ring wrap-around of the warp-specialised amax / MX cast kernels (capped grid), and the previous kernels
ops.set_knob("cast_grid", 3)
ops.amax(X, "row"), ops.amax(X, "col")
ops.cast(X, "e5m2", "mx32_rm", want_q=True, want_qt=True)
ops.reset_knobs()
ops.set_knob("amax_rc", 0)
ops.set_knob("mx_cast_ws", 0)
ops.amax(X, "row"), ops.amax(X, "col")
ops.cast(X, "e5m2", "mx32_rm", want_q=True, want_qt=True)
ops.reset_knobs()
torch.cuda.synchronize()
print("ok")
