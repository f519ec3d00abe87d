"""Child process of test_gpu_parity.test_p2p_per_rank_calls_on_streams (run with
CUDA_DEVICE_MAX_CONNECTIONS=32 so every simulated rank's stream gets its own hardware queue): the
PER-RANK P2P entry points (fp8_fsdp_allgather_p2p, fp8_linear_bwd_rs, fp8_tp_allgather_linear_fwd),
each simulated rank issuing its calls on its own stream exactly as one process per GPU would, the
cross-rank waits resolved by the other streams running concurrently."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import fp8  # noqa: E402
from paper_2507_16099_b200 import ops  # noqa: E402
from paper_2507_16099_b200.fsdp import P2PWindow  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()


def run(P):
    streams = [torch.cuda.Stream() for _ in range(P)]
    Ml, N, K = 256, 256 * P, 384
    x_np = [synth.tensor_c2("x", (Ml, K), seed=40 + r) for r in range(P)]
    dy_np = [synth.tensor_c2("dy", (Ml, N), seed=50 + r) for r in range(P)]
    w_np = synth.tensor_c2("w", (N, K), seed=60)
    X, G = [dev(v) for v in x_np], [dev(v) for v in dy_np]
    W = dev(w_np)
    shards = [W[r * (N // P):(r + 1) * (N // P)].contiguous() for r in range(P)]
    gwin = P2PWindow.local_group(P, N * K)
    rwin = P2PWindow.local_group(P, N * K * 2)
    twin = P2PWindow.local_group(P, P * Ml * K)
    trwin = P2PWindow.local_group(P, P * Ml * K * 2)
    plans = [ops.LinearPlan(Ml, N, K, recipe="tensorwise") for _ in range(P)]
    saved = [p.new_saved() for p in plans]
    q_ref, s_ref, _ = fp8.cast_tensorwise(w_np, "e4m3")
    for it in range(2):
        torch.cuda.synchronize()
        outs, dws, dxs = [None] * P, [None] * P, [None] * P
        for r in range(P):   # each simulated rank: gather -> forward -> backward with fused RS
            with torch.cuda.stream(streams[r]):
                codes, sc, _ = gwin[r].allgather_fp8(shards[r], "e4m3")
                outs[r] = (codes, sc)
                plans[r].forward(X[r], None, saved[r], w_fp8=(codes, sc))
                dws[r] = torch.empty((N // P, K), dtype=torch.bfloat16, device="cuda")
                dxs[r] = ops.linear_backward_rs(plans[r], G[r], saved[r], rwin[r], dws[r], w_fp8=(codes, sc))
        torch.cuda.synchronize()
        for r in range(P):
            assert np.array_equal(outs[r][0].cpu().numpy(), q_ref), f"gather rank {r}"
        # reference: each rank's plain backward dW (bf16), summed in rank order in fp32, one rounding
        full = []
        for r in range(P):
            ps = plans[r].new_saved()
            plans[r].forward(X[r], W, ps)
            dxr, dwr = plans[r].backward(G[r], ps)
            assert torch.equal(dxr, dxs[r]), f"dx rank {r}"
            full.append(dwr.float())
        acc = full[0].clone()
        for f in full[1:]:
            acc += f
        ref = acc.to(torch.bfloat16)
        for r in range(P):
            assert torch.equal(dws[r], ref[r * (N // P):(r + 1) * (N // P)]), f"dw shard {r} (iter {it})"
        # async-TP forward, per-rank calls on their own streams
        Xs = [dev(synth.tensor_c2("x", (Ml, K), seed=70 + r + it)) for r in range(P)]
        Wl = [dev(synth.tensor_c2("w", (272, K), seed=80 + r)) for r in range(P)]
        ys = [None] * P
        torch.cuda.synchronize()
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                ys[r] = twin[r].tp_linear_fwd(Xs[r], Wl[r], out_dtype=torch.float32)
        torch.cuda.synchronize()
        Xf = torch.cat(Xs)
        pl = ops.LinearPlan(P * Ml, 272, K, recipe="tensorwise", out_dtype=torch.float32)
        for r in range(P):
            assert torch.equal(ys[r], pl.forward(Xf, Wl[r], None)), f"tp rank {r}"
        # async-TP backward (fused dX reduce-scatter), per-rank calls on their own streams
        dYs = [dev(synth.tensor_c2("dy", (P * Ml, 272), seed=90 + r + it)) for r in range(P)]
        bw = [None] * P
        torch.cuda.synchronize()
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                bw[r] = twin[r].tp_linear_bwd(dYs[r], twin[r].last_tp_ws, trwin[r], K)
        torch.cuda.synchronize()
        plb = ops.LinearPlan(P * Ml, 272, K, recipe="tensorwise")
        parts = []
        for r in range(P):
            sv = plb.new_saved()
            plb.forward(Xf, Wl[r], sv)
            dxr, dwr = plb.backward(dYs[r], sv)
            assert torch.equal(bw[r][1], dwr), f"tp dw rank {r}"
            parts.append(dxr.float())
        acc = parts[0].clone()
        for f in parts[1:]:
            acc += f
        ref = acc.to(torch.bfloat16)
        for r in range(P):
            assert torch.equal(bw[r][0], ref[r * Ml:(r + 1) * Ml]), f"tp dx shard {r}"
    for w_ in gwin + rwin + twin + trwin:
        w_.close()


if __name__ == "__main__":
    for P in (1, 2, 3):
        run(P)
    print("ok")
