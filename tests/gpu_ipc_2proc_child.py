"""One rank of test_gpu_parity.test_p2p_two_processes_ipc: two OS processes on the same GPU, windows
mapped with real CUDA IPC handles exchanged over a gloo group (fp8_p2p_alloc / fp8_p2p_open), then
the per-rank P2P entry points across the process boundary: FSDP FP8 gather, dW GEMM with fused
reduce-scatter, async-TP forward + backward.  Every rank checks its own outputs against references
it computes locally from the (deterministic, seeded) inputs of all ranks."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import fp8  # noqa: E402
from paper_2507_16099_b200 import ops  # noqa: E402
from paper_2507_16099_b200.fsdp import P2PWindow  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = world
    Ml, N, K = 256, 256 * P, 384
    w_np = synth.tensor_c2("w", (N, K), seed=60)
    W = dev(w_np)
    shard = W[rank * (N // P):(rank + 1) * (N // P)].contiguous()
    gwin = P2PWindow.over_group(N * K)
    rwin = P2PWindow.over_group(N * K * 2)
    twin = P2PWindow.over_group(P * Ml * K)
    trwin = P2PWindow.over_group(P * Ml * K * 2)
    X = [dev(synth.tensor_c2("x", (Ml, K), seed=40 + r)) for r in range(P)]
    G = [dev(synth.tensor_c2("dy", (Ml, N), seed=50 + r)) for r in range(P)]
    plan = ops.LinearPlan(Ml, N, K, recipe="tensorwise")
    q_ref = fp8.cast_tensorwise(w_np, "e4m3")[0]
    for it in range(2):
        # FSDP: gather -> forward -> backward with the fused dW reduce-scatter
        codes, sc, _ = gwin.allgather_fp8(shard, "e4m3")
        saved = plan.new_saved()
        plan.forward(X[rank], None, saved, w_fp8=(codes, sc))
        dws = torch.empty((N // P, K), dtype=torch.bfloat16, device="cuda")
        dx = ops.linear_backward_rs(plan, G[rank], saved, rwin, dws, w_fp8=(codes, sc))
        torch.cuda.synchronize()
        assert np.array_equal(codes.cpu().numpy(), q_ref), "gather"
        acc = None
        for r in range(P):
            sv = plan.new_saved()
            plan.forward(X[r], W, sv)
            dxr, dwr = plan.backward(G[r], sv)
            if r == rank:
                assert torch.equal(dxr, dx), "dx"
            acc = dwr.float() if acc is None else acc + dwr.float()
        torch.cuda.synchronize()
        assert torch.equal(dws, acc.to(torch.bfloat16)[rank * (N // P):(rank + 1) * (N // P)]), "dw shard"
        # async-TP forward + backward
        Xs = [dev(synth.tensor_c2("x", (Ml, K), seed=70 + r + it)) for r in range(P)]
        Wl = [dev(synth.tensor_c2("w", (272, K), seed=80 + r)) for r in range(P)]
        dYs = [dev(synth.tensor_c2("dy", (P * Ml, 272), seed=90 + r + it)) for r in range(P)]
        y = twin.tp_linear_fwd(Xs[rank], Wl[rank], out_dtype=torch.bfloat16)
        dxs, dwl = twin.tp_linear_bwd(dYs[rank], twin.last_tp_ws, trwin, K)
        torch.cuda.synchronize()
        Xf = torch.cat(Xs)
        pl = ops.LinearPlan(P * Ml, 272, K, recipe="tensorwise")
        parts = []
        for r in range(P):
            sv = pl.new_saved()
            yr = pl.forward(Xf, Wl[r], sv)
            dxr, dwr = pl.backward(dYs[r], sv)
            if r == rank:
                assert torch.equal(y, yr), "tp y"
                assert torch.equal(dwl, dwr), "tp dw"
            parts.append(dxr.float())
        acc = parts[0].clone()
        for f in parts[1:]:
            acc += f
        assert torch.equal(dxs, acc.to(torch.bfloat16)[rank * Ml:(rank + 1) * Ml]), "tp dx shard"
        dist.barrier()
    for w_ in (gwin, rwin, twin, trwin):
        w_.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank} ok", flush=True)


if __name__ == "__main__":
    main()
