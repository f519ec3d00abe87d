"""Full-size parity at BASELINE.json configs[1] (C2: M=16384, K=4096, N=14336, tensorwise), in the
launch configuration bench.py times (fp8_linear_fwd / fp8_linear_bwd, bf16 in/out).

The oracle cannot run the full GEMMs in reasonable time, so (SURVEY §4 "GPU integration"):
  * amax and scales are checked over the full tensors, bit-exact;
  * FP8 codes are checked bit-exact on sampled rows (cast entry point, same kernels);
  * Y and dX on 48 sampled rows x all columns, dW on 48 sampled rows x all columns, each computed
    by the oracle from its own casts (full-tensor scales) within the north-star tolerance.
"""

import numpy as np
import pytest
import torch

import synth
from oracle import codecs, fp8, gemm as ogemm
from oracle.codecs import E4M3, E5M2

pytestmark = pytest.mark.gpu

M, N, K = 16384, 14336, 4096


def _bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def _tol(got, ref, bound, tol=1e-2):
    err = np.abs(got - ref)
    ratio = float(np.max(err / (bound + 1e-30)))
    assert ratio <= tol, f"max err/bound {ratio:.3e}"
    return ratio


@pytest.fixture(scope="module")
def c2():
    x, w, dy = synth.linear_inputs("c2", M, N, K, seed=0)
    return x, w, dy


def test_c2_fullsize_tensorwise(c2):
    from paper_2507_16099_b200 import ops
    x, w, dy = c2
    bf = torch.bfloat16
    X = torch.from_numpy(x).to(bf).cuda()
    W = torch.from_numpy(w).to(bf).cuda()
    G = torch.from_numpy(dy).to(bf).cuda()
    plan = ops.LinearPlan(M, N, K, recipe="tensorwise", out_dtype=bf)
    saved = plan.new_saved()
    Y = plan.forward(X, W, saved)
    DX, DW = plan.backward(G, saved)
    cx = ops.cast(X, "e4m3", "tensor")
    cw = ops.cast(W, "e4m3", "tensor")
    cg = ops.cast(G, "e5m2", "tensor")
    torch.cuda.synchronize()

    # full-tensor amax / scale (oracle), bit-exact
    sx = fp8.scale_from_amax(fp8.amax(x), E4M3)
    sw = fp8.scale_from_amax(fp8.amax(w), E4M3)
    sg = fp8.scale_from_amax(fp8.amax(dy), E5M2)
    for out, a, s in ((cx, fp8.amax(x), sx), (cw, fp8.amax(w), sw), (cg, fp8.amax(dy), sg)):
        assert _bits(out["amax"].cpu().numpy())[0] == _bits(a).reshape(-1)[0]
        assert _bits(out["scale"].cpu().numpy())[0] == _bits(s).reshape(-1)[0]

    rng = np.random.default_rng(2024)
    rows_m = np.sort(rng.choice(M, 48, replace=False))
    rows_n = np.sort(rng.choice(N, 48, replace=False))
    # sampled codes, bit-exact
    assert np.array_equal(cx["q"][torch.from_numpy(rows_m).cuda()].cpu().numpy(), fp8.cast_scaled(x[rows_m], sx, E4M3))
    assert np.array_equal(cw["q"][torch.from_numpy(rows_n).cuda()].cpu().numpy(), fp8.cast_scaled(w[rows_n], sw, E4M3))
    assert np.array_equal(cg["q"][torch.from_numpy(rows_m).cuda()].cpu().numpy(), fp8.cast_scaled(dy[rows_m], sg, E5M2))

    # oracle operands (its own casts with the full-tensor scales)
    wq = fp8.cast_scaled(w, sw, E4M3)                       # [N, K]
    xq = fp8.cast_scaled(x, sx, E4M3)                       # [M, K]
    gq_rows = fp8.cast_scaled(dy[rows_m], sg, E5M2)         # [48, N]
    gq_cols = fp8.cast_scaled(dy[:, rows_n], sg, E5M2)      # [M, 48]

    # Y[rows_m, :] = Xq[rows_m] Wq^T / (sx sw)
    ref = ogemm.gemm_ref(xq[rows_m], E4M3, sx, wq, E4M3, sw)
    bd = ogemm.abs_bound(xq[rows_m], E4M3, sx, wq, E4M3, sw)
    _tol(Y[torch.from_numpy(rows_m).cuda()].float().cpu().numpy().astype(np.float64), ref, bd)
    # dX[rows_m, :] = Gq[rows_m] Wq / (sg sw)
    ref = ogemm.gemm_ref(gq_rows, E5M2, sg, wq.T, E4M3, sw)
    bd = ogemm.abs_bound(gq_rows, E5M2, sg, wq.T, E4M3, sw)
    _tol(DX[torch.from_numpy(rows_m).cuda()].float().cpu().numpy().astype(np.float64), ref, bd)
    # dW[rows_n, :] = Gq[:, rows_n]^T Xq / (sg sx)
    ref = ogemm.gemm_ref(gq_cols.T, E5M2, sg, xq.T, E4M3, sx)
    bd = ogemm.abs_bound(gq_cols.T, E5M2, sg, xq.T, E4M3, sx)
    _tol(DW[torch.from_numpy(rows_n).cuda()].float().cpu().numpy().astype(np.float64), ref, bd)


def _sample(n, k, seed):
    return np.sort(np.random.default_rng(seed).choice(n, k, replace=False))


def _gpu_rows_cols(T, rows, cols):
    r = torch.from_numpy(rows).cuda()
    c = torch.from_numpy(cols).cuda()
    return T[r][:, c].float().cpu().numpy().astype(np.float64)


def test_c3w1_fullsize_rowwise():
    """BASELINE.json configs[2] (rowwise) at the Llama-3-8B w1 shape M=16384, N=14336, K=4096, bf16,
    through fp8_linear_fwd / fp8_linear_bwd as bench.py runs it.  Every rowwise scaling unit is a row
    or a column, so the oracle quantizes only the sampled rows / columns (P:597 operand plan, DESIGN
    §2): Y, dX and dW on 48 x 48 sampled outputs, each a full-length contraction, within tolerance."""
    from paper_2507_16099_b200 import ops
    M3, N3, K3 = 16384, 14336, 4096
    x, w, dy = synth.linear_inputs("c3", M3, N3, K3, seed=0)
    bf = torch.bfloat16
    X, W, G = (torch.from_numpy(a).to(bf).cuda() for a in (x, w, dy))
    plan = ops.LinearPlan(M3, N3, K3, recipe="rowwise", out_dtype=bf)
    saved = plan.new_saved()
    Y = plan.forward(X, W, saved)
    DX, DW = plan.backward(G, saved)
    torch.cuda.synchronize()
    rm, rn, rk = _sample(M3, 48, 1), _sample(N3, 48, 2), _sample(K3, 48, 3)
    # Y[m, n] = Xq_row[m] . Wq_row[n] / (sx[m] sw[n])
    xq, sx, _ = fp8.cast_rowwise(x[rm], E4M3)
    wq, sw, _ = fp8.cast_rowwise(w[rn], E4M3)
    _tol(_gpu_rows_cols(Y, rm, rn), ogemm.gemm_ref(xq, E4M3, sx, wq, E4M3, sw),
         ogemm.abs_bound(xq, E4M3, sx, wq, E4M3, sw))
    # dX[m, k] = Gq_row[m] . Wq_col[:, k] / (sg[m] sw_col[k])   (W scaled per column k over N)
    gq, sg, _ = fp8.cast_rowwise(dy[rm], E5M2)
    wcq, swc, _ = fp8.cast_colwise(w[:, rk], E4M3)
    _tol(_gpu_rows_cols(DX, rm, rk), ogemm.gemm_ref(gq, E5M2, sg, wcq.T, E4M3, swc),
         ogemm.abs_bound(gq, E5M2, sg, wcq.T, E4M3, swc))
    # dW[n, k] = Gq_col[:, n] . Xq_col[:, k] / (sg_col[n] sx_col[k])   (scaled per column over M)
    gcq, sgc, _ = fp8.cast_colwise(dy[:, rn], E5M2)
    xcq, sxc, _ = fp8.cast_colwise(x[:, rk], E4M3)
    _tol(_gpu_rows_cols(DW, rn, rk), ogemm.gemm_ref(gcq.T, E5M2, sgc, xcq.T, E4M3, sxc),
         ogemm.abs_bound(gcq.T, E5M2, sgc, xcq.T, E4M3, sxc))


def test_c4_fullsize_mxfp8():
    """BASELINE.json configs[3] (MXFP8 block-32 E8M0, FLOOR) at the Llama-3-70B w1 shape M=16384,
    N=28672, K=8192, bf16, through fp8_linear_fwd / fp8_linear_bwd (the bench's launch configuration:
    row-major dim1 codes read MN-major by the block-scaled GEMM).  A 32-block never leaves its row
    (dim0) or column (dim1), so the oracle quantizes only the sampled rows / columns: Y, dX, dW on
    48 x 48 sampled outputs, full-length contractions, within tolerance."""
    from oracle import mx as omx
    from paper_2507_16099_b200 import ops
    M4, N4, K4 = 16384, 28672, 8192
    x, w, dy = synth.linear_inputs("c4", M4, N4, K4, seed=0)
    bf = torch.bfloat16
    X, W, G = (torch.from_numpy(a).to(bf).cuda() for a in (x, w, dy))
    plan = ops.LinearPlan(M4, N4, K4, recipe="mxfp8", out_dtype=bf)
    saved = plan.new_saved()
    Y = plan.forward(X, W, saved)
    DX, DW = plan.backward(G, saved)
    torch.cuda.synchronize()
    rm, rn, rk = _sample(M4, 48, 4), _sample(N4, 48, 5), _sample(K4, 48, 6)
    # Y = X dim0 . W dim0 (blocks along K)
    a, sa = omx.quantize_dim0(x[rm], E4M3)
    b, sb = omx.quantize_dim0(w[rn], E4M3)
    _tol(_gpu_rows_cols(Y, rm, rn), ogemm.mx_gemm_ref(a, sa, E4M3, b, sb, E4M3),
         ogemm.mx_abs_bound(a, sa, E4M3, b, sb, E4M3))
    # dX = dY dim0 (blocks along N) . W dim1 (blocks along N)
    a, sa = omx.quantize_dim0(dy[rm], E5M2)
    b, sb = omx.quantize_dim1(w[:, rk], E4M3)
    _tol(_gpu_rows_cols(DX, rm, rk), ogemm.mx_gemm_ref(a, sa, E5M2, b, sb, E4M3),
         ogemm.mx_abs_bound(a, sa, E5M2, b, sb, E4M3))
    # dW = dY dim1 (blocks along M) . X dim1 (blocks along M)
    a, sa = omx.quantize_dim1(dy[:, rn], E5M2)
    b, sb = omx.quantize_dim1(x[:, rk], E4M3)
    _tol(_gpu_rows_cols(DW, rn, rk), ogemm.mx_gemm_ref(a, sa, E5M2, b, sb, E4M3),
         ogemm.mx_abs_bound(a, sa, E5M2, b, sb, E4M3))


def test_c5_fullsize_fsdp_tensorwise():
    """BASELINE.json configs[4] (Llama-3.1-405B w1: K=16384, N=53248; 8192 tokens per rank, tensorwise)
    at full size on one rank, as `bench.py --config c5 --fsdp` runs it at N=1: the FP8 weight gather
    (fp8_fsdp_allgather: amax -> NCCL all-reduce MAX -> cast into slot 0 -> all-gather) feeds the linear's
    pre-cast weight path.  Global amax and scale bit-exact over the full 872M-element weight, sampled
    gathered rows bit-exact, Y / dX / dW on 48 x 48 sampled outputs (full contractions) within tolerance."""
    import os
    import torch.distributed as dist
    from paper_2507_16099_b200 import ops
    from paper_2507_16099_b200.fsdp import Comm
    M5, N5, K5 = 8192, 53248, 16384
    x, w, dy = synth.linear_inputs("c5", M5, N5, K5, seed=0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29541"
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = Comm()
        bf = torch.bfloat16
        X, W, G = (torch.from_numpy(a).to(bf).cuda() for a in (x, w, dy))
        wq_d, ws_d, wa_d = comm.allgather_fp8(W, "e4m3")
        plan = ops.LinearPlan(M5, N5, K5, recipe="tensorwise", out_dtype=bf)
        saved = plan.new_saved()
        Y = plan.forward(X, None, saved, w_fp8=(wq_d, ws_d))
        DX, DW = plan.backward(G, saved, w_fp8=(wq_d, ws_d))
        cx = ops.cast(X, "e4m3", "tensor")
        cg = ops.cast(G, "e5m2", "tensor")
        torch.cuda.synchronize()
        aw = fp8.amax(w)
        sw = fp8.scale_from_amax(aw, E4M3)
        assert _bits(wa_d.cpu().numpy())[0] == _bits(aw).reshape(-1)[0]
        assert _bits(ws_d.cpu().numpy())[0] == _bits(sw).reshape(-1)[0]
        sx = fp8.scale_from_amax(fp8.amax(x), E4M3)
        sg = fp8.scale_from_amax(fp8.amax(dy), E5M2)
        assert _bits(cx["scale"].cpu().numpy())[0] == _bits(sx).reshape(-1)[0]
        assert _bits(cg["scale"].cpu().numpy())[0] == _bits(sg).reshape(-1)[0]
        rm, rn, rk = _sample(M5, 48, 7), _sample(N5, 48, 8), _sample(K5, 48, 9)
        wq_rows = fp8.cast_scaled(w[rn], sw, E4M3)
        assert np.array_equal(wq_d[torch.from_numpy(rn).cuda()].cpu().numpy(), wq_rows)
        xq = fp8.cast_scaled(x[rm], sx, E4M3)
        _tol(_gpu_rows_cols(Y, rm, rn), ogemm.gemm_ref(xq, E4M3, sx, wq_rows, E4M3, sw),
             ogemm.abs_bound(xq, E4M3, sx, wq_rows, E4M3, sw))
        gq = fp8.cast_scaled(dy[rm], sg, E5M2)
        wcols = fp8.cast_scaled(w[:, rk], sw, E4M3).T            # [48 (k), N]
        _tol(_gpu_rows_cols(DX, rm, rk), ogemm.gemm_ref(gq, E5M2, sg, wcols, E4M3, sw),
             ogemm.abs_bound(gq, E5M2, sg, wcols, E4M3, sw))
        gcols = fp8.cast_scaled(dy[:, rn], sg, E5M2).T           # [48 (n), M]
        xcols = fp8.cast_scaled(x[:, rk], sx, E4M3).T            # [48 (k), M]
        _tol(_gpu_rows_cols(DW, rn, rk), ogemm.gemm_ref(gcols, E5M2, sg, xcols, E4M3, sx),
             ogemm.abs_bound(gcols, E5M2, sg, xcols, E4M3, sx))
        comm.close()
    finally:
        dist.destroy_process_group()
