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
