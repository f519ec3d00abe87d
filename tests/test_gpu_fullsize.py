"""Full-size parity at BASELINE.json configs[1..4] (C2 tensorwise, C3 rowwise at all seven layer shapes,
C4 MXFP8, C5 FSDP tensorwise), in the launch configuration bench.py times (fp8_linear_fwd /
fp8_linear_bwd, bf16 in/out), on the bytes the linear ITSELF writes (fp8_linear_buffers).

The oracle cannot run the full GEMMs in reasonable time, so (SURVEY §4 "GPU integration"):
  * amax and scales (every row / column vector, every E8M0 code) over the full tensors, bit-exact;
  * FP8 codes bit-exact on sampled rows / columns of the linear's own operand buffers;
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
    torch.cuda.synchronize()
    fb = plan.buffers(saved)          # what the linear itself wrote (the dual X/W amax + cast launches)
    f_amax = fb["amax_fwd"].cpu().numpy()
    DX, DW = plan.backward(G, saved)
    torch.cuda.synchronize()
    bb = plan.buffers(saved)

    # full-tensor amax / scale (oracle), bit-exact
    ax, aw, ag = fp8.amax(x), fp8.amax(w), fp8.amax(dy)
    sx = fp8.scale_from_amax(ax, E4M3)
    sw = fp8.scale_from_amax(aw, E4M3)
    sg = fp8.scale_from_amax(ag, E5M2)
    assert _bits(f_amax)[0] == _bits(ax).reshape(-1)[0] and _bits(f_amax)[1] == _bits(aw).reshape(-1)[0]
    assert _bits(bb["amax_bwd"].cpu().numpy())[0] == _bits(ag).reshape(-1)[0]
    for buf, s in ((bb["x_bwd_scale"], sx), (bb["w_bwd_scale"], sw), (bb["dy_dx_scale"], sg)):
        assert _bits(buf.cpu().numpy())[0] == _bits(s).reshape(-1)[0]

    rng = np.random.default_rng(2024)
    rows_m = np.sort(rng.choice(M, 48, replace=False))
    rows_n = np.sort(rng.choice(N, 48, replace=False))
    # sampled codes of the saved operands and the backward's dY operand, bit-exact
    im, in_ = torch.from_numpy(rows_m).cuda(), torch.from_numpy(rows_n).cuda()
    assert np.array_equal(bb["x_bwd"][im].cpu().numpy(), fp8.cast_scaled(x[rows_m], sx, E4M3))
    assert np.array_equal(bb["w_bwd"][in_].cpu().numpy(), fp8.cast_scaled(w[rows_n], sw, E4M3))
    assert np.array_equal(bb["dy_dx"][im].cpu().numpy(), fp8.cast_scaled(dy[rows_m], sg, E5M2))

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


def _cpu(t):
    return t.detach().cpu().numpy()


def _eq_bits(name, got, want):
    got, want = np.asarray(got), np.asarray(want)
    if want.dtype == np.float32:
        got, want = got.view(np.uint32), want.view(np.uint32)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    bad = np.count_nonzero(got != want)
    assert bad == 0, f"{name}: {bad} of {want.size} differ"


def _unblock(buf, R, C):
    """E8M0 blocked layout (fp8train.h) -> logical [R, C/32] codes (pure index permutation)."""
    C32 = C // 32
    b = _cpu(buf).reshape(R // 128, C32 // 4, 32, 4, 4)
    return b.transpose(0, 3, 2, 1, 4).reshape(R, C32)


C3_LINEARS = [("wq", 4096, 4096), ("wk", 1024, 4096), ("wv", 1024, 4096), ("wo", 4096, 4096),
              ("w1", 14336, 4096), ("w3", 14336, 4096), ("w2", 4096, 14336)]


@pytest.mark.parametrize("name,N3,K3", C3_LINEARS, ids=[c[0] for c in C3_LINEARS])
def test_c3_fullsize_rowwise(name, N3, K3):
    """BASELINE.json configs[2] (rowwise) at all seven Llama-3-8B layer shapes (M = 16384 tokens), bf16,
    through fp8_linear_fwd / fp8_linear_bwd as bench.py runs them, checking what the linear ITSELF
    wrote (fp8_linear_buffers):
      * every row- and column-amax vector and every row / column scale vector over the FULL tensors
        (X rows + cols, W rows + cols, dY rows + cols), bit-exact vs the oracle (P:597 operand plan);
      * FP8 codes of 64 sampled rows of each row-scaled copy and 64 sampled columns of each
        column-scaled copy, bit-exact;
      * Y, dX, dW on 48 x 48 sampled outputs (full-length contractions) within tolerance."""
    from paper_2507_16099_b200 import ops
    M3 = 16384
    seed = [c[0] for c in C3_LINEARS].index(name)
    x, w, dy = synth.linear_inputs("c3", M3, N3, K3, seed=seed)
    bf = torch.bfloat16
    X, W, G = (torch.from_numpy(a).to(bf).cuda() for a in (x, w, dy))
    plan = ops.LinearPlan(M3, N3, K3, recipe="rowwise", out_dtype=bf)
    saved = plan.new_saved()
    Y = plan.forward(X, W, saved)
    torch.cuda.synchronize()
    pr_m, pr_n, pc_k, pc_n = _sample(M3, 64, 11), _sample(N3, 64, 12), _sample(K3, 64, 13), _sample(N3, 64, 14)
    fb = plan.buffers(saved)
    f_amax, f_sx, f_sw = _cpu(fb["amax_fwd"]), _cpu(fb["x_fwd_scale"]), _cpu(fb["w_fwd_scale"])
    f_xrows = _cpu(fb["x_fwd"][torch.from_numpy(pr_m).cuda()])
    f_wrows = _cpu(fb["w_fwd"][torch.from_numpy(pr_n).cuda()])
    DX, DW = plan.backward(G, saved)
    torch.cuda.synchronize()
    bb = plan.buffers(saved)
    ic_k, ic_n = torch.from_numpy(pc_k).cuda(), torch.from_numpy(pc_n).cuda()

    # full amax / scale vectors
    ax_r, ax_c = fp8.amax(x, axis=1), fp8.amax(x, axis=0)
    aw_r, aw_c = fp8.amax(w, axis=1), fp8.amax(w, axis=0)
    ag_r, ag_c = fp8.amax(dy, axis=1), fp8.amax(dy, axis=0)
    _eq_bits("amax X rows", f_amax[:M3], ax_r)
    _eq_bits("amax X cols", f_amax[M3:M3 + K3], ax_c)
    _eq_bits("amax W rows", f_amax[M3 + K3:M3 + K3 + N3], aw_r)
    _eq_bits("amax W cols", f_amax[M3 + K3 + N3:], aw_c)
    _eq_bits("amax dY rows", _cpu(bb["amax_bwd"])[:M3], ag_r)
    _eq_bits("amax dY cols", _cpu(bb["amax_bwd"])[M3:], ag_c)
    _eq_bits("X row scales", f_sx, fp8.scale_from_amax(ax_r, E4M3))
    _eq_bits("W row scales", f_sw, fp8.scale_from_amax(aw_r, E4M3))
    _eq_bits("X col scales (saved)", _cpu(bb["x_bwd_scale"]), fp8.scale_from_amax(ax_c, E4M3))
    _eq_bits("W col scales (saved)", _cpu(bb["w_bwd_scale"]), fp8.scale_from_amax(aw_c, E4M3))
    _eq_bits("dY row scales", _cpu(bb["dy_dx_scale"]), fp8.scale_from_amax(ag_r, E5M2))
    _eq_bits("dY col scales", _cpu(bb["dy_dw_scale"]), fp8.scale_from_amax(ag_c, E5M2))

    # sampled codes from the linear's own buffers
    _eq_bits("X row-scaled rows", f_xrows, fp8.cast_rowwise(x[pr_m], E4M3)[0])
    _eq_bits("W row-scaled rows", f_wrows, fp8.cast_rowwise(w[pr_n], E4M3)[0])
    _eq_bits("dY row-scaled rows", _cpu(bb["dy_dx"][torch.from_numpy(pr_m).cuda()]), fp8.cast_rowwise(dy[pr_m], E5M2)[0])
    _eq_bits("X col-scaled cols (saved)", _cpu(bb["x_bwd"][:, ic_k]), fp8.cast_colwise(x[:, pc_k], E4M3)[0])
    _eq_bits("W col-scaled cols (saved)", _cpu(bb["w_bwd"][:, ic_k]), fp8.cast_colwise(w[:, pc_k], E4M3)[0])
    _eq_bits("dY col-scaled cols", _cpu(bb["dy_dw"][:, ic_n]), fp8.cast_colwise(dy[:, pc_n], E5M2)[0])

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


def _mx_codes_dim0(x, fmt):
    """Full E8M0 code array of the dim0 copy (blocks along the row): the oracle's block amax + code."""
    from oracle import mx as omx
    out = np.empty((x.shape[0], x.shape[1] // 32), np.uint8)
    for r0 in range(0, x.shape[0], 4096):
        out[r0:r0 + 4096] = omx.scale_code(omx.block_amax(x[r0:r0 + 4096]), fmt)
    return out


def _mx_codes_dim1(x, fmt):
    """Full E8M0 code array of the dim1 copy [C, R/32] (blocks along the column), chunked over columns."""
    from oracle import mx as omx
    out = np.empty((x.shape[1], x.shape[0] // 32), np.uint8)
    for c0 in range(0, x.shape[1], 2048):
        out[c0:c0 + 2048] = omx.scale_code(omx.block_amax(np.ascontiguousarray(x[:, c0:c0 + 2048].T)), fmt)
    return out


def test_c4_fullsize_mxfp8():
    """BASELINE.json configs[3] (MXFP8 block-32 E8M0, FLOOR) at the Llama-3-70B w1 shape M=16384,
    N=28672, K=8192, bf16, through fp8_linear_fwd / fp8_linear_bwd (the bench's launch configuration:
    row-major dim1 codes read MN-major by the block-scaled GEMM), checking what the linear ITSELF wrote
    (fp8_linear_buffers):
      * the FULL E8M0 code arrays of all six operand copies (X, W dim0; dY dim0; X, W, dY dim1), bit-exact
        vs the oracle's block amax -> code (R-c12);
      * FP8 codes of 64 sampled rows of each dim0 copy and 64 sampled columns of each dim1 copy;
      * Y, dX, dW on 48 x 48 sampled outputs, full-length contractions, within tolerance (a 32-block never
        leaves its row (dim0) or column (dim1), so the oracle quantizes only the sampled rows / columns)."""
    from oracle import mx as omx
    from paper_2507_16099_b200 import ops
    M4, N4, K4 = 16384, 28672, 8192
    x, w, dy = synth.linear_inputs("c4", M4, N4, K4, seed=0)
    bf = torch.bfloat16
    X, W, G = (torch.from_numpy(a).to(bf).cuda() for a in (x, w, dy))
    plan = ops.LinearPlan(M4, N4, K4, recipe="mxfp8", out_dtype=bf)
    saved = plan.new_saved()
    Y = plan.forward(X, W, saved)
    torch.cuda.synchronize()
    pr_m, pr_n, pc_k, pc_n = _sample(M4, 64, 21), _sample(N4, 64, 22), _sample(K4, 64, 23), _sample(N4, 64, 24)
    fb = plan.buffers(saved)
    assert not fb["bwd_transposed"]
    f_sx, f_sw = _unblock(fb["x_fwd_scale"], M4, K4), _unblock(fb["w_fwd_scale"], N4, K4)
    f_xrows = _cpu(fb["x_fwd"][torch.from_numpy(pr_m).cuda()])
    f_wrows = _cpu(fb["w_fwd"][torch.from_numpy(pr_n).cuda()])
    DX, DW = plan.backward(G, saved)
    torch.cuda.synchronize()
    bb = plan.buffers(saved)
    ic_k, ic_n = torch.from_numpy(pc_k).cuda(), torch.from_numpy(pc_n).cuda()

    _eq_bits("X E8M0 dim0", f_sx, _mx_codes_dim0(x, E4M3))
    _eq_bits("W E8M0 dim0", f_sw, _mx_codes_dim0(w, E4M3))
    _eq_bits("dY E8M0 dim0", _unblock(bb["dy_dx_scale"], M4, N4), _mx_codes_dim0(dy, E5M2))
    _eq_bits("X E8M0 dim1 (saved)", _unblock(bb["x_bwd_scale"], K4, M4), _mx_codes_dim1(x, E4M3))
    _eq_bits("W E8M0 dim1 (saved)", _unblock(bb["w_bwd_scale"], K4, N4), _mx_codes_dim1(w, E4M3))
    _eq_bits("dY E8M0 dim1", _unblock(bb["dy_dw_scale"], N4, M4), _mx_codes_dim1(dy, E5M2))

    _eq_bits("X dim0 rows", f_xrows, omx.quantize_dim0(x[pr_m], E4M3)[0])
    _eq_bits("W dim0 rows", f_wrows, omx.quantize_dim0(w[pr_n], E4M3)[0])
    _eq_bits("dY dim0 rows", _cpu(bb["dy_dx"][torch.from_numpy(pr_m).cuda()]), omx.quantize_dim0(dy[pr_m], E5M2)[0])
    _eq_bits("X dim1 cols (saved)", _cpu(bb["x_bwd"][:, ic_k]).T, omx.quantize_dim1(x[:, pc_k], E4M3)[0])
    _eq_bits("W dim1 cols (saved)", _cpu(bb["w_bwd"][:, ic_k]).T, omx.quantize_dim1(w[:, pc_k], E4M3)[0])
    _eq_bits("dY dim1 cols", _cpu(bb["dy_dw"][:, ic_n]).T, omx.quantize_dim1(dy[:, pc_n], E5M2)[0])

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


@pytest.mark.parametrize("cfg,recipe,shape", [("c2", "tensorwise", (16384, 14336, 4096)),
                                              ("c3", "rowwise", (16384, 14336, 4096)),
                                              ("c3", "rowwise", (16384, 4096, 14336)),
                                              ("c4", "mxfp8", (16384, 28672, 8192))],
                         ids=["c2-tensorwise", "c3w1-rowwise", "c3w2-rowwise", "c4-mxfp8"])
def test_fullsize_power_of_two_invariance(cfg, recipe, shape):
    """A property that holds at any size ("linearity in scales"; R-c3): scaling X by 2^3 scales
    every amax over X by 8, every scale by 1/8 exactly (E8M0 codes by +3), and leaves every FP8 code of X
    unchanged, so Y' = 8 Y, dX' = dX and dW' = 8 dW bit for bit (power-of-two factors are exact in fp32 and
    bf16).  Checked over the FULL bench-size tensors and outputs, on the linear's own buffers.  MX: blocks
    whose code is clamped (0 for the bf16-subnormal blocks of the c4 recipe, or > 251) are excluded from the
    code check and Y is compared only on rows without a clamped nonzero block (all-zero blocks are fine)."""
    from paper_2507_16099_b200 import ops
    M, N, K = shape
    from synth import device as sd
    X = sd.tensor(cfg, "x", (M, K), 0, "cuda")
    W = sd.tensor(cfg, "w", (N, K), 0, "cuda")
    G = sd.tensor(cfg, "dy", (M, N), 0, "cuda")
    X8 = X * 8   # exact in bf16 (exponent + 3; the recipes stay far below the bf16 maximum)
    plan = ops.LinearPlan(M, N, K, recipe=recipe, out_dtype=torch.bfloat16)
    runs = []
    for x in (X, X8):
        saved = plan.new_saved()
        Y = plan.forward(x, W, saved)
        torch.cuda.synchronize()
        fb = {k: (v.clone() if torch.is_tensor(v) else v) for k, v in plan.buffers(saved).items()}
        DX, DW = plan.backward(G, saved)
        torch.cuda.synchronize()
        runs.append((Y, DX, DW, fb, {k: (v.clone() if torch.is_tensor(v) else v) for k, v in plan.buffers(saved).items()}))
    (Y, DX, DW, fb, bb), (Y8, DX8, DW8, fb8, bb8) = runs
    if recipe != "mxfp8":
        assert torch.equal(fb["x_fwd"], fb8["x_fwd"]) and torch.equal(bb["x_bwd"], bb8["x_bwd"])
        for k_ in ("x_fwd_scale", "x_bwd_scale"):
            assert torch.equal(fb[k_] if k_ == "x_fwd_scale" else bb[k_], 8 * (fb8[k_] if k_ == "x_fwd_scale" else bb8[k_]))
        assert torch.equal(Y8.float(), 8 * Y.float())
        assert torch.equal(DX8, DX)
        assert torch.equal(DW8.float(), 8 * DW.float())
        return
    # MXFP8: E8M0 codes of X (dim0 along K, dim1 along M) shift by +3 wherever not clamped, element codes kept
    for key_q, key_s in (("x_fwd", "x_fwd_scale"),):
        s0 = fb[key_s].to(torch.int32)
        s1 = fb8[key_s].to(torch.int32)
        ok = (s0 >= 1) & (s0 <= 251)
        assert torch.equal(s1[ok], s0[ok] + 3)
    s0b = bb["x_bwd_scale"].to(torch.int32)
    s1b = bb8["x_bwd_scale"].to(torch.int32)
    okb = (s0b >= 1) & (s0b <= 251)
    assert torch.equal(s1b[okb], s0b[okb] + 3)
    # rows of X whose dim0 blocks are all unclamped: their codes match and Y' = 8 Y exactly there
    # (the blocked E8M0 layout is a permutation; compare through the logical [M, K/32] view)
    def unblock(buf, R, C):
        C32 = C // 32
        return buf.view(R // 128, C32 // 4, 32, 4, 4).permute(0, 3, 2, 1, 4).reshape(R, C32)
    c0 = unblock(fb["x_fwd_scale"], M, K).to(torch.int32)
    zero_blk = (X.view(M, K // 32, 32) == 0).all(dim=2)          # all-zero blocks contribute 0 either way
    good_rows = (((c0 >= 1) & (c0 <= 251)) | zero_blk).all(dim=1)
    assert int(good_rows.sum()) > M // 2
    assert torch.equal(fb["x_fwd"][good_rows], fb8["x_fwd"][good_rows])
    assert torch.equal(Y8[good_rows].float(), 8 * Y[good_rows].float())
    assert torch.equal(DX8, DX)
