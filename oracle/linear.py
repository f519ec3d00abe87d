"""Float8Linear forward / backward references, per recipe.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Notation: X [M,K] activations, W [N,K] weight (nn.Linear layout),
dY [M,N] output gradient.  Y = X W^T; dX = dY W; dW = dY^T X.

Operand plan (Appendix A, P:596-597 -- "rows of the left GEMM operand,
columns of the right"):

  GEMM          contraction  tensorwise        rowwise                              MXFP8 (block axis)
  Y  = X W^T    K            X:1, W:1          X per row m, W per row n (over K)     X dim0, W dim0
  dX = dY W     N            dY:1, W reuse     dY per row m, W per col k (over N)    dY dim0, W dim1
  dW = dY^T X   M            dY, X reuse       dY per col n, X per col k (over M)    dY dim1, X dim1

Formats: e4m3 for X/W, e5m2 for dY by default for every recipe (north star,
SURVEY §8c.8, c.14); both selectable.

Each function returns the fp64 results plus every intermediate the GPU path
must reproduce bit-exactly (codes and scales), keyed by name.
"""

import numpy as np

from . import fp8, mx, gemm
from .codecs import E4M3, E5M2

TENSORWISE = "tensorwise"
ROWWISE = "rowwise"
MXFP8 = "mxfp8"
ROWWISE_GW_HP = "rowwise_gw_hp"


def forward(x, w, recipe, fmt_fwd=E4M3, mx_mode=mx.FLOOR):
    """Y = X W^T with the recipe's casts.  Returns (y fp64 [M,N], bound, saved dict)."""
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    if recipe == TENSORWISE:
        xq, sx, ax = fp8.cast_tensorwise(x, fmt_fwd)
        wq, sw, aw = fp8.cast_tensorwise(w, fmt_fwd)
        y = gemm.gemm_ref(xq, fmt_fwd, sx, wq, fmt_fwd, sw)
        bd = gemm.abs_bound(xq, fmt_fwd, sx, wq, fmt_fwd, sw)
        saved = dict(xq=xq, sx=sx, amax_x=ax, wq=wq, sw=sw, amax_w=aw)
    elif recipe in (ROWWISE, ROWWISE_GW_HP):
        xq, sx, ax = fp8.cast_rowwise(x, fmt_fwd)
        wq, sw, aw = fp8.cast_rowwise(w, fmt_fwd)
        y = gemm.gemm_ref(xq, fmt_fwd, sx, wq, fmt_fwd, sw)
        bd = gemm.abs_bound(xq, fmt_fwd, sx, wq, fmt_fwd, sw)
        saved = dict(xq=xq, sx=sx, amax_x=ax, wq=wq, sw=sw, amax_w=aw)
    elif recipe == MXFP8:
        xq, xsc = mx.quantize_dim0(x, fmt_fwd, mx_mode)
        wq, wsc = mx.quantize_dim0(w, fmt_fwd, mx_mode)
        y = gemm.mx_gemm_ref(xq, xsc, fmt_fwd, wq, wsc, fmt_fwd)
        bd = gemm.mx_abs_bound(xq, xsc, fmt_fwd, wq, wsc, fmt_fwd)
        saved = dict(xq=xq, xsc=xsc, wq=wq, wsc=wsc)
    else:
        raise ValueError(recipe)
    return y, bd, saved


def backward(x, w, dy, recipe, fmt_fwd=E4M3, fmt_grad=E5M2, mx_mode=mx.FLOOR):
    """dX = dY W and dW = dY^T X with the recipe's casts.

    Returns (dx fp64 [M,K], dx_bound, dw fp64 [N,K], dw_bound, casts dict).
    """
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    dy = np.asarray(dy, dtype=np.float32)
    if recipe == TENSORWISE:
        xq, sx, _ = fp8.cast_tensorwise(x, fmt_fwd)
        wq, sw, _ = fp8.cast_tensorwise(w, fmt_fwd)
        gq, sg, ag = fp8.cast_tensorwise(dy, fmt_grad)
        # dX[m,k] = sum_n dY[m,n] W[n,k]: left = dYq [M,N], right (K-major over N) = Wq^T [K,N]
        dx = gemm.gemm_ref(gq, fmt_grad, sg, wq.T, fmt_fwd, sw)
        dxb = gemm.abs_bound(gq, fmt_grad, sg, wq.T, fmt_fwd, sw)
        # dW[n,k] = sum_m dY[m,n] X[m,k]: left = dYq^T [N,M], right = Xq^T [K,M]
        dw = gemm.gemm_ref(gq.T, fmt_grad, sg, xq.T, fmt_fwd, sx)
        dwb = gemm.abs_bound(gq.T, fmt_grad, sg, xq.T, fmt_fwd, sx)
        casts = dict(gq=gq, sg=sg, amax_g=ag)
    elif recipe == ROWWISE:
        g_r, sg_r, _ = fp8.cast_rowwise(dy, fmt_grad)      # dY per row m (over N)
        w_c, sw_c, _ = fp8.cast_colwise(w, fmt_fwd)        # W per column k (over N)
        dx = gemm.gemm_ref(g_r, fmt_grad, sg_r, w_c.T, fmt_fwd, sw_c)
        dxb = gemm.abs_bound(g_r, fmt_grad, sg_r, w_c.T, fmt_fwd, sw_c)
        g_c, sg_c, _ = fp8.cast_colwise(dy, fmt_grad)      # dY per column n (over M)
        x_c, sx_c, _ = fp8.cast_colwise(x, fmt_fwd)        # X per column k (over M)
        dw = gemm.gemm_ref(g_c.T, fmt_grad, sg_c, x_c.T, fmt_fwd, sx_c)
        dwb = gemm.abs_bound(g_c.T, fmt_grad, sg_c, x_c.T, fmt_fwd, sx_c)
        casts = dict(g_r=g_r, sg_r=sg_r, w_c=w_c, sw_c=sw_c, g_c=g_c, sg_c=sg_c, x_c=x_c, sx_c=sx_c)
    elif recipe == ROWWISE_GW_HP:
        # Appendix A: "like rowwise but it keeps the dL/dW computation in bfloat16";
        # grad_weight = gemm_ref(grad_out^T, x) with no FP8 casting.
        g_r, sg_r, _ = fp8.cast_rowwise(dy, fmt_grad)
        w_c, sw_c, _ = fp8.cast_colwise(w, fmt_fwd)
        dx = gemm.gemm_ref(g_r, fmt_grad, sg_r, w_c.T, fmt_fwd, sw_c)
        dxb = gemm.abs_bound(g_r, fmt_grad, sg_r, w_c.T, fmt_fwd, sw_c)
        G = dy.astype(np.float64)
        X = x.astype(np.float64)
        dw = G.T @ X
        dwb = np.abs(G).T @ np.abs(X)
        casts = dict(g_r=g_r, sg_r=sg_r, w_c=w_c, sw_c=sw_c)
    elif recipe == MXFP8:
        g0, g0s = mx.quantize_dim0(dy, fmt_grad, mx_mode)   # dY along N  -> [M,N]
        w1, w1s = mx.quantize_dim1(w, fmt_fwd, mx_mode)     # W along N   -> [K,N]
        dx = gemm.mx_gemm_ref(g0, g0s, fmt_grad, w1, w1s, fmt_fwd)
        dxb = gemm.mx_abs_bound(g0, g0s, fmt_grad, w1, w1s, fmt_fwd)
        g1, g1s = mx.quantize_dim1(dy, fmt_grad, mx_mode)   # dY along M  -> [N,M]
        x1, x1s = mx.quantize_dim1(x, fmt_fwd, mx_mode)     # X along M   -> [K,M]
        dw = gemm.mx_gemm_ref(g1, g1s, fmt_grad, x1, x1s, fmt_fwd)
        dwb = gemm.mx_abs_bound(g1, g1s, fmt_grad, x1, x1s, fmt_fwd)
        casts = dict(g0=g0, g0s=g0s, w1=w1, w1s=w1s, g1=g1, g1s=g1s, x1=x1, x1s=x1s)
    else:
        raise ValueError(recipe)
    return dx, dxb, dw, dwb, casts
