"""Scaled grouped GEMM for MoE training ("scaled_grouped_mm: differentiable
scaled grouped GEMM for MoE FP8 training"), per group the Float8Linear recipe of
``oracle.linear``.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Layout (reading R-c22): tokens routed to experts are stored contiguously by
expert, X [T,K] and dY [T,N]; offs[0] = 0 <= offs[1] <= ... <= offs[E] = T; expert g
owns rows [offs[g], offs[g+1]); the expert weights are stacked W [E*N, K] (nn.Linear
layout per expert, W_g = W[g*N:(g+1)*N]).  Then for every expert g

    Y_g  = X_g W_g^T          dX_g = dY_g W_g          dW_g = dY_g^T X_g

with exactly the casts of ``oracle.linear`` applied to (X_g, W_g, dY_g): the scaling
units never cross an expert (tensorwise: one scale for the whole X, W, dY as in the
non-grouped recipe; rowwise: per token row over K / N, per expert weight row over K,
per expert weight column over N, per (expert, column) over the expert's tokens).  An
expert with no tokens contributes no rows and dW_g = 0.

The oracle follows that definition literally: a loop over experts calling the
single-linear recipe on the slices.  For tensorwise the scales are global (the paper's
tensorwise recipe scales each tensor as a whole), so the slices are cast with the
full tensors' scales.
"""

import numpy as np

from . import fp8, gemm, linear
from .codecs import E4M3, E5M2


def _groups(offs):
    offs = [int(o) for o in offs]
    return list(zip(offs[:-1], offs[1:]))


def forward(x, w, offs, recipe, fmt_fwd=E4M3):
    """Returns (y fp64 [T,N], bound [T,N])."""
    x = np.asarray(x, np.float32)
    w = np.asarray(w, np.float32)
    E = len(offs) - 1
    N = w.shape[0] // E
    y = np.zeros((x.shape[0], N))
    bd = np.zeros_like(y)
    if recipe == linear.TENSORWISE:
        xq, sx, _ = fp8.cast_tensorwise(x, fmt_fwd)
        wq, sw, _ = fp8.cast_tensorwise(w, fmt_fwd)
    for g, (a, b) in enumerate(_groups(offs)):
        if a == b:
            continue
        wg = w[g * N:(g + 1) * N]
        if recipe == linear.TENSORWISE:
            xg, wgq = xq[a:b], wq[g * N:(g + 1) * N]
            y[a:b] = gemm.gemm_ref(xg, fmt_fwd, sx, wgq, fmt_fwd, sw)
            bd[a:b] = gemm.abs_bound(xg, fmt_fwd, sx, wgq, fmt_fwd, sw)
        else:
            y[a:b], bd[a:b], _ = linear.forward(x[a:b], wg, recipe, fmt_fwd)
    return y, bd


def backward(x, w, dy, offs, recipe, fmt_fwd=E4M3, fmt_grad=E5M2):
    """Returns (dx fp64 [T,K], dx_bound, dw fp64 [E*N,K], dw_bound)."""
    x = np.asarray(x, np.float32)
    w = np.asarray(w, np.float32)
    dy = np.asarray(dy, np.float32)
    E = len(offs) - 1
    N = w.shape[0] // E
    dx = np.zeros(x.shape)
    dxb = np.zeros_like(dx)
    dw = np.zeros(w.shape)
    dwb = np.zeros_like(dw)
    if recipe == linear.TENSORWISE:
        xq, sx, _ = fp8.cast_tensorwise(x, fmt_fwd)
        wq, sw, _ = fp8.cast_tensorwise(w, fmt_fwd)
        gq, sg, _ = fp8.cast_tensorwise(dy, fmt_grad)
    for g, (a, b) in enumerate(_groups(offs)):
        if a == b:
            continue
        r = slice(g * N, (g + 1) * N)
        if recipe == linear.TENSORWISE:
            dx[a:b] = gemm.gemm_ref(gq[a:b], fmt_grad, sg, wq[r].T, fmt_fwd, sw)
            dxb[a:b] = gemm.abs_bound(gq[a:b], fmt_grad, sg, wq[r].T, fmt_fwd, sw)
            dw[r] = gemm.gemm_ref(gq[a:b].T, fmt_grad, sg, xq[a:b].T, fmt_fwd, sx)
            dwb[r] = gemm.abs_bound(gq[a:b].T, fmt_grad, sg, xq[a:b].T, fmt_fwd, sx)
        else:
            dx[a:b], dxb[a:b], dw[r], dwb[r], _ = linear.backward(x[a:b], w[r], dy[a:b], recipe, fmt_fwd,
                                                                   fmt_grad)
    return dx, dxb, dw, dwb


def column_scales(v, offs, fmt):
    """Per (group, column) scales over each group's rows (the rowwise dW operands' scaling unit):
    float32 [G, C]; empty groups get the zero-amax scale."""
    v = np.asarray(v, np.float32)
    out = []
    for a, b in _groups(offs):
        am = fp8.amax(v[a:b], 0) if b > a else np.zeros(v.shape[1], np.float32)
        out.append(fp8.scale_from_amax(am, fmt))
    return np.stack(out)
