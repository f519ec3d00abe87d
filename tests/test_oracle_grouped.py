"""Pins for oracle.grouped (MoE scaled grouped GEMM; reading R-c22).

Each pin checks the grouped oracle against something other than itself: exact fp64
products on lossless grids, locality of the per-expert scaling units (a plausible bug is
computing a column scale over all tokens instead of the expert's), empty experts,
expert permutation equivariance, and the one-expert case = the plain Float8Linear oracle.
"""

import numpy as np
import pytest

from oracle import codecs, fp8, grouped, linear

E4, E5 = codecs.E4M3, codecs.E5M2


def _lossless(rows_per_group, C, fmt, rng):
    """Values that every scaling unit of the recipes maps losslessly: entries are codes of `fmt`
    whose magnitude fits, and every row, every column and every (group, column) slice holds one
    entry of magnitude fmax, so every scale is exactly 1."""
    fmax = 448.0 if fmt == E4 else 57344.0
    small = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6, 8], np.float64)
    T = sum(rows_per_group)
    v = rng.choice(small, size=(T, C)) * rng.choice([-1, 1], size=(T, C))
    a = 0
    for n in rows_per_group:
        for c in range(C):            # (group, column) slices
            v[a + c % max(n, 1), c] = fmax if n else 0
        for r in range(n):            # rows
            v[a + r, r % C] = -fmax
        a += n
    return v.astype(np.float32)


@pytest.mark.parametrize("recipe", [linear.TENSORWISE, linear.ROWWISE])
def test_grouped_exact_on_lossless_grid(recipe):
    rng = np.random.default_rng(0)
    sizes = [32, 0, 48, 16]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    E, N, K = len(sizes), 16, 24
    x = _lossless(sizes, K, E4, rng)
    w = np.concatenate([_lossless([N], K, E4, rng) for _ in range(E)])
    dy = _lossless(sizes, N, E5, rng)
    for name, v, f in (("x", x, E4), ("w", w, E4), ("dy", dy, E5)):   # the grid really is lossless
        assert np.array_equal(codecs.decode(fp8.cast_tensorwise(v, f)[0], f), v.astype(np.float64)), name
    y, _ = grouped.forward(x, w, offs, recipe)
    dx, _, dw, _ = grouped.backward(x, w, dy, offs, recipe)
    X, W, G = (v.astype(np.float64) for v in (x, w, dy))
    for g, (a, b) in enumerate(zip(offs[:-1], offs[1:])):
        Wg = W[g * N:(g + 1) * N]
        assert np.array_equal(y[a:b], X[a:b] @ Wg.T)
        assert np.array_equal(dx[a:b], G[a:b] @ Wg)
        assert np.array_equal(dw[g * N:(g + 1) * N], G[a:b].T @ X[a:b])


def test_rowwise_scaling_units_stay_inside_an_expert():
    # dW_g must not change when tokens of OTHER experts change (their column amax is not g's)
    rng = np.random.default_rng(1)
    offs = np.array([0, 32, 64, 96])
    N, K = 16, 32
    x = rng.standard_normal((96, K)).astype(np.float32)
    w = rng.standard_normal((3 * N, K)).astype(np.float32) * 0.02
    dy = rng.standard_normal((96, N)).astype(np.float32) * 1e-3
    _, _, dw1, _ = grouped.backward(x, w, dy, offs, linear.ROWWISE)
    x2, dy2 = x.copy(), dy.copy()
    x2[40:60] *= 1000.0          # expert 1's tokens only
    dy2[70:90] *= 1000.0         # expert 2's tokens only
    _, _, dw2, _ = grouped.backward(x2, w, dy2, offs, linear.ROWWISE)
    assert np.array_equal(dw1[:N], dw2[:N])
    assert not np.array_equal(dw1[N:2 * N], dw2[N:2 * N])
    # and the per-(expert, column) scales differ from scales taken over all tokens
    cs = grouped.column_scales(x2, offs, E4)
    assert not np.array_equal(cs[0], fp8.scale_from_amax(fp8.amax(x2, 0), E4))


def test_empty_expert_and_single_expert():
    rng = np.random.default_rng(2)
    N, K = 16, 32
    x = rng.standard_normal((64, K)).astype(np.float32)
    w = rng.standard_normal((2 * N, K)).astype(np.float32)
    dy = rng.standard_normal((64, N)).astype(np.float32)
    for recipe in (linear.TENSORWISE, linear.ROWWISE):
        _, _, dw, _ = grouped.backward(x, w, dy, [0, 0, 64], recipe)
        assert not np.any(dw[:N])
        # one expert == the plain Float8Linear recipe
        y1, _ = grouped.forward(x, w[:N], [0, 64], recipe)
        y2, _, _ = linear.forward(x, w[:N], recipe)
        assert np.array_equal(y1, y2)
        dx1, _, dw1, _ = grouped.backward(x, w[:N], dy, [0, 64], recipe)
        dx2, _, dw2, _, _ = linear.backward(x, w[:N], dy, recipe)
        assert np.array_equal(dx1, dx2) and np.array_equal(dw1, dw2)


def test_expert_permutation_equivariance():
    rng = np.random.default_rng(3)
    sizes = [16, 48, 32]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    N, K = 16, 32
    x = rng.standard_normal((96, K)).astype(np.float32)
    w = rng.standard_normal((3 * N, K)).astype(np.float32)
    dy = rng.standard_normal((96, N)).astype(np.float32)
    perm = [2, 0, 1]
    rows = np.concatenate([np.arange(offs[p], offs[p + 1]) for p in perm])
    wrows = np.concatenate([np.arange(p * N, (p + 1) * N) for p in perm])
    offs_p = np.concatenate([[0], np.cumsum([sizes[p] for p in perm])])
    y, _ = grouped.forward(x, w, offs, linear.ROWWISE)
    dx, _, dw, _ = grouped.backward(x, w, dy, offs, linear.ROWWISE)
    yp, _ = grouped.forward(x[rows], w[wrows], offs_p, linear.ROWWISE)
    dxp, _, dwp, _ = grouped.backward(x[rows], w[wrows], dy[rows], offs_p, linear.ROWWISE)
    assert np.array_equal(yp, y[rows]) and np.array_equal(dxp, dx[rows]) and np.array_equal(dwp, dw[wrows])
