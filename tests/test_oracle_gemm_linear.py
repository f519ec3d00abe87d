"""Pins for oracle/gemm.py, oracle/linear.py and oracle/fsdp.py.

* gemm_ref / mx_gemm_ref vs exact-rational (fractions.Fraction) triple-loop brute force
  on tiny inputs, tensorwise and rowwise scale vectors
* identity and zero operands
* integer-grid operands: the scaled product equals the exact integer matmul of the
  original values (scales are powers of two)
* linear: grad_out = 0 -> zero grads under every recipe; recipe agreement on
  lossless unit-scale grids, equal to the exact X W^T / dY W / dY^T X
* FSDP: gathered shard casts with the global amax == unsharded tensorwise cast
"""

from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import codecs, fp8, fsdp, gemm, linear, mx
from oracle.codecs import E4M3, E5M2


def _frac_gemm(A, B, sa, sb):
    M, K = A.shape
    N = B.shape[0]
    out = np.zeros((M, N))
    for m in range(M):
        for n in range(N):
            acc = Fraction(0)
            for k in range(K):
                acc += Fraction(float(A[m, k])) * Fraction(float(B[n, k]))
            out[m, n] = float(acc / (Fraction(float(sa[m])) * Fraction(float(sb[n]))))
    return out


@pytest.mark.parametrize("fa,fb", [(E4M3, E4M3), (E5M2, E4M3), (E4M3, E5M2)])
def test_gemm_ref_vs_fraction(fa, fb):
    rng = np.random.default_rng(0)
    M, N, K = 5, 7, 9
    a = rng.integers(0, 256, (M, K)).astype(np.uint8)
    b = rng.integers(0, 256, (N, K)).astype(np.uint8)
    a[(a & 0x7F) >= (0x7F if fa == E4M3 else 0x7C)] = 0x11   # finite codes only
    b[(b & 0x7F) >= (0x7F if fb == E4M3 else 0x7C)] = 0x22
    sa = (rng.uniform(0.1, 100, M)).astype(np.float32)
    sb = (rng.uniform(0.1, 100, N)).astype(np.float32)
    got = gemm.gemm_ref(a, fa, sa, b, fb, sb)
    want = _frac_gemm(codecs.decode(a, fa), codecs.decode(b, fb), sa, sb)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-300)
    # scalar scales broadcast identically
    got_t = gemm.gemm_ref(a, fa, sa[0], b, fb, sb[0])
    want_t = _frac_gemm(codecs.decode(a, fa), codecs.decode(b, fb), np.full(M, sa[0]), np.full(N, sb[0]))
    np.testing.assert_allclose(got_t, want_t, rtol=1e-13)


def test_mx_gemm_vs_fraction():
    rng = np.random.default_rng(1)
    M, N, K = 3, 4, 64
    a = rng.integers(0, 0x7E, (M, K)).astype(np.uint8) | (rng.integers(0, 2, (M, K)) << 7).astype(np.uint8)
    b = rng.integers(0, 0x7B, (N, K)).astype(np.uint8)
    asc = rng.integers(100, 150, (M, 2)).astype(np.uint8)
    bsc = rng.integers(100, 150, (N, 2)).astype(np.uint8)
    got = gemm.mx_gemm_ref(a, asc, E4M3, b, bsc, E5M2)
    A = codecs.decode(a, E4M3)
    B = codecs.decode(b, E5M2)
    for m in range(M):
        for n in range(N):
            acc = Fraction(0)
            for k in range(K):
                acc += (Fraction(float(A[m, k])) * Fraction(2) ** (int(asc[m, k // 32]) - 127)
                        * Fraction(float(B[n, k])) * Fraction(2) ** (int(bsc[n, k // 32]) - 127))
            assert abs(got[m, n] - float(acc)) <= 1e-13 * abs(float(acc)) + 1e-300


def test_identity_and_zero():
    one = 0x38  # e4m3 1.0
    I = np.where(np.eye(16, dtype=bool), one, 0).astype(np.uint8)
    rng = np.random.default_rng(2)
    b = rng.integers(0, 0x7E, (16, 16)).astype(np.uint8)
    y = gemm.gemm_ref(I, E4M3, np.float32(1), b, E4M3, np.float32(1))
    assert np.array_equal(y, codecs.decode(b, E4M3).T)
    z = gemm.gemm_ref(np.zeros((4, 16), np.uint8), E4M3, np.float32(3), b, E4M3, np.float32(1))
    assert np.all(z == 0)


def test_integer_grid_exact():
    # App. A.12: e4m3 values in {-14..14} with amax 14 -> s = 32 lossless; e5m2 values on
    # {0, +-1..8, +-10, +-12, +-14} with amax 14 -> s = 4096 lossless.  y must equal X W^T exactly.
    vals4 = np.arange(-14, 15)
    vals5 = np.array([0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14, -1, -2, -3, -4, -5, -6, -7, -8, -10, -12, -14])
    x = synth.integer_grid(synth.stream_key("t", "gx"), (48, 160), vals4)
    w = synth.integer_grid(synth.stream_key("t", "gw"), (40, 160), vals4)
    g = synth.integer_grid(synth.stream_key("t", "gg"), (48, 40), vals5)
    x[0, 0] = w[0, 0] = g[0, 0] = 14.0
    xq, sx, _ = fp8.cast_tensorwise(x, E4M3)
    wq, sw, _ = fp8.cast_tensorwise(w, E4M3)
    gq, sg, _ = fp8.cast_tensorwise(g, E5M2)
    assert sx == 32 and sw == 32 and sg == 4096
    X, W, G = (a.astype(np.int64) for a in (x, w, g))
    assert np.array_equal(gemm.gemm_ref(xq, E4M3, sx, wq, E4M3, sw), (X @ W.T).astype(np.float64))
    dx, _, dw, _, _ = linear.backward(x, w, g, linear.TENSORWISE)
    assert np.array_equal(dx, (G @ W).astype(np.float64))
    assert np.array_equal(dw, (G.T @ X).astype(np.float64))


@pytest.mark.parametrize("recipe", [linear.TENSORWISE, linear.ROWWISE, linear.MXFP8])
def test_zero_grad_out_gives_zero_grads(recipe):
    x, w, _ = synth.linear_inputs("c2", 64, 96, 128, seed=0)
    dy = np.zeros((64, 96), np.float32)
    dx, _, dw, _, _ = linear.backward(x, w, dy, recipe)
    assert np.all(dx == 0) and np.all(dw == 0)


def _lossless_grid(rng, shape, fmt, fill):
    grid = codecs.decode(np.arange(0x80), fmt)
    grid = grid[np.isfinite(grid) & (grid <= codecs.FMAX[fmt])]
    x = rng.choice(grid, size=shape) * rng.choice([-1.0, 1.0], size=shape)
    # every row and every column (and every 32-block both ways) holds fmax -> all scales 1
    x[np.arange(shape[0]), (np.arange(shape[0]) * 32) % shape[1]] = fill
    for c in range(shape[1]):
        for r0 in range(0, shape[0], 32):
            x[r0 + (c % 32), c] = fill
    for r in range(shape[0]):
        for c0 in range(0, shape[1], 32):
            x[r, c0 + (r % 32)] = fill
    return x.astype(np.float32)


def test_recipe_agreement_on_unit_scale_grid():
    rng = np.random.default_rng(3)
    M, N, K = 64, 64, 96
    x = _lossless_grid(rng, (M, K), E4M3, 448.0)
    w = _lossless_grid(rng, (N, K), E4M3, 448.0)
    dy = _lossless_grid(rng, (M, N), E5M2, 57344.0)
    exact_y = x.astype(np.float64) @ w.astype(np.float64).T
    exact_dx = dy.astype(np.float64) @ w.astype(np.float64)
    exact_dw = dy.astype(np.float64).T @ x.astype(np.float64)
    for recipe in (linear.TENSORWISE, linear.ROWWISE, linear.MXFP8):
        y, _, _ = linear.forward(x, w, recipe)
        dx, _, dw, _, _ = linear.backward(x, w, dy, recipe)
        assert np.array_equal(y, exact_y), recipe
        assert np.array_equal(dx, exact_dx), recipe
        assert np.array_equal(dw, exact_dw), recipe


def test_linear_close_to_high_precision():
    # The FP8 linear approximates the exact linear to within FP8 resolution.
    x, w, dy = synth.linear_inputs("c2", 128, 96, 160, seed=1)
    X, W, G = (a.astype(np.float64) for a in (x, w, dy))
    for recipe in (linear.TENSORWISE, linear.ROWWISE, linear.MXFP8):
        y, _, _ = linear.forward(x, w, recipe)
        dx, _, dw, _, _ = linear.backward(x, w, dy, recipe)
        for got, ref in ((y, X @ W.T), (dx, G @ W), (dw, G.T @ X)):
            rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert rel < 0.15, (recipe, rel)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_fsdp_gather_equals_unsharded_cast(P):
    w = synth.tensor_c2("w", (64, 48), seed=0)
    w[13, 7] = 0.9  # the global amax lives on one shard only
    shards = np.split(w, P, axis=0)
    q, s, a = fsdp.allgather_ref(shards, E4M3)
    q1, s1, a1 = fp8.cast_tensorwise(w, E4M3)
    assert np.array_equal(q, q1) and s == s1 and a == a1


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("fmt,mode", [(E4M3, mx.FLOOR), (E5M2, mx.RCEIL)])
def test_fsdp_mx_gather_equals_unsharded_quantize(P, fmt, mode):
    # MX scales are shard-local, so per-shard quantization + concatenation equals
    # the unsharded dim0 / dim1 quantization (no amax exchange), when shards hold whole 32-blocks
    w = synth.tensor_c4("w", (256, 128), seed=1)
    q0, s0, q1, s1 = fsdp.allgather_mx_ref(np.split(w, P, axis=0), fmt, mode)
    f0, g0 = mx.quantize_dim0(w, fmt, mode)
    f1, g1 = mx.quantize_dim1(w, fmt, mode)
    assert np.array_equal(q0, f0) and np.array_equal(s0, g0)
    assert np.array_equal(q1, f1) and np.array_equal(s1, g1)


def test_fsdp_mx_gather_needs_block_aligned_shards():
    # the alignment rule is load-bearing: 16-row shards split dim1 blocks, and a block whose
    # amax sits in one half gets a different (smaller) code in the other half
    w = synth.tensor_c2("w", (64, 32), seed=2)
    w[3, 5] = 7.0
    full = mx.quantize_dim1(w, E4M3)[1][5, 0]          # block rows 0..31 of column 5
    half = mx.scale_code(np.array([[np.max(np.abs(w[16:32, 5]))]], np.float32), E4M3)[0, 0]
    assert full == mx.scale_code(np.array([[np.float32(7.0)]]), E4M3)[0, 0] and half < full


def test_rowwise_gw_hp_weight_grad_is_high_precision():
    # S:300-301 "RowwiseGwHp grad_weight = gemm_ref(grad_out^T, x) bit-exactly" (no FP8 casting);
    # its grad_input equals the rowwise recipe's (same casts, "like rowwise").
    x, w, dy = synth.linear_inputs("c3", 48, 40, 64, seed=2)
    dx_r, _, _, _, _ = linear.backward(x, w, dy, linear.ROWWISE)
    dx_h, _, dw_h, _, _ = linear.backward(x, w, dy, linear.ROWWISE_GW_HP)
    assert np.array_equal(dx_h, dx_r)
    want = _frac_gemm(dy.T, x.T, np.ones(40, np.float32), np.ones(64, np.float32))
    np.testing.assert_allclose(dw_h, want, rtol=1e-12)


# ---------------------------------------------------------------- tolerance-scale pins
# abs_bound / mx_abs_bound set the scale of every random-data GEMM verdict
# (|err| <= 1e-2 * sum_k |a||b|, BASELINE.json north_star), so they are pinned
# against things other than themselves: an exact-rational brute force over the
# ml_dtypes decoders (not oracle.codecs), the invariants bound >= |y| with
# equality for non-negative operands, the exact 1/(s_a s_b) scaling, and the
# high-precision product sum_k |x||w| of the unquantised inputs.

def _ml_decode(codes, fmt):
    import ml_dtypes
    dt = ml_dtypes.float8_e4m3fn if fmt == E4M3 else ml_dtypes.float8_e5m2
    return np.asarray(codes, np.uint8).view(dt).astype(np.float64)


def _frac_abs(A, B, sa, sb):
    M, K = A.shape
    N = B.shape[0]
    out = np.zeros((M, N))
    for m in range(M):
        for n in range(N):
            acc = Fraction(0)
            for k in range(K):
                acc += abs(Fraction(float(A[m, k]))) * abs(Fraction(float(B[n, k])))
            out[m, n] = float(acc / (Fraction(float(sa[m])) * Fraction(float(sb[n]))))
    return out


def _finite_codes(rng, shape, fmt):
    c = rng.integers(0, 256, shape).astype(np.uint8)
    c[(c & 0x7F) >= (0x7F if fmt == E4M3 else 0x7C)] = 0x91   # finite, negative
    return c


@pytest.mark.parametrize("fa,fb", [(E4M3, E4M3), (E5M2, E4M3), (E4M3, E5M2)])
def test_abs_bound_vs_fraction(fa, fb):
    rng = np.random.default_rng(11)
    M, N, K = 4, 6, 11
    a, b = _finite_codes(rng, (M, K), fa), _finite_codes(rng, (N, K), fb)
    sa = rng.uniform(0.01, 3000, M).astype(np.float32)
    sb = rng.uniform(0.01, 3000, N).astype(np.float32)
    want = _frac_abs(_ml_decode(a, fa), _ml_decode(b, fb), sa, sb)
    np.testing.assert_allclose(gemm.abs_bound(a, fa, sa, b, fb, sb), want, rtol=1e-13, atol=1e-300)
    want_t = _frac_abs(_ml_decode(a, fa), _ml_decode(b, fb), np.full(M, sa[1]), np.full(N, sb[2]))
    np.testing.assert_allclose(gemm.abs_bound(a, fa, sa[1], b, fb, sb[2]), want_t, rtol=1e-13, atol=1e-300)


def test_mx_abs_bound_vs_fraction():
    rng = np.random.default_rng(12)
    M, N, K = 3, 5, 64
    a, b = _finite_codes(rng, (M, K), E4M3), _finite_codes(rng, (N, K), E5M2)
    asc = rng.integers(90, 160, (M, K // 32)).astype(np.uint8)
    bsc = rng.integers(90, 160, (N, K // 32)).astype(np.uint8)
    A, B = _ml_decode(a, E4M3), _ml_decode(b, E5M2)
    got = gemm.mx_abs_bound(a, asc, E4M3, b, bsc, E5M2)
    for m in range(M):
        for n in range(N):
            acc = Fraction(0)
            for k in range(K):
                acc += (abs(Fraction(float(A[m, k]))) * Fraction(2) ** (int(asc[m, k // 32]) - 127)
                        * abs(Fraction(float(B[n, k]))) * Fraction(2) ** (int(bsc[n, k // 32]) - 127))
            assert abs(got[m, n] - float(acc)) <= 1e-13 * float(acc) + 1e-300


def test_abs_bound_invariants():
    rng = np.random.default_rng(13)
    M, N, K = 24, 20, 96
    a, b = _finite_codes(rng, (M, K), E5M2), _finite_codes(rng, (N, K), E4M3)
    sa = rng.uniform(1, 1e4, M).astype(np.float32)
    sb = rng.uniform(1, 1e4, N).astype(np.float32)
    bd = gemm.abs_bound(a, E5M2, sa, b, E4M3, sb)
    y = gemm.gemm_ref(a, E5M2, sa, b, E4M3, sb)
    assert np.all(bd >= np.abs(y) * (1 - 1e-15))
    assert np.any(bd > 2 * np.abs(y))                       # mixed signs: the bound is not |y|
    # non-negative operands: bound == y exactly (same products, no cancellation)
    ap, bp = a & 0x7F, b & 0x7F
    np.testing.assert_array_equal(gemm.abs_bound(ap, E5M2, sa, bp, E4M3, sb),
                                  gemm.gemm_ref(ap, E5M2, sa, bp, E4M3, sb))
    # sign flips of operands do not move the bound
    np.testing.assert_array_equal(gemm.abs_bound(a ^ 0x80, E5M2, sa, b, E4M3, sb), bd)
    # exact 1/(s_a s_b) scaling: doubling a scale halves the bound (powers of two are exact)
    np.testing.assert_array_equal(gemm.abs_bound(a, E5M2, sa * 2, b, E4M3, sb), bd / 2)
    np.testing.assert_array_equal(gemm.abs_bound(a, E5M2, sa, b, E4M3, sb * 4), bd / 4)
    # mx: code +1 on one operand's block doubles that block's share only
    asc = rng.integers(110, 140, (M, K // 32)).astype(np.uint8)
    bsc = rng.integers(110, 140, (N, K // 32)).astype(np.uint8)
    mb = gemm.mx_abs_bound(a, asc, E5M2, b, bsc, E4M3)
    assert np.all(mb >= np.abs(gemm.mx_gemm_ref(a, asc, E5M2, b, bsc, E4M3)) * (1 - 1e-15))
    np.testing.assert_array_equal(gemm.mx_abs_bound(a, asc + 1, E5M2, b, bsc, E4M3), 2 * mb)


@pytest.mark.parametrize("recipe", [linear.TENSORWISE, linear.ROWWISE, linear.MXFP8])
def test_linear_bounds_track_unquantised_product(recipe):
    """The bound of each linear GEMM is sum_k |dec(a)/s_a||dec(b)/s_b|, i.e. the absolute
    product of the DEQUANTISED operands, which are the hp inputs up to one FP8 rounding each
    (relative error <= 2^-4 e4m3, 2^-3 e5m2, for normal values).  So it must sit within
    [(1-2^-4)(1-2^-3), (1+2^-4)(1+2^-3)] of sum_k |x||w| of the hp inputs.  A dropped or
    inverted 1/(s_a s_b) factor moves it by s_a s_b (>= 1e2 here)."""
    # unit-variance data keeps every element away from FP8 underflow (exact relative bounds)
    rng = np.random.default_rng(14)
    M, N, K = 64, 96, 128
    x = (rng.standard_normal((M, K)) * 3).astype(np.float32)
    w = (rng.standard_normal((N, K)) * 0.02).astype(np.float32)
    dy = (rng.standard_normal((M, N)) * 1e-3).astype(np.float32)
    x[np.abs(x) < 0.1] = 0.1
    w[np.abs(w) < 2e-3] = 2e-3
    dy[np.abs(dy) < 1e-4] = 1e-4
    _, yb, _ = linear.forward(x, w, recipe)
    _, dxb, _, dwb, _ = linear.backward(x, w, dy, recipe)
    X, W, G = (np.abs(t.astype(np.float64)) for t in (x, w, dy))
    lo, hi = (1 - 2.0 ** -4) * (1 - 2.0 ** -3), (1 + 2.0 ** -4) * (1 + 2.0 ** -3)
    for got, ref in ((yb, X @ W.T), (dxb, G @ W), (dwb, G.T @ X)):
        r = got / ref
        assert lo <= r.min() and r.max() <= hi, (recipe, r.min(), r.max())
