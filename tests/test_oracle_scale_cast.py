"""Pins for oracle/fp8.py (amax, scale, cast) against values and invariants fixed
by the paper/SPEC/mathematics, not by the oracle itself.

* SPEC S:270-272 and SURVEY App. A.5 scale bit patterns (tests/golden/scale.txt)
* SURVEY App. A.6 double-rounding vectors and A.7 convention vector
* invariants: the element at amax always encodes to the max code; scaling x by 2^k
  leaves codes identical and s scales by 2^-k exactly; fp32 division == fp64 division
  rounded once (innocuous double rounding, a theorem for binary32/binary64)
* SPEC S:277-279 / S:307: single-row rowwise == tensorwise; outlier robustness
"""

import numpy as np
import pytest

from oracle import codecs, fp8
from oracle.codecs import E4M3, E5M2


def _f32(bits):
    return np.array([int(bits, 16)], dtype=np.uint32).view(np.float32)[0]


def test_eps_bits():
    assert fp8.EPS.view(np.uint32) == 0x2B8CBCCC


def test_scale_golden(golden):
    for fmt, amax, sbits, _ in golden("scale.txt"):
        s = fp8.scale_from_amax(np.float32(float(amax)), fmt)
        assert int(np.asarray(s).view(np.uint32)) == int(sbits, 16), (fmt, amax, hex(int(np.asarray(s).view(np.uint32))))


def test_scale_fp32_div_equals_fp64_div_rounded():
    rng = np.random.default_rng(3)
    a = (10.0 ** rng.uniform(-12, 38, 200000)).astype(np.float32)
    for fmt in (E4M3, E5M2):
        s32 = fp8.scale_from_amax(a, fmt)
        s64 = (codecs.FMAX[fmt] / np.maximum(a, fp8.EPS).astype(np.float64)).astype(np.float32)
        assert np.array_equal(s32, s64)


def test_cast_double_rounding_vectors(golden):
    for fmt, kind, xb, sb, want, single in golden("cast.txt"):
        if kind == "f32":
            x = _f32(xb)
        else:
            x = np.array([int(xb, 16) << 16], dtype=np.uint32).view(np.float32)[0]
        s = _f32(sb)
        got = int(fp8.cast_scaled(np.float32(x), s, fmt))
        assert got == int(want, 16), (xb, hex(got))
        # the single-rounding (exact product) answer differs: the fixture really tests c4
        exact = np.float64(x) * np.float64(s)
        assert int(codecs.encode(np.float64(exact), fmt)) == int(single, 16)


def test_multiplicative_convention_vector(golden):
    (xb, ab, mul_code, div_code), = golden("convention.txt")
    x, a = _f32(xb), _f32(ab)
    s = fp8.scale_from_amax(a, E4M3)
    assert int(fp8.cast_scaled(x, s, E4M3)) == int(mul_code, 16)
    div = np.float32(x / np.float32(a / np.float32(448.0)))
    assert int(codecs.encode(div, E4M3)) == int(div_code, 16)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_amax_element_maps_to_max_code(fmt):
    rng = np.random.default_rng(5)
    a = (10.0 ** rng.uniform(-11, 37, 300000)).astype(np.float32)
    s = fp8.scale_from_amax(a, fmt)
    q = fp8.cast_scaled(a, s, fmt)
    q_neg = fp8.cast_scaled(-a, s, fmt)
    maxcode = 0x7E if fmt == E4M3 else 0x7B
    assert np.all(q == maxcode) and np.all(q_neg == (maxcode | 0x80))


@pytest.mark.parametrize("k", [-20, -3, 5, 40])
def test_power_of_two_invariance(k):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((64, 96)).astype(np.float32)
    q, s, a = fp8.cast_tensorwise(x, E4M3)
    xk = (x * np.float32(2.0 ** k)).astype(np.float32)
    qk, sk, ak = fp8.cast_tensorwise(xk, E4M3)
    assert np.array_equal(q, qk)
    assert sk == np.float32(s * np.float32(2.0 ** -k))


def test_amax_and_zero_tensor():
    x = np.zeros((4, 8), np.float32)
    q, s, a = fp8.cast_tensorwise(x, E4M3)
    assert a == 0 and np.asarray(s).view(np.uint32) == 0x57CBBA10 and np.all(q == 0)
    x = np.array([[1.0, -3.0], [2.0, 0.5]], np.float32)
    assert fp8.amax(x) == 3.0
    assert np.array_equal(fp8.amax(x, axis=1), np.array([3.0, 2.0], np.float32))
    assert np.array_equal(fp8.amax(x, axis=0), np.array([2.0, 3.0], np.float32))


def test_signed_zero_preserved():
    x = np.array([[-0.0, 0.0, -1e-30, 1.0]], np.float32)
    q, _, _ = fp8.cast_tensorwise(x, E4M3)
    assert list(q[0]) == [0x80, 0x00, 0x80, 0x7E]


def test_single_row_rowwise_equals_tensorwise():
    # S:279 "single-row matrix -> rowwise equals tensorwise bit-exactly"
    rng = np.random.default_rng(2)
    x = rng.standard_normal((1, 300)).astype(np.float32)
    qt, st, _ = fp8.cast_tensorwise(x, E4M3)
    qr, sr, _ = fp8.cast_rowwise(x, E4M3)
    assert np.array_equal(qt, qr) and st == sr[0]
    qc, sc, _ = fp8.cast_colwise(x.T, E4M3)
    assert np.array_equal(qc.T, qt) and sc[0] == st


def test_outlier_robustness():
    # with one outlier row, rowwise reconstruction MSE on the other rows < tensorwise.
    rng = np.random.default_rng(9)
    x = rng.standard_normal((32, 256)).astype(np.float32)
    x[5] *= 1e4
    qt, st, _ = fp8.cast_tensorwise(x, E4M3)
    qr, sr, _ = fp8.cast_rowwise(x, E4M3)
    rt = codecs.decode(qt, E4M3) / st
    rr = codecs.decode(qr, E4M3) / sr[:, None]
    keep = np.arange(32) != 5
    assert np.mean((rr[keep] - x[keep]) ** 2) < np.mean((rt[keep] - x[keep]) ** 2)


def test_grid_points_round_trip_at_unit_scale():
    # S:277 "x with amax 448 tensorwise -> scale 1.0; grid-point entries round-trip exactly"
    grid = codecs.decode(np.arange(0x7F), E4M3)
    x = np.concatenate([grid, -grid]).astype(np.float32).reshape(2, -1)
    q, s, a = fp8.cast_tensorwise(x, E4M3)
    assert s == 1.0 and np.array_equal(codecs.decode(q, E4M3), x.astype(np.float64))
