"""Pins for oracle/mx.py.

* SURVEY App. A.8 table (tests/golden/mx.txt): FLOOR / RCEIL codes and element bytes
* zero block -> minimum scale and zero elements; amax = fmax*2^j ->
  exponent j, grid points lossless
* FLOOR == integer rule clamp(expbits_f32(amax) - emax, 0, 254) (bit-field form, App. A.9)
* RCEIL == exact-rational brute force of ceil(log2(amax/fmax))
* FLOOR == RCEIL exactly when the amax mantissa is <= 1.75 (fmax mantissa)
* scale codes decode to powers of two; re-quantizing the dequantized tensor is lossless
"""

from fractions import Fraction

import numpy as np
import pytest

from oracle import codecs, mx
from oracle.codecs import E4M3, E5M2


def _parse(v):
    if v.startswith("0x"):
        return np.array([int(v, 16)], np.uint32).view(np.float32)[0]
    return np.float32(float(v))


def test_mx_golden_table(golden):
    for a, fl, rc, byte in golden("mx.txt"):
        amax = _parse(a)
        assert int(mx.scale_code(amax, E4M3, mx.FLOOR)) == int(fl), a
        assert int(mx.scale_code(amax, E4M3, mx.RCEIL)) == int(rc), a
        if byte != "-":
            blk = np.zeros((1, 32), np.float32)
            blk[0, 0] = amax
            q, sc = mx.quantize_dim0(blk, E4M3, mx.FLOOR)
            assert int(sc[0, 0]) == int(fl) and int(q[0, 0]) == int(byte, 16), (a, hex(q[0, 0]))


def test_zero_block():
    q, sc = mx.quantize_dim0(np.zeros((2, 64), np.float32), E4M3)
    assert np.all(sc == 0) and np.all(q == 0)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_amax_fmax_power_of_two_lossless(fmt):
    grid = codecs.decode(np.arange(0x80), fmt)
    grid = grid[np.isfinite(grid)]
    rng = np.random.default_rng(4)
    for j in (-30, -3, 0, 7, 40):
        blk = rng.choice(grid, size=(1, 32)).astype(np.float64)
        blk[0, 3] = codecs.FMAX[fmt]
        x = (blk * 2.0 ** j).astype(np.float32)
        q, sc = mx.quantize_dim0(x, fmt)
        assert int(sc[0, 0]) == 127 + j
        assert np.array_equal(mx.dequantize(q, sc, fmt), x.astype(np.float64))


def _random_amax(n, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(1, 0x7F7FFFFF, size=n, dtype=np.uint64).astype(np.uint32)
    return bits.view(np.float32)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_floor_equals_exponent_field_rule(fmt):
    a = _random_amax(200000, 1)
    expbits = (a.view(np.uint32) >> 23).astype(np.int64) & 0xFF
    want = np.clip(expbits - codecs.EMAX[fmt], 0, 254)
    assert np.array_equal(mx.scale_code(a, fmt, mx.FLOOR).astype(np.int64), want)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_rceil_vs_rational_brute_force(fmt):
    a = np.concatenate([_random_amax(3000, 2), np.float32([448.0, 448.0 * 2 ** -20, 57344.0, 1.75, 1.7500001])])
    fmax = Fraction(codecs.FMAX[fmt])
    got = mx.scale_code(a, fmt, mx.RCEIL)
    for v, g in zip(a, got):
        r = Fraction(float(v)) / fmax
        e = -300
        while Fraction(2) ** e < r:
            e += 1
        assert int(g) == min(max(127 + e, 0), 254), (v, g, e)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_floor_rceil_agree_iff_mantissa_le_175(fmt):
    a = _random_amax(200000, 3)
    a = a[(a.view(np.uint32) >> 23) > 20]   # normals well inside range (no clamping)
    a = a[(a.view(np.uint32) >> 23) < 230]
    m, _ = np.frexp(a.astype(np.float64))  # a = m * 2^e, m in [0.5, 1)
    small = (2 * m) <= 1.75
    fl = mx.scale_code(a, fmt, mx.FLOOR)
    rc = mx.scale_code(a, fmt, mx.RCEIL)
    assert np.array_equal(fl == rc, small)


@pytest.mark.parametrize("fmt", [E4M3, E5M2])
def test_requantize_lossless_and_pow2(fmt):
    rng = np.random.default_rng(8)
    x = (rng.standard_normal((8, 128)) * np.exp2(rng.uniform(-20, 10, (8, 1)))).astype(np.float32)
    q, sc = mx.quantize_dim0(x, fmt)
    d = mx.dequantize(q, sc, fmt).astype(np.float32)
    q2, sc2 = mx.quantize_dim0(d, fmt)
    assert np.array_equal(mx.dequantize(q2, sc2, fmt), d.astype(np.float64))
    s = codecs.decode_e8m0(sc)
    assert np.all(np.frexp(s)[0] == 0.5)


def test_dim1_is_dim0_of_transpose():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((64, 96)).astype(np.float32)
    q1, s1 = mx.quantize_dim1(x, E4M3)
    assert q1.shape == (96, 64) and s1.shape == (96, 2)
    # block (c, j) covers rows 32j..32j+31 of column c
    for c in (0, 17, 95):
        for j in (0, 1):
            blk = x[32 * j:32 * j + 32, c]
            fl = int(np.floor(np.log2(np.max(np.abs(blk))))) - 8 + 127
            assert int(s1[c, j]) == fl


def test_mx_underflows_less_than_tensorwise():
    # with one scale per tensor "more values may underflow to 0"; per-block MX
    # scales keep small-magnitude blocks representable.
    from oracle import fp8
    rng = np.random.default_rng(12)
    x = (rng.standard_normal((16, 256)) * np.repeat(np.exp2(rng.uniform(-16, 8, (16, 8))), 32, axis=1)).astype(np.float32)
    q, sc = mx.quantize_dim0(x, E4M3)
    qt, st, _ = fp8.cast_tensorwise(x, E4M3)
    zero_mx = np.mean((q & 0x7F) == 0)
    zero_t = np.mean((qt & 0x7F) == 0)
    assert zero_mx < zero_t
