"""Pins for oracle/codecs.py against things other than itself.

* exhaustive 256-code decode vs ml_dtypes and torch float8 dtypes (library decoders)
* SPEC / SURVEY App. A fixture values (tests/golden/decode.txt, encode.txt)
* encode vs exact-rational brute force (nearest, ties-to-even) on crafted + random values
* encode vs the library RNE routine  clip(x, +-fmax) -> ml_dtypes astype  on 2^22 random
  fp32 bit patterns and all 2^16 bf16 patterns (all 2^32 with FP8_EXHAUSTIVE=1)
* round-trip and monotonicity invariants
"""

import os
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest
import torch

from oracle import codecs
from oracle.codecs import E4M3, E5M2

ML = {E4M3: ml_dtypes.float8_e4m3fn, E5M2: ml_dtypes.float8_e5m2}
TORCH = {E4M3: torch.float8_e4m3fn, E5M2: torch.float8_e5m2}
FMTS = [E4M3, E5M2]


@pytest.mark.parametrize("fmt", FMTS)
def test_decode_all_codes_vs_ml_dtypes(fmt):
    codes = np.arange(256, dtype=np.uint8)
    ours = codecs.decode(codes, fmt)
    lib = codes.view(ML[fmt]).astype(np.float64)
    assert np.array_equal(np.isnan(ours), np.isnan(lib))
    ok = ~np.isnan(lib)
    assert np.array_equal(ours[ok], lib[ok])
    assert np.array_equal(np.signbit(ours[ok]), np.signbit(lib[ok]))


@pytest.mark.parametrize("fmt", FMTS)
def test_decode_all_codes_vs_torch(fmt):
    codes = torch.arange(256, dtype=torch.int32).to(torch.uint8)
    lib = codes.view(TORCH[fmt]).to(torch.float64).numpy()
    ours = codecs.decode(np.arange(256), fmt)
    assert np.array_equal(np.isnan(ours), np.isnan(lib))
    ok = ~np.isnan(lib)
    assert np.array_equal(ours[ok], lib[ok])


def test_code_space_census():
    # App. A.1/A.2: e4m3 has 254 finite codes; e5m2 has 248 finite, 2 inf, 6 NaN.
    d4 = codecs.decode(np.arange(256), E4M3)
    d5 = codecs.decode(np.arange(256), E5M2)
    assert np.isfinite(d4).sum() == 254 and np.isnan(d4).sum() == 2
    assert np.isfinite(d5).sum() == 248 and np.isinf(d5).sum() == 2 and np.isnan(d5).sum() == 6
    assert np.nanmax(d4) == 448.0 and np.max(d5[np.isfinite(d5)]) == 57344.0


def test_decode_golden(golden):
    for fmt, code, val in golden("decode.txt"):
        c = int(code, 0)
        got = codecs.decode_e8m0(c) if fmt == "e8m0" else codecs.decode(c, fmt)
        want = float(val)
        if np.isnan(want):
            assert np.isnan(got), (fmt, code)
        else:
            assert float(got) == want and np.signbit(got) == np.signbit(want), (fmt, code, got, want)


def test_encode_golden(golden):
    for fmt, x, code in golden("encode.txt"):
        got = int(codecs.encode(np.float32(float(x)), fmt))
        assert got == int(code, 0), (fmt, x, hex(got), code)


def _brute_force(v, fmt):
    """Nearest finite code by exact rational distance; ties -> even code; saturate."""
    fmax = Fraction(codecs.FMAX[fmt])
    x = Fraction(float(v))
    neg = np.signbit(v)
    a = min(abs(x), fmax)
    best, bestd = None, None
    for c in range(0x80):
        d = codecs.decode(c, fmt)
        if not np.isfinite(d):
            continue
        dist = abs(Fraction(float(d)) - a)
        if bestd is None or dist < bestd or (dist == bestd and c % 2 == 0):
            best, bestd = c, dist
    return best | (0x80 if neg else 0)


@pytest.mark.parametrize("fmt", FMTS)
def test_encode_vs_brute_force(fmt):
    rng = np.random.default_rng(1234)
    table = codecs.decode(np.arange(0x80), fmt)
    table = table[np.isfinite(table)]
    mids = (table[1:] + table[:-1]) / 2          # exact ties
    vals = list(mids) + list(-mids[::7]) + list(table) + [0.0, -0.0, 1e-30, -1e-30, 1e30, -1e30,
                                                           codecs.FMAX[fmt] * 1.01, 2.0 ** -149]
    vals += list(rng.standard_normal(400) * 10.0 ** rng.integers(-8, 6, 400))
    vals = np.array(vals, dtype=np.float32)
    got = codecs.encode(vals, fmt)
    want = np.array([_brute_force(v, fmt) for v in vals], dtype=np.uint8)
    assert np.array_equal(got, want)


def _lib_encode(x32, fmt):
    fmax = np.float32(codecs.FMAX[fmt])
    return np.clip(x32, -fmax, fmax).astype(ML[fmt]).view(np.uint8)


@pytest.mark.parametrize("fmt", FMTS)
def test_encode_vs_library_random_fp32(fmt):
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 2 ** 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[~np.isnan(x)]
    assert np.array_equal(codecs.encode(x, fmt), _lib_encode(x, fmt))


@pytest.mark.parametrize("fmt", FMTS)
def test_encode_vs_library_all_bf16(fmt):
    bits = np.arange(1 << 16, dtype=np.uint32) << np.uint32(16)
    x = bits.view(np.float32)
    x = x[~np.isnan(x)]
    assert np.array_equal(codecs.encode(x, fmt), _lib_encode(x, fmt))


@pytest.mark.skipif(os.environ.get("FP8_EXHAUSTIVE") != "1", reason="set FP8_EXHAUSTIVE=1 (minutes)")
@pytest.mark.parametrize("fmt", FMTS)
def test_encode_vs_library_all_fp32(fmt):
    step = 1 << 24
    for start in range(0, 1 << 32, step):
        x = np.arange(start, start + step, dtype=np.uint64).astype(np.uint32).view(np.float32)
        x = x[~np.isnan(x)]
        assert np.array_equal(codecs.encode(x, fmt), _lib_encode(x, fmt)), hex(start)


@pytest.mark.parametrize("fmt", FMTS)
def test_round_trip_and_monotone(fmt):
    codes = np.arange(256)
    vals = codecs.decode(codes, fmt)
    fin = np.isfinite(vals)
    assert np.array_equal(codecs.encode(vals[fin], fmt), codes[fin].astype(np.uint8))
    pos = vals[:0x80][np.isfinite(vals[:0x80])]
    assert np.all(np.diff(pos) > 0)


def test_e8m0():
    c = np.arange(256)
    v = codecs.decode_e8m0(c)
    assert np.isnan(v[255])
    assert np.all(v[:255] == 2.0 ** (c[:255] - 127.0))
    lib = c.astype(np.uint8).view(ml_dtypes.float8_e8m0fnu).astype(np.float64)
    assert np.array_equal(v[:255], lib[:255])
