"""MXFP8: per-32-element block E8M0 shared scale + FP8 elements.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: "MX formats: mxfp4, mxfp6, and mxfp8 for training" (Appendix E
prototypes); the north star names "MXFP8 block-32 E8M0 granularities".  The
paper gives no construction, so the SPEC rule is followed
(mx_quant S:339-347) with the readings of SURVEY §8c.12-c.15:

  per block of 32 consecutive elements along the blocked axis:
    FLOOR (default): e = floor(log2(amax_blk)) - emax_elem
    RCEIL (option):  e = ceil(log2(amax_blk / fmax_elem))        (§8c.12)
    code = clamp(127 + e, 0, 254); all-zero block -> code 0      (§8c.13)
    element q = satRNE( RN32( fp32(x) * 2^(127 - code) ) )        ("encode(x / 2^e)")

emax_elem = 8 for e4m3 (448 = 1.75 * 2^8), 15 for e5m2 (57344 = 1.75 * 2^15).
Scales are returned as a plain row-major uint8 array [R, C/32].
"""

import numpy as np

from .codecs import EMAX, FMAX, encode

FLOOR = "floor"
RCEIL = "rceil"
BLOCK = 32


def block_amax(x):
    """amax of each 32-element block along the last axis -> float32 [R, C/32]."""
    x = np.asarray(x, dtype=np.float32)
    R, C = x.shape
    assert C % BLOCK == 0
    return np.max(np.abs(x.reshape(R, C // BLOCK, BLOCK)), axis=2).astype(np.float32)


def _floor_log2(a):
    """floor(log2(a)) for a > 0, exactly (frexp is exact on float64)."""
    _, e = np.frexp(np.asarray(a, dtype=np.float64))
    return e.astype(np.int64) - 1


def scale_code(amax_blk, fmt, mode=FLOOR):
    """E8M0 code per block from the block amax (§8c.12, c.13)."""
    a = np.asarray(amax_blk, dtype=np.float64)
    pos = a > 0
    a_safe = np.where(pos, a, 1.0)
    fl = _floor_log2(a_safe)
    if mode == FLOOR:
        e = fl - EMAX[fmt]
    elif mode == RCEIL:
        # smallest integer e with amax <= fmax * 2^e.  amax/fmax lies in
        # [2^(fl-emax)/1.75, 2^(fl-emax+1)/1.75), so e is fl-emax or fl-emax+1.
        # fmax * 2^e and the comparison are exact in float64.
        e0 = fl - EMAX[fmt]
        e = np.where(a_safe <= np.ldexp(FMAX[fmt], e0), e0, e0 + 1)
    else:
        raise ValueError(mode)
    code = np.clip(127 + e, 0, 254)
    return np.where(pos, code, 0).astype(np.uint8)


def quantize_dim0(x, fmt, mode=FLOOR):
    """Blocks of 32 along the last (contiguous) axis.

    Returns (codes uint8 [R,C], scale codes uint8 [R, C/32]).
    """
    x = np.asarray(x, dtype=np.float32)
    R, C = x.shape
    sc = scale_code(block_amax(x), fmt, mode)
    mult = np.ldexp(np.float32(1.0), (127 - sc.astype(np.int64))).astype(np.float32)  # exact powers of two
    mult_full = np.repeat(mult, BLOCK, axis=1)
    prod = (x * mult_full).astype(np.float32)
    return encode(prod, fmt), sc


def quantize_dim1(x, fmt, mode=FLOOR):
    """Blocks of 32 along the row axis, output in the transposed orientation.

    This is the MX "dim1" copy: the block axis becomes contiguous.
    Returns (codes uint8 [C,R], scale codes uint8 [C, R/32]).
    """
    return quantize_dim0(np.asarray(x, dtype=np.float32).T, fmt, mode)


def dequantize(codes, sc, fmt):
    """decode(code) * 2^(sc-127) per block, float64."""
    from .codecs import decode
    vals = decode(codes, fmt)
    R, C = vals.shape
    mult = np.ldexp(1.0, sc.astype(np.int64) - 127)
    return vals * np.repeat(mult, BLOCK, axis=1)
