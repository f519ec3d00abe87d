"""FP8 (E4M3 "FN", E5M2) and E8M0 codecs -- the plain definitions.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Formats (SPEC lp_dtypes; design decision S:83):
  * E4M3 "FN": 1 sign, 4 exponent bits (bias 7), 3 mantissa bits, no
    infinity, NaN = 0x7F / 0xFF, max finite 448.
  * E5M2: 1 sign, 5 exponent bits (bias 15), 2 mantissa bits, +-inf at
    0x7C / 0xFC, NaN = 0x7D-0x7F / 0xFD-0xFF, max finite 57344.
  * E8M0 (MX shared scale): code c in 0..254 is 2^(c-127); 255 is NaN
    (S:27).

Encoding rule: saturate to the
largest finite magnitude, then pick the nearer of the two adjacent finite
codes, ties to the code with an even (zero) least significant bit; the sign
bit is the sign of the input, so -0 and negative underflow give 0x80.
The paper itself is silent on rounding/overflow.
"""

import numpy as np

E4M3 = "e4m3"
E5M2 = "e5m2"

# (exponent bits, mantissa bits, bias, largest finite positive code)
_FMT = {
    E4M3: (4, 3, 7, 0x7E),
    E5M2: (5, 2, 15, 0x7B),
}

FMAX = {E4M3: 448.0, E5M2: 57344.0}
# emax of the element format: floor(log2(fmax)) (used by the MX rule)
EMAX = {E4M3: 8, E5M2: 15}


def decode(codes, fmt):
    """Exact value of each 8-bit code as float64 (S:39-47 decode_float).

    Closed form: E = exponent field, m = mantissa field, p = mantissa bits,
    b = bias.  E == 0 -> m * 2^(1-b-p) (subnormal); otherwise
    (2^p + m) * 2^(E-b-p).  E4M3: E=15,m=7 is NaN.  E5M2: E=31 is inf (m=0)
    or NaN.
    """
    ebits, mbits, bias, _ = _FMT[fmt]
    c = np.asarray(codes, dtype=np.int64)
    sign = np.where((c >> 7) & 1, -1.0, 1.0)
    E = (c >> mbits) & ((1 << ebits) - 1)
    m = c & ((1 << mbits) - 1)
    sub = m.astype(np.float64) * np.ldexp(1.0, 1 - bias - mbits)
    nrm = ((1 << mbits) + m).astype(np.float64) * np.ldexp(1.0, (E - bias - mbits).astype(np.int64))
    val = sign * np.where(E == 0, sub, nrm)
    emax_field = (1 << ebits) - 1
    if fmt == E4M3:
        val = np.where((E == emax_field) & (m == (1 << mbits) - 1), np.nan, val)
    else:
        val = np.where((E == emax_field) & (m == 0), sign * np.inf, val)
        val = np.where((E == emax_field) & (m != 0), np.nan, val)
    return val


def _positive_table(fmt):
    """Sorted exact values of the non-negative finite codes 0x00..maxcode.

    Index i of the table is code i (codes of one sign are monotone).
    """
    maxcode = _FMT[fmt][3]
    return decode(np.arange(maxcode + 1), fmt)


def encode(values, fmt):
    """Saturating round-to-nearest-even encode of exact fp32/fp64 values.

    ``values`` is an array of real numbers, each exactly representable in
    float64 (fp32 inputs always are).  Returns uint8 codes.

    Plain definition:
      a = min(|v|, fmax); lo/hi = adjacent finite codes around a;
      a < midpoint -> lo, a > midpoint -> hi, a == midpoint -> the even code.
    Midpoints of adjacent FP8 values have at most 5 significant bits, so
    every comparison below is exact in float64.  NaN -> 0x7F (canonical;
    out of contract).
    """
    v = np.asarray(values, dtype=np.float64)
    table = _positive_table(fmt)
    maxcode = len(table) - 1
    neg = np.signbit(v)
    a = np.minimum(np.abs(v), FMAX[fmt])
    nan = np.isnan(v)
    a = np.where(nan, 0.0, a)
    lo = np.searchsorted(table, a, side="right") - 1          # table[lo] <= a
    lo = np.clip(lo, 0, maxcode)
    hi = np.minimum(lo + 1, maxcode)
    mid = (table[lo] + table[hi]) / 2.0                          # exact
    code = np.where(a < mid, lo, np.where(a > mid, hi, np.where(lo % 2 == 0, lo, hi)))
    code = np.where(table[lo] == a, lo, code)
    out = (code | np.where(neg, 0x80, 0)).astype(np.uint8)
    out = np.where(nan, np.uint8(0x7F), out)
    return out.astype(np.uint8)


def decode_e8m0(codes):
    """E8M0 scale code -> 2^(c-127); 255 -> NaN."""
    c = np.asarray(codes, dtype=np.int64)
    return np.where(c == 255, np.nan, np.ldexp(1.0, c - 127))
