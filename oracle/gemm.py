"""Scaled FP8 GEMM reference: the exact dequantized product in fp64.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: FP8 training "leverages specialized GEMM kernels to take advantage of
the FP8 tensor cores" (§2.1).  The emulation contract is SPEC
scaled_gemm and gemm_ref:

    y[m,n] = ( sum_k dec(a[m,k]) * dec(b[n,k]) ) * (1/s_a[m]) * (1/s_b[n])

in fp64 (products of FP8 values are exact in fp64; the K-sum's fp64 rounding
is ~K*2^-53 relative, far below the graded tolerance).  Both operands are
given "K-major": a is [M,K], b is [N,K] (nn.Linear weight layout), so
y = a @ b^T.  Tensorwise scales are scalars; rowwise scales are vectors over
rows of a and rows of b (= columns of the logical right operand).

``abs_bound`` returns sum_k |dec(a)||dec(b)| / (s_a s_b), the per-element
scale of the north-star tolerance |err| <= 1e-2 * abs_bound (BASELINE.json).
"""

import numpy as np

from .codecs import decode
from . import mx as _mx


def _inv(s, n):
    """1/s in fp64 as a length-n vector (scalar s broadcasts)."""
    s = np.asarray(s, dtype=np.float64)
    if s.ndim == 0 or s.size == 1:
        return np.full(n, 1.0 / float(s.reshape(-1)[0]))
    assert s.shape == (n,), (s.shape, n)
    return 1.0 / s


def gemm_ref(a_codes, a_fmt, s_a, b_codes, b_fmt, s_b):
    """Scaled FP8 GEMM, tensorwise or rowwise scales.  Returns fp64 [M,N]."""
    A = decode(a_codes, a_fmt)
    B = decode(b_codes, b_fmt)
    M, N = A.shape[0], B.shape[0]
    return (A @ B.T) * _inv(s_a, M)[:, None] * _inv(s_b, N)[None, :]


def abs_bound(a_codes, a_fmt, s_a, b_codes, b_fmt, s_b):
    """sum_k |dec(a)||dec(b)| / (s_a s_b) per output element (tolerance scale)."""
    A = np.abs(decode(a_codes, a_fmt))
    B = np.abs(decode(b_codes, b_fmt))
    M, N = A.shape[0], B.shape[0]
    return (A @ B.T) * _inv(s_a, M)[:, None] * _inv(s_b, N)[None, :]


def mx_gemm_ref(a_codes, a_sc, a_fmt, b_codes, b_sc, b_fmt):
    """MX GEMM = gemm_ref(mx_dequantize(a), mx_dequantize(b)).

    a: codes [M,K] with E8M0 codes [M,K/32]; b: codes [N,K], E8M0 [N,K/32].
    """
    A = _mx.dequantize(a_codes, a_sc, a_fmt)
    B = _mx.dequantize(b_codes, b_sc, b_fmt)
    return A @ B.T


def mx_abs_bound(a_codes, a_sc, a_fmt, b_codes, b_sc, b_fmt):
    A = np.abs(_mx.dequantize(a_codes, a_sc, a_fmt))
    B = np.abs(_mx.dequantize(b_codes, b_sc, b_fmt))
    return A @ B.T


def gemm_ref_rows(rows, a_codes, a_fmt, s_a, b_codes, b_fmt, s_b):
    """gemm_ref restricted to a subset of output rows (for full-size sampled parity)."""
    rows = np.asarray(rows)
    s_a = np.asarray(s_a, dtype=np.float32)
    sa = s_a[rows] if s_a.ndim else s_a
    return gemm_ref(a_codes[rows], a_fmt, sa, b_codes, b_fmt, s_b), \
        abs_bound(a_codes[rows], a_fmt, sa, b_codes, b_fmt, s_b)
