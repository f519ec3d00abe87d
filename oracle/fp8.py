"""amax -> scale -> saturating RNE cast, tensorwise / rowwise / colwise.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: "TorchAO's FP8 training dynamically casts activations, weights, and
gradients to FP8" (§2.1).  Recipes (Appendix A):
  * tensorwise -- "computes a single scaling factor for each tensor"
  * rowwise -- "scaling factors along logical rows of the left GEMM operand,
    and along logical columns of the right GEMM operand"

Written-out definitions (SPEC float8_train S:266-279):
  amax  = max |x| over the scaling unit (exact)
  s     = RN32( fmax / max(amax, EPS) ),  EPS = fp32(1e-12)      (§8c.3, c.5, c.6)
  q     = satRNE_fmt( RN32( fp32(x) * s ) )                     (§8c.4: two roundings)
The scale is multiplicative (fp8 ~= x*s); GEMM epilogues divide it back out.
"""

import numpy as np

from .codecs import FMAX, encode

# eps = fp32(1e-12), bit pattern 0x2B8CBCCC.
EPS = np.float32(1e-12)


def amax(x, axis=None):
    """max |x| over the whole tensor (axis=None), rows (axis=1) or cols (axis=0).

    Exact: |x| and max are exact on fp32 values.  Returns float32.
    """
    x = np.asarray(x, dtype=np.float32)
    return np.max(np.abs(x), axis=axis).astype(np.float32)


def scale_from_amax(a, fmt):
    """s = RN32(fmax / max(amax, EPS)) in IEEE fp32 division (§8c.6).

    numpy float32 '/' is the correctly rounded IEEE binary32 division.
    """
    a = np.asarray(a, dtype=np.float32)
    return (np.float32(FMAX[fmt]) / np.maximum(a, EPS)).astype(np.float32)


def cast_scaled(x, s, fmt):
    """q = satRNE(RN32(fp32(x) * s)) elementwise; s broadcasts (§8c.4).

    The product is rounded to fp32 first (numpy float32 multiply), then
    encoded -- the two roundings the GPU path must reproduce.
    """
    x = np.asarray(x, dtype=np.float32)
    s = np.asarray(s, dtype=np.float32)
    prod = (x * s).astype(np.float32)
    return encode(prod, fmt)


def cast_tensorwise(x, fmt):
    """One scale for the whole tensor.  Returns (codes, s, amax)."""
    a = amax(x)
    s = scale_from_amax(a, fmt)
    return cast_scaled(x, s, fmt), s, a


def cast_rowwise(x, fmt):
    """One scale per row, reduced over the contiguous (last) dim (§8c.17).

    Returns (codes [R,C], s [R], amax [R]).
    """
    a = amax(x, axis=1)
    s = scale_from_amax(a, fmt)
    return cast_scaled(x, s[:, None], fmt), s, a


def cast_colwise(x, fmt):
    """One scale per column, reduced over rows (right-operand columns).

    Returns (codes [R,C] in the original row-major orientation, s [C], amax [C]).
    The GPU writes these codes transposed ([C,R]); tests transpose to compare.
    """
    a = amax(x, axis=0)
    s = scale_from_amax(a, fmt)
    return cast_scaled(x, s[None, :], fmt), s, a
