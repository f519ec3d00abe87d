"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no amax, scale, cast or GEMM):
only a counter-based random generator and the value recipes of the five
BASELINE.json configurations (SURVEY §8d "Configs as concrete synthetic
inputs"; recipe stated in DESIGN.md "Input recipe").

Generator: splitmix64 over a counter ("splitmix-style 64-bit
generator") -> 53-bit uniforms -> Box-Muller in float64 -> scaled -> rounded
to bfloat16 with round-to-nearest-even (fp32 for config 1).  Every tensor is
addressed by (config, name, seed), so any sub-block can be regenerated
independently of the others, on any host.
"""

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 22


def stream_key(*parts):
    """64-bit stream id from a tuple of names/ints (stable across hosts)."""
    h = hashlib.sha256(repr(parts).encode()).digest()
    return int.from_bytes(h[:8], "little")


def splitmix64(key, counter):
    """splitmix64 output for counter values (uint64 array), stream `key`."""
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (counter.astype(np.uint64) + np.uint64(1)) * _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def _uniform53(key, counter):
    """Uniform in (0, 1]: ((z >> 11) + 1) * 2^-53."""
    z = splitmix64(key, counter)
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def _normal_chunk(key, start, n):
    c = np.arange(start, start + n, dtype=np.uint64)
    u1 = _uniform53(key, 2 * c)
    u2 = _uniform53(key, 2 * c + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def _uniform_chunk(key, start, n):
    c = np.arange(start, start + n, dtype=np.uint64)
    return _uniform53(key, c)


def _fill(fn, key, total):
    out = np.empty(total, dtype=np.float64)
    starts = list(range(0, total, _CHUNK))

    def work(s):
        n = min(_CHUNK, total - s)
        out[s:s + n] = fn(key, s, n)

    if len(starts) <= 1:
        for s in starts:
            work(s)
    else:
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
            list(ex.map(work, starts))
    return out


def normal(key, shape):
    """Standard normals (float64) for stream `key`."""
    return _fill(_normal_chunk, key, int(np.prod(shape))).reshape(shape)


def normal_rows(key, shape, r0, r1):
    """Rows [r0, r1) of ``normal(key, shape)`` without generating the rest
    (counter-based: element (r, c) is counter r*C + c)."""
    R, C = shape
    n = (r1 - r0) * C
    out = np.empty(n, dtype=np.float64)
    base = r0 * C
    starts = list(range(0, n, _CHUNK))

    def work(s):
        m = min(_CHUNK, n - s)
        out[s:s + m] = _normal_chunk(key, base + s, m)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(work, starts))
    return out.reshape(r1 - r0, C)


def uniform(key, shape):
    """Uniforms in (0, 1] (float64) for stream `key`."""
    return _fill(_uniform_chunk, key, int(np.prod(shape))).reshape(shape)


def bf16_bits(x):
    """Round float64 values to bfloat16 (via fp32, RNE) -> uint16 bit patterns.

    Input preparation only: produces the bf16 tensors the path consumes.
    """
    f = np.asarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    r = r.astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        r = np.where(nan, np.uint16(0x7FC0), r)
    return r


def bf16_to_f32(bits):
    """Exact float32 values of bf16 bit patterns."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def as_bf16_f32(x):
    """float64 -> bf16-representable float32 values."""
    return bf16_to_f32(bf16_bits(x))


# --------------------------------------------------------------------------
# Value recipes
# --------------------------------------------------------------------------

def _outlier_channels(cfg, seed, K, count=8):
    u = uniform(stream_key(cfg, "outlier_ch", seed), (count,))
    return np.unique((u * K).astype(np.int64) % K)


def _z(cfg, name, seed, shape, rows):
    key = stream_key(cfg, name, seed, shape)
    if rows is None:
        return normal(key, shape)
    return normal_rows(key, shape, rows[0], rows[1])


def tensor_c2(name, shape, seed, cfg="c2", rows=None):
    """C2/C5 value structure (Llama linears, tensorwise):
    X ~ N(0,1) with 8 outlier channels x20; W ~ N(0, 0.02^2); dY ~ N(0, 1e-3^2).
    rows=(r0, r1): only those rows of the same tensor (counter-based)."""
    z = _z(cfg, name, seed, shape, rows)
    if name == "x":
        z[:, _outlier_channels(cfg, seed, shape[1])] *= 20.0
    elif name == "w":
        z *= 0.02
    elif name == "dy":
        z *= 1e-3
    return as_bf16_f32(z)


def tensor_c3(name, shape, seed, cfg="c3", rows=None):
    """C3 (rowwise): C2 distributions, rows additionally scaled by 2^U(-8,8)
    (X, dY) or 2^U(-4,4) (W) so per-row scales differ."""
    z = _z(cfg, name, seed, shape, rows)
    if name == "x":
        z[:, _outlier_channels(cfg, seed, shape[1])] *= 20.0
    elif name == "w":
        z *= 0.02
    elif name == "dy":
        z *= 1e-3
    span = 4.0 if name == "w" else 8.0
    u = uniform(stream_key(cfg, name + "_rowscale", seed, shape), (shape[0],))
    if rows is not None:
        u = u[rows[0]:rows[1]]
    z *= np.exp2((2.0 * u - 1.0) * span)[:, None]
    return as_bf16_f32(z)


def tensor_c4(name, shape, seed, cfg="c4", rows=None):
    """C4 (MXFP8): per-32-block magnitude 2^U(-20,10) along rows; ~1% all-zero
    blocks; ~0.2% blocks at bf16-subnormal magnitude (2^-130)."""
    R, C = shape
    r0, r1 = rows if rows is not None else (0, R)
    z = _z(cfg, name, seed, shape, rows).reshape(r1 - r0, C // 32, 32)
    u = uniform(stream_key(cfg, name + "_blk", seed, shape), (R, C // 32))[r0:r1]
    mag = np.exp2(-20.0 + 30.0 * u)
    v = uniform(stream_key(cfg, name + "_kind", seed, shape), (R, C // 32))[r0:r1]
    mag = np.where(v < 0.01, 0.0, mag)
    mag = np.where((v >= 0.01) & (v < 0.012), 2.0 ** -130, mag)
    z = z * mag[:, :, None]
    return as_bf16_f32(z.reshape(r1 - r0, C))


def tensor_c1(name, shape, seed, cfg="c1"):
    """C1: N(0,1) in fp32 (config 1 is fp32 in)."""
    return normal(stream_key(cfg, name, seed, shape), shape).astype(np.float32)


RECIPES = {"c1": tensor_c1, "c2": tensor_c2, "c3": tensor_c3, "c4": tensor_c4, "c5": tensor_c2}


def weight_shard_c5(shape, seed, rank, world):
    """Rows [r*N/P, (r+1)*N/P) of the C5 weight W ~ N(0, 0.02^2) (bf16-valued).

    The full W is defined identically on every rank (same stream), each rank
    materialises only its own shard."""
    N, K = shape
    assert N % world == 0
    r0, r1 = rank * N // world, (rank + 1) * N // world
    z = normal_rows(stream_key("c5", "w", seed, tuple(shape)), shape, r0, r1) * 0.02
    return as_bf16_f32(z)


def linear_inputs(cfg, M, N, K, seed=0):
    """(x [M,K], w [N,K], dy [M,N]) float32 arrays (bf16-valued except c1)."""
    f = RECIPES[cfg]
    return f("x", (M, K), seed, cfg), f("w", (N, K), seed, cfg), f("dy", (M, N), seed, cfg)


def integer_grid(key, shape, values):
    """Uniform draw from a finite set of values (integer-grid GEMM fixtures,
    SURVEY App. A.12)."""
    u = uniform(key, shape)
    vals = np.asarray(values, dtype=np.float32)
    return vals[np.minimum((u * len(vals)).astype(np.int64), len(vals) - 1)]


def sha256(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
