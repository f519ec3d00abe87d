"""Device (torch) port of synth's counter-based generator, for inputs too large to make on the host.

Same stream keys, counters and value recipes as ``synth`` (splitmix64 over a counter -> 53-bit
uniforms -> Box-Muller in float64 -> recipe scaling -> RNE to float32 -> RNE to bfloat16), written
with torch int64 / float64 ops so it runs on the GPU.  Like ``synth`` it holds no arithmetic of the
method.  Integer steps are bit-exact by construction (int64 wrap-around multiply = uint64 multiply;
logical right shifts are masked arithmetic shifts); float64 add / multiply / sqrt are correctly
rounded on both sides; log / cos / exp2 come from two different math libraries (CUDA vs the host
libm), so agreement with ``synth`` is verified, not assumed: tests/test_gpu_synth.py compares
sampled rows of every bench tensor at full size bit for bit, and bench.py records the SHA-256 of
the exact tensors it times.
"""

import math

import torch

from . import _outlier_channels, stream_key

_GOLD = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def _s64(v):
    """uint64 constant -> the int64 with the same bits."""
    return v - (1 << 64) if v >= 1 << 63 else v


def _shr(z, k):
    """Logical right shift of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(key, counter):
    """splitmix64 of int64 counters (bit patterns of synth.splitmix64's uint64 outputs)."""
    z = (counter + 1) * _s64(_GOLD) + _s64(key)
    z = (z ^ _shr(z, 30)) * _s64(_C1)
    z = (z ^ _shr(z, 27)) * _s64(_C2)
    return z ^ _shr(z, 31)


def _uniform53(key, counter):
    z = splitmix64(key, counter)
    return (_shr(z, 11).to(torch.float64) + 1.0) * (2.0 ** -53)


def normal_rows(key, shape, r0, r1, device, chunk_rows=None):
    """Rows [r0, r1) of synth.normal(key, shape) (float64), generated on `device` in row chunks."""
    R, C = shape
    out = torch.empty((r1 - r0, C), dtype=torch.float64, device=device)
    step = chunk_rows or max(1, (1 << 24) // C)
    for a in range(r0, r1, step):
        b = min(r1, a + step)
        c = torch.arange(a * C, b * C, dtype=torch.int64, device=device)
        u1 = _uniform53(key, 2 * c)
        u2 = _uniform53(key, 2 * c + 1)
        out[a - r0:b - r0] = (torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)).view(b - a, C)
    return out


def uniform(key, n, device):
    c = torch.arange(0, n, dtype=torch.int64, device=device)
    return _uniform53(key, c)


def _to_bf16(z64):
    return z64.to(torch.float32).to(torch.bfloat16)


def tensor(cfg, name, shape, seed, device, rows=None):
    """bf16 tensor of synth.RECIPES[cfg](name, shape, seed), rows [r0, r1) (default: all) -- c2/c5,
    c3 and c4 value recipes."""
    R, C = shape
    r0, r1 = rows if rows is not None else (0, R)
    key = stream_key(cfg, name, seed, tuple(shape))
    out = torch.empty((r1 - r0, C), dtype=torch.bfloat16, device=device)
    if cfg in ("c2", "c3", "c5"):
        mult = {"x": 1.0, "w": 0.02, "dy": 1e-3}[name]
        ch = torch.from_numpy(_outlier_channels(cfg, seed, C)).to(device) if name == "x" else None
        if cfg == "c3":
            span = 4.0 if name == "w" else 8.0
            u = uniform(stream_key(cfg, name + "_rowscale", seed, tuple(shape)), R, device)[r0:r1]
            rs = torch.exp2((2.0 * u - 1.0) * span)
        step = max(1, (1 << 25) // C)
        for a in range(r0, r1, step):
            b = min(r1, a + step)
            z = normal_rows(key, shape, a, b, device, chunk_rows=b - a)
            if ch is not None:
                z[:, ch] *= 20.0
            elif mult != 1.0:
                z *= mult
            if cfg == "c3":
                z *= rs[a - r0:b - r0, None]
            out[a - r0:b - r0] = _to_bf16(z)
        return out
    if cfg == "c4":
        kb = stream_key(cfg, name + "_blk", seed, tuple(shape))
        kk = stream_key(cfg, name + "_kind", seed, tuple(shape))
        nb = C // 32
        step = max(1, (1 << 25) // C)
        for a in range(r0, r1, step):
            b = min(r1, a + step)
            z = normal_rows(key, shape, a, b, device, chunk_rows=b - a).view(b - a, nb, 32)
            cnt = torch.arange(a * nb, b * nb, dtype=torch.int64, device=device)
            u = _uniform53(kb, cnt).view(b - a, nb)
            v = _uniform53(kk, cnt).view(b - a, nb)
            mag = torch.exp2(-20.0 + 30.0 * u)
            mag = torch.where(v < 0.01, torch.zeros_like(mag), mag)
            mag = torch.where((v >= 0.01) & (v < 0.012), torch.full_like(mag, 2.0 ** -130), mag)
            out[a - r0:b - r0] = _to_bf16((z * mag[:, :, None]).view(b - a, C))
        return out
    raise ValueError(cfg)


def weight_shard_c5(shape, seed, rank, world, device):
    """Device form of synth.weight_shard_c5 (rows of the full C5 W owned by `rank`)."""
    N, K = shape
    r0, r1 = rank * N // world, (rank + 1) * N // world
    key = stream_key("c5", "w", seed, tuple(shape))
    out = torch.empty((r1 - r0, K), dtype=torch.bfloat16, device=device)
    step = max(1, (1 << 25) // K)
    for a in range(r0, r1, step):
        b = min(r1, a + step)
        out[a - r0:b - r0] = _to_bf16(normal_rows(key, shape, a, b, device, chunk_rows=b - a) * 0.02)
    return out
