"""The seeded input generator: determinism, row-addressability, bf16 rounding."""

import numpy as np
import pytest

import synth


def test_deterministic_and_seeded():
    a = synth.tensor_c2("x", (32, 64), seed=0)
    b = synth.tensor_c2("x", (32, 64), seed=0)
    c = synth.tensor_c2("x", (32, 64), seed=1)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_rows_match_full():
    full = synth.tensor_c2("w", (64, 48), seed=3, cfg="c5")
    for r in range(4):
        assert np.array_equal(synth.weight_shard_c5((64, 48), 3, r, 4), full[16 * r:16 * r + 16])


def test_bf16_rounding_is_rne_and_values_representable():
    x = np.array([1.0, 1.00390625, 1.01171875, -3.5e-39, 65504.0], dtype=np.float64)
    bits = synth.bf16_bits(x)
    # 1 + 2^-8 is a tie between 1.0 (even) and 1.0078125 -> 1.0; 1 + 3*2^-8 ties to 1.015625
    assert list(bits[:3]) == [0x3F80, 0x3F80, 0x3F82]
    v = synth.as_bf16_f32(np.random.default_rng(0).standard_normal(1000))
    assert np.all((v.view(np.uint32) & 0xFFFF) == 0)


def test_normal_moments():
    z = synth.normal(synth.stream_key("moments"), (200000,))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_recipe_rows_match_full(cfg):
    f = synth.RECIPES[cfg]
    for name in ("x", "w", "dy"):
        full = f(name, (96, 256), 4, cfg)
        part = f(name, (96, 256), 4, cfg, rows=(37, 71))
        assert np.array_equal(full[37:71].view(np.uint32), part.view(np.uint32)), (cfg, name)


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_device_port_matches_host_generator(cfg):
    """synth.device (torch ops; bench.py's generator) reproduces synth bit for bit -- here with torch on
    the CPU; tests/test_gpu_synth.py repeats it on the GPU at the full bench shapes."""
    import torch
    from synth import device as sd
    f = synth.RECIPES[cfg]
    for name, shape in (("x", (80, 256)), ("w", (64, 256)), ("dy", (80, 64 * 4))):
        ref = f(name, shape, 2, cfg)
        got = sd.tensor(cfg, name, shape, 2, "cpu").float().numpy()
        assert np.array_equal(ref.view(np.uint32), got.view(np.uint32)), (cfg, name)
        part = sd.tensor(cfg, name, shape, 2, "cpu", rows=(17, 50)).float().numpy()
        assert np.array_equal(ref[17:50].view(np.uint32), part.view(np.uint32)), (cfg, name)
    ws = synth.weight_shard_c5((64, 256), 1, 1, 4)
    got = sd.weight_shard_c5((64, 256), 1, 1, 4, "cpu").float().numpy()
    assert np.array_equal(ws.view(np.uint32), got.view(np.uint32))
