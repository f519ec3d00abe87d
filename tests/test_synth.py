"""The seeded input generator: determinism, row-addressability, bf16 rounding."""

import numpy as np

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
