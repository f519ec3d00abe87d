"""synth.device (bench.py's input generator, run on the GPU) vs synth (numpy, the parity tests'
generator): bit-identical bf16 values, on sampled row blocks of every tensor bench.py times at its full
shapes, and on one full tensor.  The integer counter steps are exact on both sides; float64 log / cos /
exp2 come from different math libraries, so this is checked, not assumed (synth/device.py)."""

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

BENCH_TENSORS = [
    ("c2", "x", (16384, 4096)), ("c2", "w", (14336, 4096)), ("c2", "dy", (16384, 14336)),
    ("c4", "x", (16384, 8192)), ("c4", "w", (28672, 8192)), ("c4", "dy", (16384, 28672)),
    ("c5", "x", (8192, 16384)), ("c5", "w", (53248, 16384)), ("c5", "dy", (8192, 53248)),
    ("c3", "x", (16384, 4096)), ("c3", "w", (1024, 4096)), ("c3", "dy", (16384, 1024)),
    ("c3", "x", (16384, 14336)), ("c3", "w", (4096, 14336)), ("c3", "dy", (16384, 4096)),
]


@pytest.mark.parametrize("cfg,name,shape", BENCH_TENSORS, ids=[f"{c}-{n}-{s[0]}x{s[1]}" for c, n, s in BENCH_TENSORS])
def test_device_generator_rows(cfg, name, shape):
    from synth import device as sd
    R = shape[0]
    rng = np.random.default_rng(hash((cfg, name, shape)) & 0xFFFF)
    for r0 in sorted({0, R - 8, int(rng.integers(8, R - 16))}):
        ref = synth.RECIPES[cfg](name, shape, 0, cfg, rows=(r0, r0 + 8))
        got = sd.tensor(cfg, name, shape, 0, "cuda", rows=(r0, r0 + 8)).float().cpu().numpy()
        bad = np.count_nonzero(ref.view(np.uint32) != got.view(np.uint32))
        assert bad == 0, f"rows {r0}..{r0 + 8}: {bad} of {ref.size} differ"


def test_device_generator_full_tensor():
    """A whole bench tensor (c2 X, 67M elements, the same call bench.py makes) equals synth's."""
    from synth import device as sd
    ref = synth.RECIPES["c2"]("x", (16384, 4096), 0, "c2")
    got = sd.tensor("c2", "x", (16384, 4096), 0, "cuda").float().cpu().numpy()
    assert np.count_nonzero(ref.view(np.uint32) != got.view(np.uint32)) == 0


def test_device_generator_c5_shard():
    from synth import device as sd
    ref = synth.weight_shard_c5((53248, 16384), 0, 3, 8)[:16]
    got = sd.weight_shard_c5((53248, 16384), 0, 3, 8, "cuda")[:16].float().cpu().numpy()
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))
