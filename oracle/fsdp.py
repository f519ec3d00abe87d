"""FSDP2-style FP8 weight all-gather with a global amax (tensorwise only).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: "When training with FSDP, tensorwise scaling also supports an
additional optimization enable_fp8_all_gather which will perform the
all-gathers in FSDP using FP8 to reduce communication overhead" (P:596,
Appendix A).  Reading: one global scale per weight tensor
from the MAX of the per-shard amaxes, so every rank casts with the same s.

Per rank r with shard W_r = W[r*N/P:(r+1)*N/P]:
  1. a_r = amax(W_r)
  2. a = max_r a_r               (all-reduce MAX)
  3. s = RN32(fmax / max(a, EPS))
  4. q_r = satRNE(RN32(W_r * s)) into slot r
  5. all-gather the bytes
"""

import numpy as np

from . import fp8


def allgather_ref(shards, fmt):
    """Returns (gathered codes [N,K], s, global amax) from the list of shards."""
    a = np.max(np.stack([fp8.amax(w) for w in shards]))
    s = fp8.scale_from_amax(a, fmt)
    q = np.concatenate([fp8.cast_scaled(w, s, fmt) for w in shards], axis=0)
    return q, s, np.float32(a)


def allgather_mx_ref(shards, fmt, mode="floor"):
    """MXFP8 FSDP gather (MX formats for training).

    No amax exchange: every 32-block lies inside one shard (rows_local % 32 == 0), so each
    rank quantizes its own shard (oracle.mx.quantize_dim0 / quantize_dim1) and the gather is
    a concatenation:
      dim0 (blocks along K):  codes and scales stacked along rows      -> [N, K], [N, K/32]
      dim1 (blocks along N):  transposed codes / scales along columns  -> [K, N], [K, N/32]
    Returns (q0, s0, q1, s1) in the orientation of oracle.mx.
    """
    from . import mx
    d0 = [mx.quantize_dim0(w, fmt, mode) for w in shards]
    d1 = [mx.quantize_dim1(w, fmt, mode) for w in shards]
    return (np.concatenate([q for q, _ in d0], axis=0), np.concatenate([s for _, s in d0], axis=0),
            np.concatenate([q for q, _ in d1], axis=1), np.concatenate([s for _, s in d1], axis=1))
