"""CPU oracle for the dynamically scaled Float8Linear step (TorchAO, arXiv 2507.16099).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2507_16099_b200``)
may import, call or link anything in this package.  The only permitted callers
are ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``).

The oracle is a plain, slow, obviously-correct numpy implementation of what
the method computes.  It shares no code with the CUDA path: no kernels, no
headers, no tables, no constant generators.  Each function cites the passage
it follows.  Citation forms:

* ``P:n``  -- PAPER.md line n (section named alongside),
* ``S:n``  -- SPEC.md line n (module named alongside; interface/test ideas only),
* ``SURVEY §8c.k`` -- the reading taken where the paper is silent (mirrored
  in DESIGN.md "Readings").

Floating point follows the paper's stated precisions where they exist:
amax/scale/cast are IEEE fp32 operations written out in numpy float32
(paper: "dynamically casts activations, weights, and gradients to FP8",
P:281-283); GEMMs are the exact dequantized product accumulated in fp64
(S:122-130).

Parity status per function: every public
function here is pinned by at least one ``-m "not gpu"`` test against
something other than itself (closed forms, exhaustive enumeration, library
RNE routines, exact rational brute force, printed example values).  The
one deliberately unpinned quantity is the GPU GEMM's fp32 accumulation
order, which is graded by tolerance.
"""

from . import codecs, fp8, mx, gemm, linear, fsdp, grouped  # noqa: F401

__all__ = ["codecs", "fp8", "mx", "gemm", "linear", "fsdp", "grouped"]
