"""B200-native dynamically scaled Float8Linear (TorchAO, arXiv 2507.16099 §2.1 + Appendix A).

Product path: libfp8train.so (hand-written sm_100a CUDA behind the C-ABI in
include/fp8train.h) + this thin Python layer.  Importing raises if the library
has not been built; there is no CPU fallback.
"""

from . import _lib  # noqa: F401  (loads libfp8train.so or raises)
from .ops import GroupedPlan, LinearPlan, SharedInputPlan, amax, cast, gemm, launch_count  # noqa: F401
from .linear import Float8Linear, convert, scaled_grouped_mm, shared_input_linears  # noqa: F401

__all__ = ["GroupedPlan", "LinearPlan", "SharedInputPlan", "amax", "cast", "gemm", "launch_count", "Float8Linear", "convert",
           "scaled_grouped_mm", "shared_input_linears"]
