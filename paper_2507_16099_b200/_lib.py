"""ctypes binding of libfp8train.so (include/fp8train.h).  Marshalling only.

The library is the product path: if it is missing this module raises at import
time -- there is no CPU or PyTorch fallback.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfp8train.so")

# enums (fp8train.h)
FP8_OK, FP8_EINVAL, FP8_EALIGN, FP8_EUNSUPPORTED, FP8_ECUDA, FP8_ENCCL, FP8_EWORKSPACE = range(7)
DT_F32, DT_BF16 = 0, 1
E4M3, E5M2 = 0, 1
GRAN_TENSOR, GRAN_ROW, GRAN_COL, GRAN_ROW_COL, GRAN_MX32, GRAN_MX32_RM = range(6)
MX_FLOOR, MX_RCEIL = 0, 1
K_MAJOR, MN_MAJOR = 0, 1
RECIPE_TENSORWISE, RECIPE_ROWWISE, RECIPE_MXFP8, RECIPE_ROWWISE_GW_HP = range(4)

STATUS_NAMES = {0: "FP8_OK", 1: "FP8_EINVAL", 2: "FP8_EALIGN", 3: "FP8_EUNSUPPORTED",
                4: "FP8_ECUDA", 5: "FP8_ENCCL", 6: "FP8_EWORKSPACE"}


class HP(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int), ("rows", ctypes.c_int64),
                ("cols", ctypes.c_int64), ("ld", ctypes.c_int64)]


class Tensor8(ctypes.Structure):
    _fields_ = [("q", ctypes.c_void_p), ("q_t", ctypes.c_void_p), ("scale", ctypes.c_void_p),
                ("scale_t", ctypes.c_void_p), ("amax", ctypes.c_void_p), ("amax_t", ctypes.c_void_p),
                ("fmt", ctypes.c_int), ("gran", ctypes.c_int), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64)]


class LinearBuffers(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "x_fwd", "x_fwd_scale", "w_fwd", "w_fwd_scale", "x_bwd", "x_bwd_scale", "w_bwd", "w_bwd_scale",
        "dy_dx", "dy_dx_scale", "dy_dw", "dy_dw_scale", "amax_fwd", "amax_bwd")] + [("bwd_transposed", ctypes.c_int)]


class LinearCfg(ctypes.Structure):
    _fields_ = [("recipe", ctypes.c_int), ("fmt_fwd", ctypes.c_int), ("fmt_grad", ctypes.c_int),
                ("mx_round", ctypes.c_int), ("out_dtype", ctypes.c_int)]


# every exported symbol of include/fp8train.h with its ctypes signature
_c = ctypes
SIGNATURES = {
    "fp8_abi_version": (_c.c_int, []),
    "fp8_last_error": (_c.c_char_p, []),
    "fp8_launch_count": (_c.c_uint64, []),
    "fp8_profile_enable": (None, [_c.c_int]),
    "fp8_set_knob": (_c.c_int, [_c.c_char_p, _c.c_int]),
    "fp8_check_async_error": (_c.c_int, []),
    "fp8_comm_check": (_c.c_int, [_c.c_void_p]),
    "fp8_get_knob": (_c.c_int, [_c.c_char_p, _c.POINTER(_c.c_int)]),
    "fp8_reset_knobs": (None, []),
    "fp8_profile_collect": (_c.c_int, [_c.POINTER(_c.c_int), _c.POINTER(_c.c_float), _c.c_int]),
    "fp8_amax_workspace_bytes": (_c.c_size_t, [HP, _c.c_int]),
    "fp8_amax": (_c.c_int, [HP, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_amax_multi": (_c.c_int, [_c.POINTER(HP), _c.c_int, _c.c_void_p, _c.c_void_p]),
    "fp8_cast_workspace_bytes": (_c.c_size_t, [HP, _c.c_int]),
    "fp8_cast_scaled": (_c.c_int, [HP, _c.c_int, _c.c_void_p, _c.POINTER(Tensor8), _c.c_void_p, _c.c_size_t,
                                   _c.c_void_p]),
    "fp8_gemm": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_int, _c.c_int,
                            _c.c_void_p, _c.c_int, _c.c_int64, _c.c_int64, _c.c_int64, _c.c_int64, _c.c_int64,
                            _c.c_void_p, _c.c_int, _c.c_int64, _c.c_void_p]),
    "fp8_linear_saved_bytes": (_c.c_size_t, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64, _c.c_int64]),
    "fp8_linear_buffers": (_c.c_int, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64, _c.c_int64, _c.c_void_p,
                                      _c.c_void_p, _c.POINTER(LinearBuffers)]),
    "fp8_linear_workspace_bytes": (_c.c_size_t, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64, _c.c_int64]),
    "fp8_linear_infer_workspace_bytes": (_c.c_size_t, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64,
                                                       _c.c_int64]),
    "fp8_linear_fwd": (_c.c_int, [_c.POINTER(LinearCfg), HP, HP, _c.POINTER(Tensor8), _c.c_void_p, _c.c_void_p,
                                  _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_linear_bwd": (_c.c_int, [_c.POINTER(LinearCfg), HP, HP, _c.c_void_p, _c.POINTER(Tensor8),
                                  _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_linear_fwd_ex": (_c.c_int, [_c.POINTER(LinearCfg), HP, _c.c_void_p, HP, _c.POINTER(Tensor8), _c.c_void_p,
                                     _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_linear_bwd_ex": (_c.c_int, [_c.POINTER(LinearCfg), HP, _c.c_void_p, HP, _c.c_void_p, _c.POINTER(Tensor8),
                                     _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_linear_shared_workspace_bytes": (_c.c_size_t, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64, _c.c_int,
                                                        _c.POINTER(_c.c_int64)]),
    "fp8_linear_fwd_shared": (_c.c_int, [_c.POINTER(LinearCfg), HP, _c.c_int, _c.POINTER(HP), _c.POINTER(_c.c_void_p),
                                         _c.POINTER(_c.c_void_p), _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_linear_bwd_shared": (_c.c_int, [_c.POINTER(LinearCfg), _c.c_int, _c.POINTER(HP), HP, _c.POINTER(_c.c_void_p),
                                         _c.POINTER(_c.c_void_p), _c.POINTER(_c.c_void_p), _c.c_void_p, _c.c_size_t,
                                         _c.c_void_p]),
    "fp8_grouped_saved_bytes": (_c.c_size_t, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64, _c.c_int64,
                                               _c.c_int64]),
    "fp8_grouped_workspace_bytes": (_c.c_size_t, [_c.POINTER(LinearCfg), _c.c_int64, _c.c_int64, _c.c_int64,
                                                   _c.c_int64]),
    "fp8_grouped_linear_fwd": (_c.c_int, [_c.POINTER(LinearCfg), HP, HP, _c.c_int64, _c.c_void_p, _c.c_void_p,
                                          _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_grouped_linear_bwd": (_c.c_int, [_c.POINTER(LinearCfg), HP, HP, _c.c_int64, _c.c_void_p, _c.c_void_p,
                                          _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_comm_get_unique_id": (_c.c_int, [_c.c_void_p]),
    "fp8_comm_init": (_c.c_int, [_c.POINTER(_c.c_void_p), _c.c_void_p, _c.c_int, _c.c_int]),
    "fp8_comm_destroy": (_c.c_int, [_c.c_void_p]),
    "fp8_fsdp_workspace_bytes": (_c.c_size_t, [HP]),
    "fp8_fsdp_allgather": (_c.c_int, [_c.c_void_p, HP, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_void_p,
                                      _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_fsdp_precompute_amax": (_c.c_int, [_c.c_void_p, _c.POINTER(HP), _c.c_int, _c.c_void_p, _c.c_void_p]),
    "fp8_fsdp_allgather_ex": (_c.c_int, [_c.c_void_p, HP, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_void_p,
                                         _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_fsdp_mx_workspace_bytes": (_c.c_size_t, [HP, _c.c_int]),
    "fp8_fsdp_allgather_mx": (_c.c_int, [_c.c_void_p, HP, _c.c_int, _c.POINTER(Tensor8), _c.c_void_p, _c.c_size_t,
                                         _c.c_void_p]),
    "fp8_p2p_create": (_c.c_int, [_c.c_void_p, _c.c_size_t, _c.POINTER(_c.c_void_p)]),
    "fp8_p2p_alloc": (_c.c_int, [_c.c_size_t, _c.c_int, _c.c_int, _c.POINTER(_c.c_void_p), _c.c_void_p]),
    "fp8_p2p_open": (_c.c_int, [_c.c_void_p, _c.c_void_p]),
    "fp8_p2p_create_local": (_c.c_int, [_c.c_int, _c.c_size_t, _c.POINTER(_c.c_void_p)]),
    "fp8_p2p_buffer": (_c.c_void_p, [_c.c_void_p]),
    "fp8_p2p_destroy": (_c.c_int, [_c.c_void_p]),
    "fp8_fsdp_allgather_p2p": (_c.c_int, [_c.c_void_p, HP, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_void_p,
                                          _c.c_void_p]),
    "fp8_fsdp_allgather_p2p_local": (_c.c_int, [_c.POINTER(_c.c_void_p), _c.c_int, _c.POINTER(HP), _c.c_int,
                                                _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p]),
    "fp8_tp_workspace_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int64]),
    "fp8_tp_allgather_linear_fwd": (_c.c_int, [_c.c_void_p, _c.POINTER(LinearCfg), HP, HP, _c.c_void_p, _c.c_void_p,
                                               _c.c_size_t, _c.c_void_p]),
    "fp8_tp_allgather_linear_fwd_local": (_c.c_int, [_c.POINTER(_c.c_void_p), _c.c_int, _c.POINTER(LinearCfg),
                                                     _c.POINTER(HP), _c.POINTER(HP), _c.c_void_p, _c.c_void_p,
                                                     _c.c_size_t, _c.c_void_p]),
    "fp8_linear_bwd_rs": (_c.c_int, [_c.POINTER(LinearCfg), HP, HP, _c.c_void_p, _c.POINTER(Tensor8), _c.c_void_p,
                                     _c.c_void_p, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_tp_bwd_workspace_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int64]),
    "fp8_tp_linear_bwd": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.POINTER(LinearCfg), HP, _c.c_int64,
                                     _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "fp8_mx_scales_unshard": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p]),
}
AMAX_MULTI_MAX = 48


class Fp8Error(RuntimeError):
    def __init__(self, status, fn, msg):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built: run `python paper_2507_16099_b200/build.py` "
            "(there is no CPU fallback for the FP8 path)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status, fn):
    if status != FP8_OK:
        raise Fp8Error(status, fn, lib.fp8_last_error().decode(errors="replace"))
