"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol the
header declares, and its host-only logic (sizes, argument validation that returns
before any launch) behaves as documented.  No compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fp8train.h")


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__._build_module().build()
    from paper_2507_16099_b200 import _lib
    return _lib


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:[\w\s\*]+?)\b(fp8_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_north_star_calls():
    names = declared_functions()
    for n in ("fp8_amax", "fp8_cast_scaled", "fp8_linear_fwd", "fp8_linear_bwd", "fp8_fsdp_allgather"):
        assert n in names


def test_library_exports_every_declared_symbol(L):
    names = declared_functions()
    lib = ctypes.CDLL(L.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding covers exactly the declared surface
    assert sorted(L.SIGNATURES) == names


def test_abi_version(L):
    assert L.lib.fp8_abi_version() == 7


def test_sizes_host_only(L):
    cfg = L.LinearCfg(L.RECIPE_TENSORWISE, L.E4M3, L.E5M2, L.MX_FLOOR, L.DT_BF16)
    M, N, K = 16384, 14336, 4096
    saved = L.lib.fp8_linear_saved_bytes(ctypes.byref(cfg), M, N, K)
    assert saved >= K * M + K * N + 8
    ws = L.lib.fp8_linear_workspace_bytes(ctypes.byref(cfg), M, N, K)
    assert ws >= M * N  # backward holds the dY codes (read K-major by dX, MN-major by dW)
    cfg.recipe = L.RECIPE_ROWWISE
    assert L.lib.fp8_linear_workspace_bytes(ctypes.byref(cfg), M, N, K) >= 2 * M * N  # row- and column-scaled
    cfg.recipe = L.RECIPE_MXFP8
    assert L.lib.fp8_linear_saved_bytes(ctypes.byref(cfg), M, N, K) >= K * M + K * N + (K * M + K * N) // 32


def test_validation_returns_before_launch(L):
    # misaligned shape: rows % 16 != 0 -> FP8_EALIGN, no CUDA call made
    x = L.HP(16, L.DT_BF16, 100, 64, 64)
    t = L.Tensor8(16, None, 32, None, None, None, L.E4M3, L.GRAN_TENSOR, 100, 64)
    st = L.lib.fp8_cast_scaled(x, L.MX_FLOOR, None, ctypes.byref(t), None, 0, None)
    assert st == L.FP8_EALIGN
    assert b"multiples of 16" in L.lib.fp8_last_error()
    # MX needs multiples of 128
    x = L.HP(16, L.DT_BF16, 128, 96, 96)
    t = L.Tensor8(16, None, 32, None, None, None, L.E4M3, L.GRAN_MX32, 128, 96)
    assert L.lib.fp8_cast_scaled(x, L.MX_FLOOR, None, ctypes.byref(t), None, 0, None) == L.FP8_EALIGN
    # bad format
    t = L.Tensor8(16, None, 32, None, None, None, 7, L.GRAN_TENSOR, 128, 96)
    assert L.lib.fp8_cast_scaled(L.HP(16, L.DT_BF16, 128, 96, 96), 0, None, ctypes.byref(t), None, 0, None) == L.FP8_EINVAL
    # ld beyond 2^25 elements (the tile casts' 32-bit row offsets) -> FP8_EINVAL before any launch
    t = L.Tensor8(16, None, 32, None, None, None, L.E4M3, L.GRAN_TENSOR, 128, 96)
    assert L.lib.fp8_cast_scaled(L.HP(16, L.DT_BF16, 128, 96, (1 << 25) + 8), 0, None, ctypes.byref(t), None, 0,
                                 None) == L.FP8_EINVAL
    assert b"ld too large" in L.lib.fp8_last_error()
    # amax gran ROW_COL is not an amax unit
    assert L.lib.fp8_amax(L.HP(16, L.DT_BF16, 128, 96, 96), L.GRAN_ROW_COL, 16, None, 0, None) == L.FP8_EINVAL
    # GEMM K not multiple of 16
    assert L.lib.fp8_gemm(16, 0, 0, 32, 48, 0, 0, 64, L.GRAN_TENSOR, 128, 128, 40, 48, 48, 80, L.DT_BF16, 128,
                          None) == L.FP8_EALIGN
    # MX GEMM needs M, N, K multiples of 128 (either operand major)
    assert L.lib.fp8_gemm(16, 0, 1, 32, 48, 0, 0, 64, L.GRAN_MX32, 128, 128, 144, 128, 144, 80, L.DT_BF16, 128,
                          None) == L.FP8_EALIGN
    # linear: workspace too small
    cfg = L.LinearCfg(L.RECIPE_TENSORWISE, L.E4M3, L.E5M2, L.MX_FLOOR, L.DT_BF16)
    st = L.lib.fp8_linear_fwd(ctypes.byref(cfg), L.HP(16, L.DT_BF16, 128, 128, 128), L.HP(32, L.DT_BF16, 128, 128, 128),
                              None, 48, 64, 80, 10, None)
    assert st == L.FP8_EWORKSPACE
    # w_fp8 with the rowwise recipe is unsupported
    cfg.recipe = L.RECIPE_ROWWISE
    wq = L.Tensor8(16, None, 32, None, None, None, L.E4M3, L.GRAN_TENSOR, 128, 128)
    ws = L.lib.fp8_linear_workspace_bytes(ctypes.byref(cfg), 128, 128, 128)
    st = L.lib.fp8_linear_fwd(ctypes.byref(cfg), L.HP(16, L.DT_BF16, 128, 128, 128), L.HP(None, L.DT_BF16, 128, 128, 128),
                              ctypes.byref(wq), 48, 64, 80, ws, None)
    assert st == L.FP8_EUNSUPPORTED


def test_product_path_has_no_oracle_dependency():
    """The product package must not import the oracle or fall back to CPU math."""
    pkg = os.path.join(ROOT, "paper_2507_16099_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                s = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in s.replace("no oracle", ""), f
                assert "import numpy" not in s, f


def test_argument_errors_return_before_any_launch(L):
    """Documented error behaviour of the newer entry points: argument / shape checks return a status
    (and a message) before anything touches the device, so they run here without a GPU.  Fake but
    16-byte-aligned addresses stand in for device pointers (never dereferenced on these paths)."""
    A = 0x100000
    hp = lambda r, c: L.HP(A, L.DT_BF16, r, c, c)  # noqa: E731
    cfg = L.LinearCfg(L.RECIPE_MXFP8, L.E4M3, L.E5M2, L.MX_FLOOR, L.DT_BF16)
    ws = ctypes.c_void_p(A)
    # grouped GEMM: MXFP8 is not a grouped recipe; T and N alignment
    st = L.lib.fp8_grouped_linear_fwd(ctypes.byref(cfg), hp(256, 256), hp(512, 256), 2, ws, ws, ws, ws, 1 << 40, None)
    assert st == L.FP8_EUNSUPPORTED and b"grouped" in L.lib.fp8_last_error()
    cfg.recipe = L.RECIPE_ROWWISE
    st = L.lib.fp8_grouped_linear_fwd(ctypes.byref(cfg), hp(272, 256), hp(512, 256), 2, ws, ws, ws, ws, 1 << 40, None)
    assert st == L.FP8_EALIGN
    st = L.lib.fp8_grouped_linear_fwd(ctypes.byref(cfg), hp(256, 256), hp(288, 256), 2, ws, ws, ws, ws, 1 << 40, None)
    assert st == L.FP8_EALIGN   # N = 144 per expert
    st = L.lib.fp8_grouped_linear_fwd(ctypes.byref(cfg), hp(256, 256), hp(512, 256), 300, ws, ws, ws, ws, 1 << 40, None)
    assert st == L.FP8_EINVAL   # E > 256 (and w.rows % E != 0)
    # fused reduce-scatter / async-TP: null windows
    cfg.recipe = L.RECIPE_TENSORWISE
    st = L.lib.fp8_linear_bwd_rs(ctypes.byref(cfg), hp(256, 256), hp(256, 256), ws, None, ws, None, 2, ws, ws, 1 << 40,
                                 None)
    assert st == L.FP8_EINVAL
    st = L.lib.fp8_tp_linear_bwd(None, ws, None, ctypes.byref(cfg), hp(512, 256), 256, ws, ws, ws, 1 << 40, None)
    assert st == L.FP8_EINVAL
    # P2P windows: bad rank counts
    arr = (ctypes.c_void_p * 1)()
    assert L.lib.fp8_p2p_create_local(0, 1024, arr) == L.FP8_EINVAL
    assert L.lib.fp8_p2p_create_local(65, 1024, arr) == L.FP8_EINVAL
    assert L.lib.fp8_fsdp_allgather_p2p(None, hp(256, 256), L.E4M3, None, ws, ws, None) == L.FP8_EINVAL
    # MX scale re-tiling: alignment
    assert L.lib.fp8_mx_scales_unshard(ws, 2, 96, 256, ws, None) == L.FP8_EALIGN
    assert L.lib.fp8_mx_scales_unshard(ctypes.c_void_p(A + 8), 2, 128, 256, ws, None) == L.FP8_EALIGN
    # MX FSDP gather: only the row-major dim1 layout
    t8 = L.Tensor8(A, A, A, A, None, None, L.E4M3, L.GRAN_MX32, 256, 256)
    assert L.lib.fp8_fsdp_allgather_mx(ctypes.c_void_p(A), hp(128, 256), L.MX_FLOOR, ctypes.byref(t8), ws, 1 << 20,
                                       None) == L.FP8_EUNSUPPORTED
    # shared-input linears: member count, a member whose K differs, a too-small workspace (sized for
    # the widest member), a dY whose rows differ -- each caught before the first launch
    cfg.recipe = L.RECIPE_ROWWISE
    ptrs = (ctypes.c_void_p * 3)(A, A, A)
    ws3 = (L.HP * 3)(hp(256, 128), hp(512, 128), hp(128, 128))
    fwd = lambda n, w, wsb: L.lib.fp8_linear_fwd_shared(ctypes.byref(cfg), hp(256, 128), n, w, ptrs, ptrs, ws, wsb,  # noqa: E731
                                                        None)
    assert fwd(0, ws3, 1 << 40) == L.FP8_EINVAL
    assert fwd(9, ws3, 1 << 40) == L.FP8_EINVAL
    assert fwd(3, (L.HP * 3)(hp(256, 128), hp(512, 144), hp(128, 128)), 1 << 40) == L.FP8_EINVAL
    need = L.lib.fp8_linear_shared_workspace_bytes(ctypes.byref(cfg), 256, 128, 3, (ctypes.c_int64 * 3)(256, 512, 128))
    assert need >= L.lib.fp8_linear_workspace_bytes(ctypes.byref(cfg), 256, 896, 128) > 0   # every member's operands
    assert L.lib.fp8_linear_shared_workspace_bytes(ctypes.byref(cfg), 256, 128, 0, (ctypes.c_int64 * 3)()) == 0
    assert fwd(3, ws3, need - 1) == L.FP8_EWORKSPACE
    dys = (L.HP * 2)(hp(256, 256), hp(272, 512))
    assert L.lib.fp8_linear_bwd_shared(ctypes.byref(cfg), 2, dys, hp(256, 128), ptrs, ptrs, ptrs, ws, 1 << 40,
                                       None) == L.FP8_EINVAL


def test_shared_workspace_holds_batched_amax_scratch(L):
    """Rowwise shared-input groups cast X and every W_i (and every dY_i) in one batched launch, so their
    workspace holds, beside the members' FP8 operands, a row and a column amax slot per tensor:
    forward M + K + sum(N_i) + n K floats, backward n M + sum(N_i) floats (host-only size query)."""
    cfg = L.LinearCfg(L.RECIPE_ROWWISE, L.E4M3, L.E5M2, L.MX_FLOOR, L.DT_BF16)
    M, K, Ns = 1024, 512, (384, 128, 256)
    n, S = len(Ns), sum(Ns)
    need = L.lib.fp8_linear_shared_workspace_bytes(ctypes.byref(cfg), M, K, n, (ctypes.c_int64 * n)(*Ns))
    fwd_codes = M * K + S * K                      # X's and every W_i's forward codes
    bwd_codes = 2 * M * S                          # every dY_i's row- and column-scaled codes
    assert need >= fwd_codes + 4 * (M + K + S + n * K)
    assert need >= bwd_codes + 4 * (n * M + S)
    cfg.recipe = L.RECIPE_TENSORWISE               # no batched rowwise scratch for the other recipes
    assert L.lib.fp8_linear_shared_workspace_bytes(ctypes.byref(cfg), M, K, n, (ctypes.c_int64 * n)(*Ns)) < need


def test_knobs_host_only(L):
    """fp8_set_knob / fp8_get_knob / fp8_reset_knobs (host-only, no GPU): every knob the header documents
    exists with its documented default, out-of-range values and unknown names are rejected without
    changing anything, and reset restores the defaults.  The library never reads the environment."""
    import ctypes
    import re
    hdr = open(os.path.join(ROOT, "include", "fp8train.h")).read()
    block = hdr[hdr.index("Kernel-variant knobs"):hdr.index("fp8_status_t fp8_set_knob")]
    documented = dict((n, int(v)) for n, v in re.findall(r"([a-z0-9_]+) \((-?\d+)", block))
    assert {"gemm_kserp", "gemm_n512", "watchdog_ms", "tw_dual", "mx_transposed"} <= set(documented)
    L.lib.fp8_reset_knobs()
    v = ctypes.c_int(0)
    for name, default in documented.items():
        assert L.lib.fp8_get_knob(name.encode(), ctypes.byref(v)) == L.FP8_OK, name
        assert v.value == default, (name, v.value, default)
    assert L.lib.fp8_set_knob(b"gemm_n512", 1) == L.FP8_OK
    assert L.lib.fp8_set_knob(b"gemm_n512", 7) == L.FP8_EINVAL          # out of range: unchanged
    L.lib.fp8_get_knob(b"gemm_n512", ctypes.byref(v))
    assert v.value == 1
    assert L.lib.fp8_set_knob(b"no_such_knob", 1) == L.FP8_EINVAL
    L.lib.fp8_reset_knobs()
    L.lib.fp8_get_knob(b"gemm_n512", ctypes.byref(v))
    assert v.value == documented["gemm_n512"]
    assert L.lib.fp8_check_async_error() == L.FP8_OK
