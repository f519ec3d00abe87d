"""Torch-facing wrappers of the C-ABI: argument marshalling only.

Every step of the path runs in libfp8train.so; torch provides device memory and
the current CUDA stream.  Names follow the paper's recipe vocabulary (Appendix A,
PAPER.md:594-598): tensorwise / rowwise / mxfp8, e4m3 forward / e5m2 gradients.
"""

import ctypes

import torch

from . import _lib as L

FORMATS = {"e4m3": L.E4M3, "e5m2": L.E5M2}
GRANS = {"tensor": L.GRAN_TENSOR, "row": L.GRAN_ROW, "col": L.GRAN_COL, "row_col": L.GRAN_ROW_COL,
         "mx32": L.GRAN_MX32, "mx32_rm": L.GRAN_MX32_RM}
RECIPES = {"tensorwise": L.RECIPE_TENSORWISE, "rowwise": L.RECIPE_ROWWISE, "mxfp8": L.RECIPE_MXFP8,
           "rowwise_gw_hp": L.RECIPE_ROWWISE_GW_HP}
MX_ROUND = {"floor": L.MX_FLOOR, "rceil": L.MX_RCEIL}


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def hp(x):
    """fp8_hp_t view of a 2-D row-major fp32/bf16 CUDA tensor (unit column stride)."""
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("expected a 2-D tensor with unit column stride")
    if x.dtype == torch.bfloat16:
        dt = L.DT_BF16
    elif x.dtype == torch.float32:
        dt = L.DT_F32
    else:
        raise TypeError(f"unsupported dtype {x.dtype}")
    if not x.is_cuda:
        raise ValueError("tensor must be on a CUDA device (no CPU fallback)")
    return L.HP(x.data_ptr(), dt, x.shape[0], x.shape[1], x.stride(0))


def sf_bytes(rows, cols):
    """Bytes of an E8M0 blocked scale buffer for an MX operand [rows, cols]."""
    return rows * cols // 32


def amax(x, gran="tensor", stream=None):
    n = {"tensor": 1, "row": x.shape[0], "col": x.shape[1]}[gran]
    out = torch.empty(n, dtype=torch.float32, device=x.device)
    L.check(L.lib.fp8_amax(hp(x), GRANS[gran], _ptr(out), None, 0, _stream(stream)), "fp8_amax")
    return out


def amax_multi(xs, out=None, stream=None):
    """fp8_amax_multi: tensorwise amax of every tensor in `xs` in one launch (per 48 tensors).
    Returns float32 [len(xs)]."""
    n = len(xs)
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=xs[0].device)
    for i in range(0, n, L.AMAX_MULTI_MAX):
        part = xs[i:i + L.AMAX_MULTI_MAX]
        arr = (L.HP * len(part))(*[hp(x) for x in part])
        L.check(L.lib.fp8_amax_multi(arr, len(part), ctypes.c_void_p(out.data_ptr() + 4 * i), _stream(stream)),
                "fp8_amax_multi")
    return out


def cast(x, fmt="e4m3", gran="tensor", want_q=True, want_qt=False, mx_round="floor", amax_in=None,
         stream=None):
    """fp8_cast_scaled.  Returns a dict with q [R,C] / q_t [C,R] (uint8), scale(s), amax.
    gran "mx32_rm": q_t holds the dim1 codes in the input's layout [R,C] (not transposed)."""
    R, C = x.shape
    dev = x.device
    out = {"q": None, "q_t": None, "scale": None, "scale_t": None, "amax": None, "amax_t": None}
    if want_q:
        out["q"] = torch.empty((R, C), dtype=torch.uint8, device=dev)
    if want_qt:
        out["q_t"] = torch.empty((R, C) if gran == "mx32_rm" else (C, R), dtype=torch.uint8, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    if gran in ("mx32", "mx32_rm"):
        if want_q:
            out["scale"] = torch.empty(sf_bytes(R, C), dtype=torch.uint8, device=dev)
        if want_qt:
            out["scale_t"] = torch.empty(sf_bytes(C, R), dtype=torch.uint8, device=dev)
    elif gran == "row_col":
        out["scale"], out["amax"] = torch.empty(R, **f32), torch.empty(R, **f32)
        out["scale_t"], out["amax_t"] = torch.empty(C, **f32), torch.empty(C, **f32)
    else:
        n = {"tensor": 1, "row": R, "col": C}[gran]
        out["scale"], out["amax"] = torch.empty(n, **f32), torch.empty(n, **f32)
        if amax_in is not None:
            out["amax"] = None
    t = L.Tensor8(*[(out[k].data_ptr() if out[k] is not None else None)
                    for k in ("q", "q_t", "scale", "scale_t", "amax", "amax_t")],
                  FORMATS[fmt], GRANS[gran], R, C)
    h = hp(x)
    wsb = L.lib.fp8_cast_workspace_bytes(h, GRANS[gran])
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    L.check(L.lib.fp8_cast_scaled(h, MX_ROUND[mx_round], _ptr(amax_in), ctypes.byref(t), _ptr(ws), wsb,
                                  _stream(stream)), "fp8_cast_scaled")
    return out


def gemm(A, fmt_a, sa, B, fmt_b, sb, gran="tensor", out_dtype=torch.bfloat16, a_mn=False, b_mn=False,
         stream=None):
    """D = A B^T with scales (fp8_gemm).  K-major: A [M,K], B [N,K]; MN-major (a_mn / b_mn):
    A stored [K,M], B stored [K,N].  uint8 codes."""
    M = A.shape[1] if a_mn else A.shape[0]
    K = A.shape[0] if a_mn else A.shape[1]
    N = B.shape[1] if b_mn else B.shape[0]
    D = torch.empty((M, N), dtype=out_dtype, device=A.device)
    od = L.DT_F32 if out_dtype == torch.float32 else L.DT_BF16
    L.check(L.lib.fp8_gemm(_ptr(A), FORMATS[fmt_a], int(a_mn), _ptr(sa), _ptr(B), FORMATS[fmt_b], int(b_mn),
                           _ptr(sb), GRANS[gran], M, N, K, A.stride(0), B.stride(0), _ptr(D), od, D.stride(0),
                           _stream(stream)), "fp8_gemm")
    return D


def linear_backward_rs(plan, dy, saved, rs_win, dw_shard, dx=None, want_dx=True, w_fp8=None, x=None, stream=None):
    """fp8_linear_bwd_rs: the backward with dW reduce-scattered to its row shards by the dW GEMM's
    epilogue over the P2P window `rs_win` (fsdp.P2PWindow); dw_shard [N/nranks, K] bf16 receives this
    rank's summed shard.  Returns dx."""
    if want_dx and dx is None:
        dx = torch.empty((plan.M, plan.K), dtype=plan.out_dtype, device=dy.device)
    wq = plan._wq(w_fp8)
    xh = hp(x) if x is not None else L.HP(None, L.DT_BF16, plan.M, plan.K, plan.K)
    L.check(L.lib.fp8_linear_bwd_rs(ctypes.byref(plan.cfg), hp(dy), xh, _ptr(saved), ctypes.byref(wq) if wq else None,
                                    _ptr(dx) if want_dx else None, rs_win._h, rs_win.world, _ptr(dw_shard),
                                    _ptr(plan.ws), plan.ws_bytes, _stream(stream)), "fp8_linear_bwd_rs")
    return dx


def mx_scales_unshard(rank_major, nranks, rows_local, cols, out=None, stream=None):
    """fp8_mx_scales_unshard: nranks shard-local blocked dim1 E8M0 buffers ([cols, rows_local/32]
    each, concatenated) -> the blocked buffer of the full [cols, nranks*rows_local/32] matrix."""
    if out is None:
        out = torch.empty_like(rank_major)
    L.check(L.lib.fp8_mx_scales_unshard(_ptr(rank_major), nranks, rows_local, cols, _ptr(out), _stream(stream)),
            "fp8_mx_scales_unshard")
    return out


class LinearPlan:
    """Sizes and buffers for one Float8Linear shape (caller-owned, as the ABI requires)."""

    def __init__(self, M, N, K, recipe="tensorwise", fmt_fwd="e4m3", fmt_grad="e5m2", mx_round="floor",
                 out_dtype=torch.bfloat16, device="cuda"):
        self.M, self.N, self.K = M, N, K
        self.out_dtype = out_dtype
        self.cfg = L.LinearCfg(RECIPES[recipe], FORMATS[fmt_fwd], FORMATS[fmt_grad], MX_ROUND[mx_round],
                               L.DT_F32 if out_dtype == torch.float32 else L.DT_BF16)
        self.saved_bytes = L.lib.fp8_linear_saved_bytes(ctypes.byref(self.cfg), M, N, K)
        self.ws_bytes = L.lib.fp8_linear_workspace_bytes(ctypes.byref(self.cfg), M, N, K)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)

    def new_saved(self, device="cuda"):
        return torch.empty(self.saved_bytes, dtype=torch.uint8, device=device)

    def _wq(self, w_fp8):
        if w_fp8 is None:
            return None
        if isinstance(w_fp8, dict):   # MXFP8 gather (Comm.allgather_mx): q/scale dim0, q_t/scale_t dim1
            return L.Tensor8(*[(w_fp8[k].data_ptr() if w_fp8.get(k) is not None else None)
                               for k in ("q", "q_t", "scale", "scale_t")], None, None, self.cfg.fmt_fwd,
                             L.GRAN_MX32_RM, self.N, self.K)
        q, s = w_fp8
        return L.Tensor8(q.data_ptr(), None, s.data_ptr(), None, None, None, self.cfg.fmt_fwd, L.GRAN_TENSOR,
                         self.N, self.K)

    def forward(self, x, w, saved, y=None, w_fp8=None, x_amax=None, y_amax=None, stream=None):
        """w_fp8: optional pre-cast weight: tensorwise (codes [N,K] uint8, scale float[1]) from
        Comm.allgather_fp8, or the mxfp8 dict of Comm.allgather_mx.
        saved=None: forward-only (inference) -- nothing is kept for a backward.
        x_amax: optional precomputed amax(|X|) (float[1]); y_amax: optional float[1] that receives
        amax(|Y|) from the GEMM epilogue."""
        if y is None:
            y = torch.empty((self.M, self.N), dtype=self.out_dtype, device=x.device)
        wq = self._wq(w_fp8)
        wh = hp(w) if w is not None else L.HP(None, L.DT_BF16, self.N, self.K, self.K)
        ws, wsb = self.ws, self.ws_bytes
        if saved is None:
            wsb = L.lib.fp8_linear_infer_workspace_bytes(ctypes.byref(self.cfg), self.M, self.N, self.K)
            if wsb > self.ws_bytes:
                ws = torch.empty(wsb, dtype=torch.uint8, device=x.device)
        L.check(L.lib.fp8_linear_fwd_ex(ctypes.byref(self.cfg), hp(x), _ptr(x_amax), wh,
                                        ctypes.byref(wq) if wq else None, _ptr(y), _ptr(y_amax), _ptr(saved),
                                        _ptr(ws), wsb, _stream(stream)), "fp8_linear_fwd_ex")
        return y

    def buffers(self, saved):
        """fp8_linear_buffers: uint8 / float32 views of the FP8 operands, scales and amaxes inside
        `saved` and this plan's workspace (what the forward / backward wrote; see fp8train.h)."""
        b = L.LinearBuffers()
        L.check(L.lib.fp8_linear_buffers(ctypes.byref(self.cfg), self.M, self.N, self.K, _ptr(saved),
                                         _ptr(self.ws), ctypes.byref(b)), "fp8_linear_buffers")
        M, N, K = self.M, self.N, self.K
        rec = self.cfg.recipe
        mx = rec == L.RECIPE_MXFP8

        def view(ptr, nbytes, dtype=torch.uint8, shape=None):
            if not ptr:
                return None
            for base in (saved, self.ws):
                off = ptr - base.data_ptr()
                if 0 <= off and off + nbytes <= base.numel():
                    t = base[off:off + nbytes]
                    t = t.view(dtype) if dtype != torch.uint8 else t
                    return t.view(shape) if shape is not None else t
            raise RuntimeError("fp8_linear_buffers: pointer outside saved / ws")

        def scale(ptr, n):   # n floats (tensorwise / rowwise) or n E8M0 bytes (mx)
            return view(ptr, n, torch.uint8) if mx else view(ptr, 4 * n, torch.float32)

        tw = rec == L.RECIPE_TENSORWISE
        tr = bool(b.bwd_transposed)
        out = {
            "x_fwd": view(b.x_fwd, M * K, shape=(M, K)), "w_fwd": view(b.w_fwd, N * K, shape=(N, K)),
            "x_bwd": view(b.x_bwd, M * K, shape=(K, M) if tr else (M, K)),
            "w_bwd": view(b.w_bwd, N * K, shape=(K, N) if tr else (N, K)),
            "dy_dx": view(b.dy_dx, M * N, shape=(M, N)),
            "dy_dw": view(b.dy_dw, M * N, shape=(N, M) if tr else (M, N)),
            "bwd_transposed": tr,
        }
        if mx:
            out.update(x_fwd_scale=scale(b.x_fwd_scale, M * K // 32), w_fwd_scale=scale(b.w_fwd_scale, N * K // 32),
                       x_bwd_scale=scale(b.x_bwd_scale, M * K // 32), w_bwd_scale=scale(b.w_bwd_scale, N * K // 32),
                       dy_dx_scale=scale(b.dy_dx_scale, M * N // 32), dy_dw_scale=scale(b.dy_dw_scale, M * N // 32),
                       amax_fwd=None, amax_bwd=None)
        elif tw:
            out.update(x_fwd_scale=scale(b.x_fwd_scale, 1), w_fwd_scale=scale(b.w_fwd_scale, 1),
                       x_bwd_scale=scale(b.x_bwd_scale, 1), w_bwd_scale=scale(b.w_bwd_scale, 1),
                       dy_dx_scale=scale(b.dy_dx_scale, 1), dy_dw_scale=scale(b.dy_dw_scale, 1),
                       amax_fwd=scale(b.amax_fwd, 2), amax_bwd=scale(b.amax_bwd, 1))
        else:
            out.update(x_fwd_scale=scale(b.x_fwd_scale, M), w_fwd_scale=scale(b.w_fwd_scale, N),
                       x_bwd_scale=scale(b.x_bwd_scale, K), w_bwd_scale=scale(b.w_bwd_scale, K),
                       dy_dx_scale=scale(b.dy_dx_scale, M), dy_dw_scale=scale(b.dy_dw_scale, N),
                       amax_fwd=scale(b.amax_fwd, M + K + N + K), amax_bwd=scale(b.amax_bwd, M + N))
        return out

    def backward(self, dy, saved, dx=None, dw=None, want_dx=True, want_dw=True, w_fp8=None, x=None,
                 dy_amax=None, dx_amax=None, stream=None):
        """x: the forward input (read by rowwise_gw_hp's BF16 dW GEMM only); dy_amax / dx_amax: amax
        hand-over as in forward()."""
        dev = dy.device
        if want_dx and dx is None:
            dx = torch.empty((self.M, self.K), dtype=self.out_dtype, device=dev)
        if want_dw and dw is None:
            dw = torch.empty((self.N, self.K), dtype=self.out_dtype, device=dev)
        wq = self._wq(w_fp8)
        xh = hp(x) if x is not None else L.HP(None, L.DT_BF16, self.M, self.K, self.K)
        L.check(L.lib.fp8_linear_bwd_ex(ctypes.byref(self.cfg), hp(dy), _ptr(dy_amax), xh, _ptr(saved),
                                        ctypes.byref(wq) if wq else None, _ptr(dx) if want_dx else None,
                                        _ptr(dx_amax), _ptr(dw) if want_dw else None, _ptr(self.ws), self.ws_bytes,
                                        _stream(stream)), "fp8_linear_bwd_ex")
        return dx, dw


class SharedInputPlan:
    """Float8Linears that read the same input X (fp8_linear_fwd_shared / _bwd_shared): e.g. wq/wk/wv
    or w1/w3 of a Llama layer.  X is cast once; outputs and saved bytes equal those of separate
    LinearPlan calls.  One workspace for the group (fp8_linear_shared_workspace_bytes); the members'
    GEMMs run as one launch per pass."""

    def __init__(self, M, Ns, K, recipe="tensorwise", fmt_fwd="e4m3", fmt_grad="e5m2", mx_round="floor",
                 out_dtype=torch.bfloat16, device="cuda"):
        self.M, self.Ns, self.K = M, list(Ns), K
        self.out_dtype = out_dtype
        self.cfg = L.LinearCfg(RECIPES[recipe], FORMATS[fmt_fwd], FORMATS[fmt_grad], MX_ROUND[mx_round],
                               L.DT_F32 if out_dtype == torch.float32 else L.DT_BF16)
        self.saved_bytes = [L.lib.fp8_linear_saved_bytes(ctypes.byref(self.cfg), M, N, K) for N in self.Ns]
        ns = (ctypes.c_int64 * len(self.Ns))(*self.Ns)
        self.ws_bytes = L.lib.fp8_linear_shared_workspace_bytes(ctypes.byref(self.cfg), M, K, len(self.Ns), ns)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)

    def new_saved(self, device="cuda"):
        return [torch.empty(b, dtype=torch.uint8, device=device) for b in self.saved_bytes]

    @staticmethod
    def _ptrs(ts):
        return (ctypes.c_void_p * len(ts))(*[_ptr(t) for t in ts])

    def forward(self, x, ws_, saved, ys=None, stream=None):
        """x [M,K]; ws_: list of weights [N_i, K]; saved: list from new_saved(); returns the list of Y_i."""
        n = len(self.Ns)
        if ys is None:
            ys = [torch.empty((self.M, N), dtype=self.out_dtype, device=x.device) for N in self.Ns]
        whs = (L.HP * n)(*[hp(w) for w in ws_])
        L.check(L.lib.fp8_linear_fwd_shared(ctypes.byref(self.cfg), hp(x), n, whs, self._ptrs(ys), self._ptrs(saved),
                                            _ptr(self.ws), self.ws_bytes, _stream(stream)), "fp8_linear_fwd_shared")
        return ys

    def backward(self, dys, saved, dxs=None, dws=None, x=None, want_dx=True, want_dw=True, stream=None):
        """dys: list of dY_i [M, N_i]; returns (list of dX_i [M,K], list of dW_i [N_i,K]) -- the caller
        sums the dX_i (as autograd does for separate linears)."""
        n = len(self.Ns)
        dev = dys[0].device
        if want_dx and dxs is None:
            dxs = [torch.empty((self.M, self.K), dtype=self.out_dtype, device=dev) for _ in range(n)]
        if want_dw and dws is None:
            dws = [torch.empty((N, self.K), dtype=self.out_dtype, device=dev) for N in self.Ns]
        dyh = (L.HP * n)(*[hp(d) for d in dys])
        xh = hp(x) if x is not None else L.HP(None, L.DT_BF16, self.M, self.K, self.K)
        L.check(L.lib.fp8_linear_bwd_shared(ctypes.byref(self.cfg), n, dyh, xh, self._ptrs(saved),
                                            self._ptrs(dxs) if want_dx else None,
                                            self._ptrs(dws) if want_dw else None, _ptr(self.ws), self.ws_bytes,
                                            _stream(stream)), "fp8_linear_bwd_shared")
        return dxs, dws


class GroupedPlan:
    """MoE scaled grouped GEMM (fp8_grouped_linear_fwd / _bwd): E experts with
    weights stacked [E*N, K], tokens [T, K] sorted by expert, device int32 offsets [E+1]."""

    def __init__(self, T, E, N, K, recipe="rowwise", fmt_fwd="e4m3", fmt_grad="e5m2", out_dtype=torch.bfloat16,
                 device="cuda"):
        self.T, self.E, self.N, self.K = T, E, N, K
        self.out_dtype = out_dtype
        self.cfg = L.LinearCfg(RECIPES[recipe], FORMATS[fmt_fwd], FORMATS[fmt_grad], L.MX_FLOOR,
                               L.DT_F32 if out_dtype == torch.float32 else L.DT_BF16)
        self.saved_bytes = L.lib.fp8_grouped_saved_bytes(ctypes.byref(self.cfg), T, E, N, K)
        self.ws_bytes = L.lib.fp8_grouped_workspace_bytes(ctypes.byref(self.cfg), T, E, N, K)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)

    def new_saved(self, device="cuda"):
        return torch.empty(self.saved_bytes, dtype=torch.uint8, device=device)

    def forward(self, x, w, offs, saved, y=None, stream=None):
        if y is None:
            y = torch.empty((self.T, self.N), dtype=self.out_dtype, device=x.device)
        if offs.dtype != torch.int32 or not offs.is_cuda:
            raise TypeError("offs must be a CUDA int32 tensor [E+1]")
        L.check(L.lib.fp8_grouped_linear_fwd(ctypes.byref(self.cfg), hp(x), hp(w), self.E, _ptr(offs), _ptr(y),
                                             _ptr(saved), _ptr(self.ws), self.ws_bytes, _stream(stream)),
                "fp8_grouped_linear_fwd")
        return y

    def backward(self, dy, offs, saved, dx=None, dw=None, want_dx=True, want_dw=True, stream=None):
        dev = dy.device
        if want_dx and dx is None:
            dx = torch.empty((self.T, self.K), dtype=self.out_dtype, device=dev)
        if want_dw and dw is None:
            dw = torch.empty((self.E * self.N, self.K), dtype=self.out_dtype, device=dev)
        xh = L.HP(None, L.DT_BF16, self.T, self.K, self.K)
        L.check(L.lib.fp8_grouped_linear_bwd(ctypes.byref(self.cfg), hp(dy), xh, self.E, _ptr(offs),
                                             _ptr(saved), _ptr(dx) if want_dx else None,
                                             _ptr(dw) if want_dw else None, _ptr(self.ws), self.ws_bytes,
                                             _stream(stream)), "fp8_grouped_linear_bwd")
        return dx, dw


def launch_count():
    return int(L.lib.fp8_launch_count())


def set_knob(name, value):
    """fp8_set_knob: select a kernel variant (A/B experiments, tests); defaults are the product path."""
    L.check(L.lib.fp8_set_knob(name.encode(), int(value)), "fp8_set_knob")


def get_knob(name):
    v = ctypes.c_int(0)
    L.check(L.lib.fp8_get_knob(name.encode(), ctypes.byref(v)), "fp8_get_knob")
    return v.value


def reset_knobs():
    L.lib.fp8_reset_knobs()


class knobs:
    """Context manager: ``with ops.knobs(gemm_sched=0): ...`` sets knobs and restores them on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_knob(k)
            set_knob(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_knob(k, v)
        return False
