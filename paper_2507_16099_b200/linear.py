"""Float8Linear: the paper's user surface over the C-ABI.

    convert(model, recipe="tensorwise")     # analog of convert_to_float8_training(model),
                                            # PAPER.md:614-615 (Appendix B, Listing)

swaps every eligible nn.Linear for a Float8Linear whose forward/backward run the
dynamically scaled FP8 step of §2.1 in libfp8train.so:
amax -> scale -> saturating RNE cast -> tcgen05 scaled GEMM, for Y, dX and dW.
"""

import torch
from torch import nn

from .ops import GroupedPlan, LinearPlan, SharedInputPlan


class _Plans:
    def __init__(self):
        self._p = {}

    def get(self, M, N, K, recipe, out_dtype, device):
        key = (M, N, K, recipe, out_dtype, str(device))
        if key not in self._p:
            self._p[key] = LinearPlan(M, N, K, recipe=recipe, out_dtype=out_dtype, device=device)
        return self._p[key]


_PLANS = _Plans()


class _Float8LinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x2d, w, recipe):
        M, K = x2d.shape
        N = w.shape[0]
        plan = _PLANS.get(M, N, K, recipe, torch.bfloat16, x2d.device)
        saved = plan.new_saved(x2d.device)
        x2d = x2d.contiguous()
        y = plan.forward(x2d, w.contiguous(), saved)
        ctx.plan, ctx.buf, ctx.wdtype = plan, saved, w.dtype
        # rowwise_gw_hp keeps dL/dW in bf16: its BF16 dW GEMM reads the hp input in
        # bf16 (a bf16 copy when the activations are fp32; the forward casts still read x2d itself).
        # Saved through save_for_backward, so an in-place change of x before backward raises.
        ctx.gw_hp = recipe == "rowwise_gw_hp"
        if ctx.gw_hp:
            ctx.save_for_backward(x2d if x2d.dtype == torch.bfloat16 else x2d.to(torch.bfloat16))
        return y

    @staticmethod
    def backward(ctx, dy):
        x_hp = None
        if ctx.gw_hp:
            (x_hp,) = ctx.saved_tensors
            if dy.dtype != torch.bfloat16:
                dy = dy.to(torch.bfloat16)
        dx, dw = ctx.plan.backward(dy.contiguous(), ctx.buf, want_dx=ctx.needs_input_grad[0],
                                   want_dw=ctx.needs_input_grad[1], x=x_hp)
        if dw is not None and dw.dtype != ctx.wdtype:
            dw = dw.to(ctx.wdtype)
        return dx, dw, None


class Float8Linear(nn.Linear):
    """nn.Linear whose matmuls run as dynamically scaled FP8 (Appendix A recipes)."""

    def __init__(self, in_features, out_features, bias=False, recipe="tensorwise", device=None, dtype=None):
        super().__init__(in_features, out_features, bias=bias, device=device, dtype=dtype)
        self.recipe = recipe

    def forward(self, x):
        shp = x.shape
        x2d = x.reshape(-1, shp[-1])
        if x2d.dtype != torch.bfloat16 and x2d.dtype != torch.float32:
            x2d = x2d.to(torch.bfloat16)
        if not torch.is_grad_enabled() or not (x2d.requires_grad or self.weight.requires_grad):
            # forward-only FP8 (inference): no backward operands are cast or kept
            M, K = x2d.shape
            plan = _PLANS.get(M, self.out_features, K, self.recipe, torch.bfloat16, x2d.device)
            y = plan.forward(x2d.contiguous(), self.weight.detach().contiguous(), None)
        else:
            y = _Float8LinearFn.apply(x2d, self.weight, self.recipe)
        if self.bias is not None:
            y = y + self.bias.to(y.dtype)
        return y.reshape(*shp[:-1], self.out_features)

    @classmethod
    def from_linear(cls, lin, recipe):
        new = cls(lin.in_features, lin.out_features, bias=lin.bias is not None, recipe=recipe,
                  device=lin.weight.device, dtype=lin.weight.dtype)
        with torch.no_grad():
            new.weight.copy_(lin.weight)
            if lin.bias is not None:
                new.bias.copy_(lin.bias)
        return new


def _eligible(lin, recipe):
    q = 128 if recipe == "mxfp8" else 16
    return lin.in_features % q == 0 and lin.out_features % q == 0


def convert(model, recipe="tensorwise", module_filter_fn=None):
    """Swap nn.Linear -> Float8Linear in place (dims must be multiples of 16, 128 for mxfp8)."""
    for name, child in list(model.named_children()):
        if isinstance(child, nn.Linear) and not isinstance(child, Float8Linear):
            if _eligible(child, recipe) and (module_filter_fn is None or module_filter_fn(child, name)):
                setattr(model, name, Float8Linear.from_linear(child, recipe))
        else:
            convert(child, recipe, module_filter_fn)
    return model


# ------------------------------------------------------------------ shared-input linears

class _SharedPlans:
    def __init__(self):
        self._p = {}

    def get(self, M, Ns, K, recipe, device):
        key = (M, tuple(Ns), K, recipe, str(device))
        if key not in self._p:
            self._p[key] = SharedInputPlan(M, Ns, K, recipe=recipe, out_dtype=torch.bfloat16, device=device)
        return self._p[key]


_SPLANS = _SharedPlans()


class _SharedInputFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x2d, recipe, *ws):
        M, K = x2d.shape
        plan = _SPLANS.get(M, [w.shape[0] for w in ws], K, recipe, x2d.device)
        saved = plan.new_saved(x2d.device)
        x2d = x2d.contiguous()
        ys = plan.forward(x2d, [w.contiguous() for w in ws], saved)
        ctx.plan, ctx.buf, ctx.wdtypes = plan, saved, [w.dtype for w in ws]
        ctx.gw_hp = recipe == "rowwise_gw_hp"
        if ctx.gw_hp:
            ctx.save_for_backward(x2d if x2d.dtype == torch.bfloat16 else x2d.to(torch.bfloat16))
        return tuple(ys)

    @staticmethod
    def backward(ctx, *dys):
        x_hp = None
        if ctx.gw_hp:
            (x_hp,) = ctx.saved_tensors
        dys = [d.to(torch.bfloat16).contiguous() for d in dys]   # (unused outputs arrive as zeros)
        want_dw = any(ctx.needs_input_grad[2:])
        dxs, dws = ctx.plan.backward(dys, ctx.buf, x=x_hp, want_dx=ctx.needs_input_grad[0], want_dw=want_dw)
        dx = None
        if dxs is not None:   # X feeds every member: its gradient is the members' sum (in member order)
            dx = dxs[0]
            for d in dxs[1:]:
                dx = dx + d
        grads = [None] * len(ctx.wdtypes)
        if dws is not None:
            grads = [dw if dw.dtype == t else dw.to(t) for dw, t in zip(dws, ctx.wdtypes)]
        return (dx, None, *grads)


def shared_input_linears(x, linears):
    """Y_i = Float8Linear_i(x) for linears that read the same x (a layer's wq/wk/wv, w1/w3): X's amax
    and FP8 copies are computed once and the members' GEMMs run as one launch per pass
    (fp8_linear_fwd_shared / _bwd_shared).  Each Y_i, dW_i and dX_i is bit-identical to the separate
    Float8Linear's; dX = sum of the dX_i in member order.  `linears`: Float8Linear modules with one
    recipe and no bias.  Returns a tuple of outputs shaped like x with the last dim N_i."""
    recipe = linears[0].recipe
    if any(lin.recipe != recipe or lin.bias is not None for lin in linears):
        raise ValueError("shared_input_linears: one recipe, no bias")
    shp = x.shape
    x2d = x.reshape(-1, shp[-1])
    if x2d.dtype != torch.bfloat16 and x2d.dtype != torch.float32:
        x2d = x2d.to(torch.bfloat16)
    ys = _SharedInputFn.apply(x2d, recipe, *[lin.weight for lin in linears])
    return tuple(y.reshape(*shp[:-1], y.shape[-1]) for y in ys)


# ----------------------------------------------------------------------------- MoE

class _GroupedPlans:
    def __init__(self):
        self._p = {}

    def get(self, T, E, N, K, recipe, device):
        key = (T, E, N, K, recipe, str(device))
        if key not in self._p:
            self._p[key] = GroupedPlan(T, E, N, K, recipe=recipe, out_dtype=torch.bfloat16, device=device)
        return self._p[key]


_GPLANS = _GroupedPlans()


class _ScaledGroupedMMFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, offs, recipe):
        T, K = x.shape
        E, N, _ = w.shape
        plan = _GPLANS.get(T, E, N, K, recipe, x.device)
        saved = plan.new_saved(x.device)
        y = plan.forward(x.contiguous(), w.reshape(E * N, K).contiguous(), offs, saved)
        ctx.plan, ctx.buf, ctx.offs, ctx.wshape, ctx.wdtype = plan, saved, offs, w.shape, w.dtype
        return y

    @staticmethod
    def backward(ctx, dy):
        dx, dw = ctx.plan.backward(dy.contiguous(), ctx.offs, ctx.buf, want_dx=ctx.needs_input_grad[0],
                                   want_dw=ctx.needs_input_grad[1])
        if dw is not None:
            dw = dw.view(ctx.wshape)
            if dw.dtype != ctx.wdtype:
                dw = dw.to(ctx.wdtype)
        return dx, dw, None, None


def scaled_grouped_mm(x, w, offs, recipe="rowwise"):
    """Differentiable FP8 scaled grouped GEMM for MoE training (reading R-c22):
    out[offs[g]:offs[g+1]] = x[offs[g]:offs[g+1]] @ w[g].T for every expert g, each GEMM (and its
    backward dX, dW) in FP8 with the recipe's dynamic scaling, in one grouped launch per pass.
      x [T, K] bf16 tokens sorted by expert; w [E, N, K] bf16 expert weights (nn.Linear layout);
      offs int32 [E+1] on the device (offs[0] = 0, offs[E] = T, multiples of 128, non-decreasing).
    Returns out [T, N] bf16."""
    if x.dtype != torch.bfloat16:
        x = x.to(torch.bfloat16)
    return _ScaledGroupedMMFn.apply(x, w, offs, recipe)
