"""Glue between planned operators, on this package's kernels: fused
residual-add + LayerNorm (the post-LN of every encoder sublayer) and the
attention core (softmax(Q K^T scale) V on the packed QKV, csrc/attn.cu)."""
from __future__ import annotations

import torch

from . import ops


class _AddLayerNorm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b, gamma, beta, eps):
        a = a.contiguous()
        b = b.contiguous() if b is not None else None
        y, s, mean, rstd = ops.layernorm_fwd(a, b, gamma, beta, eps)
        ctx.save_for_backward(s, mean, rstd)
        ctx.g_ref, ctx.b_ref = gamma, beta
        ctx.b_dtype = b.dtype if b is not None else None
        return y

    @staticmethod
    def backward(ctx, dy):
        s, mean, rstd = ctx.saved_tensors
        gamma, beta = ctx.g_ref, ctx.b_ref
        mg = getattr(gamma, "main_grad", None)
        mb = getattr(beta, "main_grad", None)
        dg = mg if mg is not None else torch.zeros_like(gamma)
        db = mb if mb is not None else torch.zeros_like(beta)
        dx = ops.layernorm_bwd(dy.contiguous(), s, mean, rstd, gamma, dg, db)
        grad_b = None
        if ctx.b_dtype is not None:
            grad_b = dx if ctx.b_dtype == torch.float32 else ops.cast(dx, ctx.b_dtype)
        return dx, grad_b, (None if mg is not None else dg), (None if mb is not None else db), None


class _Gelu(torch.autograd.Function):
    """GELU (erf form) on this package's kernel, the one the fused layer uses
    (common.cuh gelu_and_grad): y in x's dtype; the backward multiplies by the
    FP16 GELU'(x) the forward stored (the fused layer's backward does the same)."""

    @staticmethod
    def forward(ctx, x):
        x = x.contiguous()
        # a BF16 op's output: GELU in FP32, rounded once to BF16 (as torch's bf16 GELU)
        if x.dtype == torch.bfloat16:
            y, d = ops.act_cast(ops.cast(x, torch.float32), torch.float32, ops.ACT_GELU, want_dact=True)
            y = ops.cast(y, torch.bfloat16)
        else:
            y, d = ops.act_cast(x, x.dtype, ops.ACT_GELU, want_dact=True)
        ctx.save_for_backward(d)
        return y

    @staticmethod
    def backward(ctx, dy):
        (d,) = ctx.saved_tensors
        if dy.dtype == torch.bfloat16:
            g = ops.act_bwd_colsum(ops.cast(dy.contiguous(), torch.float32), d, ops.ACT_DERIV,
                                   out_dtype=torch.float32)
            return ops.cast(g, torch.bfloat16)
        return ops.act_bwd_colsum(dy.contiguous(), d, ops.ACT_DERIV, out_dtype=dy.dtype)


def gelu(x: torch.Tensor) -> torch.Tensor:
    return _Gelu.apply(x)


class _ClsHead(torch.autograd.Function):
    """Pooler (tanh) + classifier + mean cross entropy on this package's
    kernels (csrc/head.cu).  The weight gradients are ADDED into each
    parameter's ``main_grad`` when it has one (the flat buffer), and reported
    final through qlinear.GRAD_READY as the fused layers do."""

    @staticmethod
    def forward(ctx, x, wp, bp, wc, bc, labels):
        x = x.contiguous()
        loss, pooled, probs = ops.cls_head_fwd(x, wp, bp, wc, bc, labels)
        ctx.save_for_backward(x, pooled, probs, labels)
        ctx.params = (wp, bp, wc, bc)
        return loss.reshape(())

    @staticmethod
    def backward(ctx, dloss):
        from . import qlinear as _ql
        from .fused import _mark
        _mark("bwd", "loss")
        x, pooled, probs, labels = ctx.saved_tensors
        params = ctx.params
        outs = [getattr(p, "main_grad", None) for p in params]
        bufs = [o if o is not None else torch.zeros_like(p) for o, p in zip(outs, params)]
        wp, _, wc, _ = params
        dx = ops.cls_head_bwd(x, wp, wc, labels, pooled, probs, dloss.reshape(1).contiguous(), *bufs)
        if _ql.GRAD_READY is not None:
            _ql.GRAD_READY([p for p, o in zip(params, outs) if o is not None])
        return (dx,) + tuple(None if o is not None else b for o, b in zip(outs, bufs)) + (None,)


def cls_head(x: torch.Tensor, pooler, cls, labels: torch.Tensor) -> torch.Tensor:
    """Mean cross-entropy loss of cls(tanh(pooler(x[:, 0]))) -- FP32 pooler."""
    return _ClsHead.apply(x, pooler.weight, pooler.bias, cls.weight, cls.bias, labels)


class AddLayerNorm(torch.nn.Module):
    """y = LayerNorm(a + b) with FP32 statistics; b may be FP32 or FP16."""

    def __init__(self, hidden: int, eps: float = 1e-12):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.ones(hidden))
        self.bias = torch.nn.Parameter(torch.zeros(hidden))
        self.eps = eps

    def forward(self, a, b=None):
        return _AddLayerNorm.apply(a, b, self.weight, self.bias, self.eps)


class _Attention(torch.autograd.Function):
    """Attention core on packed QKV [B, S, 3, H, D] FP16 -> [B, S, H, D] FP16
    (the attention core stays floating point)."""

    @staticmethod
    def forward(ctx, qkv):
        qkv = qkv.contiguous()
        out, lse, _ = ops.attention_fwd(qkv)
        ctx.save_for_backward(qkv, out, lse)
        return out

    @staticmethod
    def backward(ctx, dout):
        qkv, out, lse = ctx.saved_tensors
        return ops.attention_bwd(qkv, out, dout.contiguous(), lse)


def attention(qkv: torch.Tensor) -> torch.Tensor:
    return _Attention.apply(qkv)


class _EmbedLN(torch.autograd.Function):
    """Embedding sum + LayerNorm of the encoder input in one kernel each way
    (word[tok] + pos[s] + typ[0] gathered, never materialised; the backward
    scatter-adds straight into the tables' gradients).  Returns (y, aux) where
    aux is the first planned op's operand hint (FP16 copy / absmax) or empty."""

    @staticmethod
    def forward(ctx, tokens, word, pos, typ, gamma, beta, eps, want_f16, want_absmax, want_quant=False):
        from .fused import _mark
        _mark("fwd", "embed")
        B, S = tokens.shape
        none = torch.empty(0, device=word.device)
        if want_quant:  # the first planned op is INT8: its operand comes out of the same kernel
            y, s, mean, rstd, q, sc, q16 = ops.embed_layernorm_fwd_quant(tokens, word, pos, typ, gamma, beta, eps)
            aux = (q, sc, q16)
        else:
            y, s, mean, rstd, y16, am = ops.embed_layernorm_fwd(tokens, word, pos, typ, gamma, beta, eps,
                                                                want_f16, want_absmax)
            aux = (y16 if want_f16 else (am if want_absmax else none), none, none)
        ctx.save_for_backward(tokens, s, mean, rstd)
        ctx.params = (word, pos, typ, gamma, beta)
        ctx.mark_non_differentiable(*aux)
        ctx.set_materialize_grads(False)
        return (y.view(B, S, -1),) + aux

    @staticmethod
    def backward(ctx, dy, _daux, _ds, _d16):
        from .fused import _mark
        _mark("bwd", "embed")
        tokens, s, mean, rstd = ctx.saved_tensors
        word, pos, typ, gamma, beta = ctx.params
        grads = []
        for p in (word, pos, typ, gamma, beta):
            mg = getattr(p, "main_grad", None)
            grads.append(mg if mg is not None else torch.zeros_like(p))
        dy = dy.reshape(-1, dy.shape[-1]).contiguous()
        ops.embed_layernorm_bwd(dy, s, mean, rstd, gamma.detach(), tokens, grads[3], grads[4], grads[0],
                                grads[1], grads[2])
        out = [None] * 10
        for i, p in enumerate((word, pos, typ, gamma, beta)):
            if getattr(p, "main_grad", None) is None:
                out[1 + i] = grads[i]
        return tuple(out)


def pack_aux(aux, s, q16):
    """The next planned op's operand hint carried between fused kernels: an
    FP16 copy or absmax tensor, or (INT8) the quantized operand itself as the
    tuple ("i8", q, s[1], FP16(q)); None when there is nothing to carry."""
    if s.numel():
        return ("i8", aux, s[:1], q16)
    return aux if aux.numel() else None


def embed_layernorm(tokens, word, pos, typ, ln, want_f16=False, want_absmax=False, want_quant=False):
    y, aux, s, q16 = _EmbedLN.apply(tokens, word.weight, pos.weight, typ.weight, ln.weight, ln.bias, ln.eps,
                                    want_f16, want_absmax, want_quant)
    return y, pack_aux(aux, s, q16)
