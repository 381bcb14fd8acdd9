"""Glue between planned operators, on this package's kernels: fused
residual-add + LayerNorm (the post-LN of every encoder sublayer)."""
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


class AddLayerNorm(torch.nn.Module):
    """y = LayerNorm(a + b) with FP32 statistics; b may be FP32 or FP16."""

    def __init__(self, hidden: int, eps: float = 1e-12):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.ones(hidden))
        self.bias = torch.nn.Parameter(torch.zeros(hidden))
        self.eps = eps

    def forward(self, a, b=None):
        return _AddLayerNorm.apply(a, b, self.weight, self.bias, self.eps)
