"""Quantized Linear: the per-operator kernel a QSync precision plan selects.

Forward (Y = X W^T + b), per the plan's ``Precision`` (precision.hpp:12):
  * INT8  -- per-tensor activation scale, per-channel weight scales
             (PAPER.md:426-427), tcgen05 kind::i8 GEMM with int32 accumulation
             and the dequant + bias epilogue fused; emits FP32
             (graph.hpp:38-40 ``output_precision``).
  * FP16  -- FP16 operands, FP32 accumulation, emits FP16.
  * FP32  -- FP32 GEMMs on the tensor cores through the 3xTF32 split
             (qsync_gemm_f32, FP32-level accuracy; training devices stay FP32,
             replayer.cpp:96-101).
Backward of INT8 and FP16 ops runs in FP16 (cost_mapper.cpp:13-15
``backward_precision``): the incoming gradient is cast once to FP16 (plus its
transpose and the bias-gradient column sums, one kernel), dgrad = dY16 W16 on
tcgen05, wgrad = dY16^T X^ (the saved quantized activation, scaled by s_x in the
epilogue) emitted in FP32 (cost_mapper.cpp:48-50).
"""
from __future__ import annotations

import torch

from . import ops

INT8, FP16, FP32 = "INT8", "FP16", "FP32"
# FP8 (E4M3) is the B200 extension of the ladder: a
# fixed-point-like rung between INT8 and FP16 -- per-tensor activation and
# per-channel weight scales, FP32 accumulation, FP32 output, FP16 backward.
# The reference planner's Precision enum (precision.hpp:12) does not know it,
# so plans from the reference never select it.
FP8 = "FP8"
# BF16: the float rung SPEC.md:324 leaves room for (indicator k = 7 instead of
# FP16's 9): BF16 operands, FP32 accumulation, emits BF16, BF16 backward (dgrad
# BF16, wgrad FP32).  Like FP8, the reference enum has no BF16; plans name it
# through this package (load_plan accepts it).
BF16 = "BF16"
PRECISIONS = (INT8, FP16, FP32)
EXTENDED = (INT8, FP8, BF16, FP16, FP32)  # the B200 ladder, coarsest first

# Profiling hook (profiler.StatsRecorder): when set, every QLinear records the
# device statistics of its input activation, weight and incoming gradient
# (qsync_tensor_stats -> OpStats fields, profile.hpp:95-108).
STATS_RECORDER = None


def _record(name, kind, t):
    if STATS_RECORDER is not None and name is not None:
        STATS_RECORDER.record(name, kind, ops.tensor_stats(t.contiguous()))


def output_dtype(precision: str) -> torch.dtype:
    """graph.hpp:38-40: fixed-point kernels emit FP32, float kernels their own format."""
    return {FP16: torch.float16, BF16: torch.bfloat16}.get(precision, torch.float32)


def backward_precision(precision: str) -> str:
    """cost_mapper.cpp:13-15 (FP8 backs off to FP16 like INT8; BF16 stays BF16)."""
    return FP16 if precision in (INT8, FP8) else precision


# Optional side stream for weight gradients (TrainStep enables it): wgrad only
# feeds the optimizer, so it runs concurrently with the rest of the backward
# chain (dgrad of the next layers); TrainStep joins it before the all-reduce.
WGRAD_STREAM: torch.cuda.Stream | None = None
# Data-parallel readiness hook (TrainStep, world > 1): called with a list of
# parameters whose gradients are final, so their all-reduce bucket can start.
GRAD_READY = None


def _main_grad(p):
    return getattr(p, "main_grad", None) if p is not None else None


def _fp16_backward(ctx, dy, x16, w16, alpha_dev, dt=torch.float16):
    """Shared FP16 backward (cost_mapper.cpp:13-15) on row-major operands.

    dgrad = dY16 W16 reads W16 [N_out, K_in] as an MN-major B operand and wgrad =
    dY16^T X16 reads dY16 [M, N_out] and X16 [M, K_in] as MN-major A and B, so no
    transposed copies are made.  When the parameters carry a ``main_grad`` (a
    slice of the flat FP32 gradient bucket), wgrad is ADDED into it by the GEMM
    epilogue's TMA reduce-add and the bias gradient by the cast kernel's column
    sums; autograd then receives None for them."""
    w, b = ctx.w_ref, ctx.b_ref
    dy = dy.contiguous()
    mw, mb = _main_grad(w), _main_grad(b)
    if dt == torch.float16:
        dy16, _, db = ops.cast_transpose(dy, True, False, b is not None and mb is None, colsum_into=mb)
    else:  # BF16 backward entry: one kernel for the cast and the bias-gradient column sums
        db = None
        if b is not None and mb is None:
            db = torch.zeros(dy.shape[-1], device=dy.device, dtype=torch.float32)
        dy16 = ops.act_bwd_colsum(dy, None, ops.ACT_NONE, dt, colsum_into=mb if mb is not None else db)
    dx = ops.gemm_f16(dy16, w16, out_dtype=ctx.x_dtype, b_mn=True)  # dgrad [M, K_in]
    if mw is not None and WGRAD_STREAM is not None:
        cur = torch.cuda.current_stream()
        WGRAD_STREAM.wait_stream(cur)
        with torch.cuda.stream(WGRAD_STREAM):
            ops.gemm_f16(dy16, x16, alpha_dev=alpha_dev, out=mw, accumulate=True, a_mn=True,
                         b_mn=True)
        for t in (dy16, x16, alpha_dev):
            if t is not None:
                t.record_stream(WGRAD_STREAM)
        dw = None
    elif mw is not None:
        ops.gemm_f16(dy16, x16, alpha_dev=alpha_dev, out=mw, accumulate=True, a_mn=True, b_mn=True)
        dw = None
    else:
        dw = ops.gemm_f16(dy16, x16, out_dtype=torch.float32, alpha_dev=alpha_dev, a_mn=True,
                          b_mn=True)
    if mb is not None:
        db = None
    return dx, dw, db


class _QLinearInt8(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, name=None):
        _record(name, "act", x)
        _record(name, "w", w)
        ctx.name = name
        # The INT8 op keeps only its 1-byte quantized activation for backward;
        # the FP16 views of it and of W are made there -- the "bp_cost" casts
        # of the paper's cost model, which buy the INT8 op its memory saving.
        xq, xs, _ = ops.quantize_per_tensor(x)
        wq, ws, _ = ops.quantize_per_channel(w)
        _, y = ops.gemm_s8(xq, wq, xs, ws, b)
        ctx.save_for_backward(xq, xs)
        ctx.x_dtype = x.dtype
        ctx.w_ref, ctx.b_ref = w, b
        return y

    @staticmethod
    def backward(ctx, dy):
        xq, xs = ctx.saved_tensors
        _record(ctx.name, "grad", dy)
        x16 = ops.cast(xq, torch.float16)              # exact: the int8 grid values
        w16 = ops.cast(ctx.w_ref.detach(), torch.float16)
        # wgrad = s_x * dY16^T X^ (activation scale applied in the GEMM epilogue)
        return _fp16_backward(ctx, dy, x16, w16, xs) + (None,)


class _QLinearFp8(torch.autograd.Function):
    """FP8 rung: E4M3 operands (per-tensor activation, per-channel weight scales),
    tcgen05 kind::f8f6f4 GEMM with the dequant epilogue -> FP32; FP16 backward
    reading the saved 1-byte activation (exact in FP16) times s_x."""

    @staticmethod
    def forward(ctx, x, w, b, name=None):
        _record(name, "act", x)
        _record(name, "w", w)
        ctx.name = name
        xq, xs = ops.quantize_fp8(x)
        wq, ws = ops.quantize_fp8_rows(w)
        y = ops.gemm_f8(xq, wq, xs, ws, b)
        ctx.save_for_backward(xq, xs)
        ctx.x_dtype = x.dtype
        ctx.w_ref, ctx.b_ref = w, b
        return y

    @staticmethod
    def backward(ctx, dy):
        xq, xs = ctx.saved_tensors
        _record(ctx.name, "grad", dy)
        x16 = ops.cast(xq, torch.float16)  # exact: E4M3 values are FP16 values
        w16 = ops.cast(ctx.w_ref.detach(), torch.float16)
        return _fp16_backward(ctx, dy, x16, w16, xs) + (None,)


class _QLinearFp16(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, name=None):
        _record(name, "act", x)
        _record(name, "w", w)
        ctx.name = name
        x16 = x if x.dtype == torch.float16 else ops.cast(x, torch.float16)
        w16 = ops.cast(w, torch.float16)
        y = ops.gemm_f16(x16, w16, out_dtype=torch.float16, bias=b)
        ctx.save_for_backward(x16, w16)
        ctx.x_dtype = x.dtype
        ctx.w_ref, ctx.b_ref = w, b
        return y

    @staticmethod
    def backward(ctx, dy):
        x16, w16 = ctx.saved_tensors
        _record(ctx.name, "grad", dy)
        return _fp16_backward(ctx, dy, x16, w16, None) + (None,)


class _QLinearBf16(torch.autograd.Function):
    """BF16 rung: BF16 operands on tcgen05 kind::f16 (BF16 format), FP32
    accumulation, emits BF16; BF16 backward (dgrad BF16 -> the input's format,
    wgrad FP32)."""

    @staticmethod
    def forward(ctx, x, w, b, name=None):
        _record(name, "act", x)
        _record(name, "w", w)
        ctx.name = name
        xb = x if x.dtype == torch.bfloat16 else ops.cast(x, torch.bfloat16)
        wb = ops.cast(w, torch.bfloat16)
        y = ops.gemm_f16(xb, wb, out_dtype=torch.bfloat16, bias=b)
        ctx.save_for_backward(xb, wb)
        ctx.x_dtype = x.dtype
        ctx.w_ref, ctx.b_ref = w, b
        return y

    @staticmethod
    def backward(ctx, dy):
        xb, wb = ctx.saved_tensors
        _record(ctx.name, "grad", dy)
        return _fp16_backward(ctx, dy, xb, wb, None, dt=torch.bfloat16) + (None,)


class _QLinearFp32(torch.autograd.Function):
    """FP32 (the training devices' plan, replayer.cpp:96-101): FP32 in, FP32 out,
    FP32 backward -- every GEMM on the tensor cores through the 3xTF32 split
    (qsync_gemm_f32, FP32-level accuracy); the bias gradient is one column-sum
    kernel."""

    @staticmethod
    def forward(ctx, x, w, b, name=None):
        _record(name, "act", x)
        _record(name, "w", w)
        ctx.name = name
        xf = x if x.dtype == torch.float32 else ops.cast(x, torch.float32)
        y = ops.gemm_f32(xf, w.detach(), bias=b.detach() if b is not None else None)
        ctx.save_for_backward(xf)
        ctx.x_dtype = x.dtype
        ctx.w_ref, ctx.b_ref = w, b
        return y

    @staticmethod
    def backward(ctx, dy):
        (xf,) = ctx.saved_tensors
        _record(ctx.name, "grad", dy)
        w, b = ctx.w_ref, ctx.b_ref
        dy = dy.contiguous().float()
        mw, mb = _main_grad(w), _main_grad(b)
        dx = ops.gemm_f32(dy, w.detach(), b_mn=True)  # dgrad [M, K_in]
        if dx.dtype != ctx.x_dtype:
            dx = ops.cast(dx, ctx.x_dtype)
        dw = db = None
        if mw is not None:
            ops.gemm_f32(dy, xf, out=mw, accumulate=True, a_mn=True, b_mn=True)
        else:
            dw = ops.gemm_f32(dy, xf, a_mn=True, b_mn=True)
        if b is not None:
            if mb is not None:
                ops.act_bwd_colsum(dy, None, ops.ACT_NONE, None, colsum_into=mb)
            else:
                db = torch.zeros(dy.shape[-1], device=dy.device, dtype=torch.float32)
                ops.act_bwd_colsum(dy, None, ops.ACT_NONE, None, colsum_into=db)
        return dx, dw, db, None


class _Cast(torch.autograd.Function):
    """Autograd-aware device cast (K4) for the glue between planned operators."""

    @staticmethod
    def forward(ctx, x, dtype):
        ctx.src = x.dtype
        return ops.cast(x.contiguous(), dtype)

    @staticmethod
    def backward(ctx, g):
        return ops.cast(g.contiguous(), ctx.src), None


def cast(x: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    return x if x.dtype == dtype else _Cast.apply(x, dtype)


def qlinear(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None, precision: str,
            name: str | None = None) -> torch.Tensor:
    """Y = X W^T + b for X [..., K] at the given plan precision."""
    shape = x.shape
    x2 = x.reshape(-1, shape[-1])
    if not x2.is_contiguous():
        x2 = x2.contiguous()
    if precision == INT8:
        y = _QLinearInt8.apply(x2, w, b, name)
    elif precision == FP16:
        y = _QLinearFp16.apply(x2, w, b, name)
    elif precision == FP8:
        y = _QLinearFp8.apply(x2, w, b, name)
    elif precision == BF16:
        y = _QLinearBf16.apply(x2, w, b, name)
    elif precision == FP32:
        y = _QLinearFp32.apply(x2, w, b, name)
    else:
        raise ValueError(f"validation: unknown precision \"{precision}\"")
    return y.reshape(*shape[:-1], w.shape[0])


class QLinear(torch.nn.Module):
    """nn.Linear whose kernel precision is set by the device's plan entry."""

    def __init__(self, in_features: int, out_features: int, name: str, bias: bool = True,
                 precision: str = FP32):
        super().__init__()
        self.name = name
        self.in_features = in_features
        self.out_features = out_features
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features))
        self.bias = torch.nn.Parameter(torch.zeros(out_features)) if bias else None
        self.precision = precision
        bound = 1.0 / in_features ** 0.5
        torch.nn.init.uniform_(self.weight, -bound, bound)

    def forward(self, x):
        return qlinear(x, self.weight, self.bias, self.precision, self.name)

    def extra_repr(self):
        return f"{self.name}: {self.in_features}->{self.out_features} {self.precision}"
