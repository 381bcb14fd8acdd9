"""Quantized Conv2d (NHWC) -- the convolution kernel a QSync plan selects.

Forward is a GEMM over the column matrix A [N*P*Q, R*S*C] and the KRSC weight
W [Cout, R*S*C] (below-16-bit convolutions are channels-last).  When
each (r,s) tap's channel run is a whole number of 128-byte K-slices or half of one
(C % 64 INT8, C % 32 FP16: every ResNet-50 conv but conv1) A is never materialised:
the GEMM's producer warp gathers it tile by tile from the NHWC input (implicit GEMM,
`qsync_conv_fwd_implicit`); a 1x1/stride-1 conv reads the NHWC tensor itself as A;
otherwise im2col builds it.
  * INT8 -- x quantized once per tensor (1 B/elem NHWC), im2col of the int8
            tensor, per-channel weight scales, tcgen05 kind::i8 GEMM with the fused
            dequant + bias epilogue -> FP32 NHWC output (graph.hpp:38-40).
  * FP16 -- FP16 im2col, tcgen05 kind::f16 GEMM -> FP16 NHWC output.
  * FP32 -- im2col (in place for 1x1/s1) + the tcgen05 3xTF32 GEMM (training
            devices stay FP32, replayer.cpp:96-101).
Backward of INT8/FP16 runs in FP16 (cost_mapper.cpp:13-15): dgrad = the implicit
GEMM over dY taps (`qsync_conv_dgrad_implicit`, Cout % 64 == 0) or col2im(dY16 W16),
FP32 out; wgrad = dY16^T A16 (times s_x for INT8) in FP32 (cost_mapper.cpp:48-50),
A16 gathered from the FP16 input by the GEMM (`qsync_conv_wgrad_implicit`, C % 64
== 0) or rebuilt by im2col.  The INT8 op keeps only its int8 input for backward
and widens it there (the paper's backward casting cost).
"""
from __future__ import annotations

import torch

from . import ops
from .qlinear import FP16, FP32, INT8


def _pad_k(w2: torch.Tensor, kp: int) -> torch.Tensor:
    if w2.shape[1] == kp:
        return w2.contiguous()
    out = torch.zeros((w2.shape[0], kp), device=w2.device, dtype=w2.dtype)
    out[:, : w2.shape[1]] = w2
    return out


def _pointwise(R, S, stride, pad, kp, C) -> bool:
    """1x1, stride 1, no padding, no K padding: the NHWC input is the column matrix."""
    return R == 1 and S == 1 and tuple(stride) == (1, 1) and tuple(pad) == (0, 0) and kp == C


class _QConv(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, geom, precision):
        R, S, stride, pad = geom
        N, H, W, C = x.shape
        cout = w.shape[0]
        K = R * S * C
        align = 16 if precision == INT8 else 8
        kp = (K + align - 1) // align * align
        w2 = _pad_k(w.reshape(cout, K), kp)
        if precision == INT8:
            xq, xs, _ = ops.quantize_per_tensor(x.reshape(1, -1))
            xq = xq.view(N, H, W, C)
            wq, ws, _ = ops.quantize_per_channel(w2)
            # Order measured on the ResNet-50 shapes: the TMA-im2col implicit GEMM
            # (whole 128-byte runs) beats a plain GEMM over the NHWC tensor for 1x1
            # convs at M = 200k; the plain GEMM beats the cp.async gather (64-byte runs).
            if C % 128 and _pointwise(R, S, stride, pad, kp, C):
                # 1x1 / stride 1: the NHWC int8 tensor IS the column matrix
                _, y = ops.gemm_s8(xq.view(N * H * W, C), wq, xs, ws, b)
                P, Q = H, W
            elif ops.implicit_conv_ok(C, torch.int8):
                # implicit GEMM: the producer warp gathers the column tiles from xq
                y, (P, Q) = ops.conv_fwd_implicit(xq, wq, R, S, stride, pad, xs, ws, b)
            else:
                A, (P, Q) = ops.im2col(xq, R, S, stride, pad, ld=kp)
                _, y = ops.gemm_s8(A, wq, xs, ws, b)
            ctx.save_for_backward(xq, xs)
        else:
            x16 = x if x.dtype == torch.float16 else ops.cast(x.contiguous(), torch.float16)
            w16 = ops.cast(w2, torch.float16)
            if C % 64 and _pointwise(R, S, stride, pad, kp, C):
                y = ops.gemm_f16(x16.reshape(N * H * W, C), w16, out_dtype=torch.float16, bias=b)
                P, Q = H, W
            elif ops.implicit_conv_ok(C, torch.float16):
                y, (P, Q) = ops.conv_fwd_implicit(x16, w16, R, S, stride, pad, bias=b,
                                                  out_dtype=torch.float16)
            else:
                A, (P, Q) = ops.im2col(x16, R, S, stride, pad, ld=kp)
                y = ops.gemm_f16(A, w16, out_dtype=torch.float16, bias=b)
            ctx.save_for_backward(x16, torch.ones(1, device=x.device))
        ctx.geom, ctx.precision, ctx.kp = geom, precision, kp
        ctx.shapes = (N, H, W, C, cout, P, Q, K)
        ctx.w_ref, ctx.has_bias, ctx.x_dtype = w, b is not None, x.dtype
        return y.view(N, P, Q, cout)

    @staticmethod
    def backward(ctx, dy):
        xs_saved, alpha = ctx.saved_tensors
        R, S, stride, pad = ctx.geom
        N, H, W, C, cout, P, Q, K = ctx.shapes
        kp = ctx.kp
        dy2 = dy.reshape(N * P * Q, cout).contiguous()
        dy16, _, db = ops.cast_transpose(dy2, True, False, ctx.has_bias)
        w_fp = ctx.w_ref.detach()
        dx = None
        if ctx.needs_input_grad[0]:
            if ops.implicit_dgrad_ok(C, cout, stride):
                # implicit dgrad: dY taps gathered by the GEMM producer, weights
                # read in place as [Cout][R*S][C] -- no column gradient, no col2im
                w16 = ops.cast(w_fp.contiguous(), torch.float16)
                dx = ops.conv_dgrad_implicit(dy16.view(N, P, Q, cout), w16, (N, H, W, C), stride, pad)
            else:
                # dgrad columns = dY16 W16 (W16 [Cout, kp] read as an MN-major B operand)
                w16 = ops.cast(_pad_k(w_fp.reshape(cout, K), kp), torch.float16)
                dcol = ops.gemm_f16(dy16, w16, out_dtype=torch.float32, b_mn=True)
                dx = ops.col2im(dcol, (N, H, W, C), R, S, stride, pad)
        alpha_dev = alpha if ctx.precision == INT8 else None
        # K of the wgrad GEMM is the pixel count (up to N*P*Q = 802,816 for conv1)
        # while M x N is tiny: accumulate into a zeroed FP32 buffer so the kernel
        # splits K across the SMs (partials reduce-added by TMA).
        dw2 = torch.zeros((cout, kp), device=dy.device, dtype=torch.float32)
        if ops.implicit_wgrad_ok(C) and kp == K:
            # implicit wgrad = dY16^T A16 with A16 gathered from the FP16 input
            # (the INT8 op's saved int8 input widened once: N*H*W*C, not R*S x that)
            x16 = xs_saved if xs_saved.dtype == torch.float16 else ops.cast(xs_saved, torch.float16)
            ops.conv_wgrad_implicit(x16, dy16, R, S, stride, pad, out=dw2, accumulate=True,
                                    alpha_dev=alpha_dev)
        else:
            # wgrad = dY16^T A16 (both read MN-major): rebuild the FP16 column matrix
            # from the saved (int8 / fp16) input.
            # from the saved input, widened to FP16 first (N*H*W*C elements, not
            # the R*S times larger column matrix).
            x16 = xs_saved if xs_saved.dtype == torch.float16 else ops.cast(xs_saved, torch.float16)
            A16, _ = ops.im2col(x16, R, S, stride, pad, ld=kp)
            ops.gemm_f16(dy16, A16, out=dw2, accumulate=True, a_mn=True, b_mn=True, alpha_dev=alpha_dev)
        dw = dw2[:, :K].reshape(ctx.w_ref.shape)
        if dx is not None and ctx.x_dtype != torch.float32:
            dx = dx.to(ctx.x_dtype)
        return dx, dw, db, None, None


def _cols32(x, R, S, stride, pad, kp):
    """FP32 column matrix [N*P*Q, kp]: a 1x1/stride-1 conv reads x in place; otherwise
    the byte-exact im2col runs over x viewed as FP16 pairs (each tap's channel run is
    contiguous, so C FP32 channels are 2C 16-bit lanes; zero padding is 0.0f)."""
    N, H, W, C = x.shape
    if _pointwise(R, S, stride, pad, kp, C):
        return x.reshape(N * H * W, C), (H, W)
    A, pq = ops.im2col(x.view(torch.float16), R, S, stride, pad, ld=2 * kp)
    return A.view(torch.float32), pq


class _QConv32(torch.autograd.Function):
    """FP32 Conv2d (training devices stay FP32, replayer.cpp:96-101) on the library's
    tcgen05 3xTF32 GEMM (qsync_gemm_f32, FP32-level accuracy): y = cols(x) W^T,
    dgrad = col2im(dY W) (1x1/s1: dY W itself), wgrad = dY^T cols(x)."""

    @staticmethod
    def forward(ctx, x, w, b, geom):
        R, S, stride, pad = geom
        N, H, W, C = x.shape
        cout = w.shape[0]
        K = R * S * C
        kp = (K + 3) // 4 * 4
        w2 = _pad_k(w.reshape(cout, K), kp)
        A, (P, Q) = _cols32(x, R, S, stride, pad, kp)
        y = ops.gemm_f32(A, w2, bias=b)
        ctx.save_for_backward(x, w2)
        ctx.geom, ctx.kp, ctx.has_bias, ctx.shapes = geom, kp, b is not None, (N, H, W, C, cout, P, Q, K)
        return y.view(N, P, Q, cout)

    @staticmethod
    def backward(ctx, dy):
        x, w2 = ctx.saved_tensors
        R, S, stride, pad = ctx.geom
        N, H, W, C, cout, P, Q, K = ctx.shapes
        dy2 = dy.reshape(N * P * Q, cout).float().contiguous()
        dx = dw = db = None
        if ctx.needs_input_grad[0]:
            dcol = ops.gemm_f32(dy2, w2, b_mn=True)  # [NPQ, kp]
            if _pointwise(R, S, stride, pad, ctx.kp, C):
                dx = dcol.view(N, H, W, C)
            else:
                dx = ops.col2im(dcol, (N, H, W, C), R, S, stride, pad)
        if ctx.needs_input_grad[1]:
            A, _ = _cols32(x, R, S, stride, pad, ctx.kp)
            # K of this GEMM is the pixel count (802,816 for conv1 at batch 64) while
            # M x N is tiny: accumulating into a zeroed buffer lets it split K over the SMs
            dw2 = torch.zeros((cout, ctx.kp), device=dy.device, dtype=torch.float32)
            ops.gemm_f32(dy2, A, out=dw2, accumulate=True, a_mn=True, b_mn=True)
            dw = dw2[:, :K].reshape(cout, R, S, C)
        if ctx.has_bias and ctx.needs_input_grad[2]:
            db = dy2.sum(0)
        return dx, dw, db, None


def qconv2d(x, w, b, stride=(1, 1), pad=(0, 0), precision=FP32):
    """x NHWC [N,H,W,C], w KRSC [Cout,R,S,C] -> y NHWC [N,P,Q,Cout]."""
    cout, R, S, C = w.shape
    if precision == FP32:
        return _QConv32.apply(x.float().contiguous(), w, b, (R, S, tuple(stride), tuple(pad)))
    if precision not in (INT8, FP16):
        raise ValueError(f"validation: unknown precision \"{precision}\"")
    return _QConv.apply(x.contiguous(), w, b, (R, S, tuple(stride), tuple(pad)), precision)


class QConv2d(torch.nn.Module):
    """NHWC Conv2d whose kernel precision is set by the device's plan entry."""

    def __init__(self, cin, cout, kernel, name, stride=1, pad=0, bias=True, precision=FP32):
        super().__init__()
        k = (kernel, kernel) if isinstance(kernel, int) else kernel
        self.name = name
        self.stride = (stride, stride) if isinstance(stride, int) else stride
        self.pad = (pad, pad) if isinstance(pad, int) else pad
        self.weight = torch.nn.Parameter(torch.empty(cout, k[0], k[1], cin))
        self.bias = torch.nn.Parameter(torch.zeros(cout)) if bias else None
        self.precision = precision
        torch.nn.init.kaiming_uniform_(self.weight.view(cout, -1), a=5 ** 0.5)

    def forward(self, x):
        return qconv2d(x, self.weight, self.bias, self.stride, self.pad, self.precision)
