"""Tensor-level front end of the C ABI (torch tensors are plumbing: device memory
and the current CUDA stream).  Every function launches this package's sm_100a
kernels through ``libqsync_b200.so``; nothing here computes on the CPU.

Numerics: symmetric INT8 grid, s = absmax/127 (IEEE FP32),
q = sat(rint(x/s)) in [-127, 127]; INT8 GEMMs accumulate in int32 and emit FP32
(graph.hpp:38-40); the FP16 backward emits dgrad in FP16 and wgrad in FP32
(cost_mapper.cpp:13-15, :48-50).
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import BF16, F16, F32, QsyncError, call

_DT = {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}
_DT_CAST = {**_DT, torch.int8: _lib.I8, torch.float8_e4m3fn: _lib.F8}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _req(t: torch.Tensor, name: str, dtypes=None) -> None:
    if not t.is_cuda:
        raise QsyncError(2, f"validation: {name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise QsyncError(2, f"validation: {name} must be contiguous")
    if dtypes is not None and t.dtype not in dtypes:
        raise QsyncError(4, f"domain: {name} has unsupported dtype {t.dtype}")


# --------------------------------------------------------------------------- K1
def absmax(x: torch.Tensor) -> torch.Tensor:
    _req(x, "x", _DT)
    out = torch.empty(1, device=x.device, dtype=torch.float32)
    call("qsync_absmax", _ptr(x), _DT[x.dtype], x.numel(), _ptr(out), _stream())
    return out


def absmax_rows(x: torch.Tensor) -> torch.Tensor:
    _req(x, "x", _DT)
    rows = x.shape[0]
    out = torch.empty(rows, device=x.device, dtype=torch.float32)
    call("qsync_absmax_rows", _ptr(x), _DT[x.dtype], rows, x.numel() // max(rows, 1), _ptr(out),
         _stream())
    return out


# --------------------------------------------------------------------------- K2
def pad8(n: int) -> int:
    """Row pitch of a transposed FP16 operand: the GEMM K it becomes must be a
    multiple of 8 (16-byte TMA pitch); pad columns are zero."""
    return (n + 7) // 8 * 8


def _transposed(cols: int, rows: int, device, dtype=torch.float16) -> torch.Tensor:
    ld = pad8(rows)
    if ld == rows:
        return torch.empty((cols, ld), device=device, dtype=dtype)
    return torch.zeros((cols, ld), device=device, dtype=dtype)


def quantize_per_tensor(x: torch.Tensor, transposed_f16: bool = False, out=None,
                        transposed_i8: bool = False):
    """Per-tensor RNE INT8 quantization of a 2-D (or flattened) tensor.

    Returns (q int8 same shape, scale float32[2] = {s, absmax}, q_t [cols, pad8(rows)] or None):
    q_t is FP16 with ``transposed_f16``, INT8 with ``transposed_i8``.
    """
    _req(x, "x", _DT)
    rows = x.shape[0] if x.dim() >= 2 else 1
    cols = x.numel() // max(rows, 1)
    q = out if out is not None else torch.empty(x.shape, device=x.device, dtype=torch.int8)
    scale = torch.empty(2, device=x.device, dtype=torch.float32)
    qt = None
    if transposed_i8:
        qt = _transposed(cols, rows, x.device, torch.int8)
    elif transposed_f16:
        qt = _transposed(cols, rows, x.device)
    call("qsync_quantize_per_tensor", _ptr(x), _DT[x.dtype], rows, cols, _ptr(q), _ptr(scale),
         _ptr(qt), _lib.I8 if transposed_i8 else F16, qt.shape[1] if qt is not None else 0,
         _stream())
    return q, scale, qt


def quantize_with_scale(x: torch.Tensor, scale: torch.Tensor) -> torch.Tensor:
    _req(x, "x", _DT)
    q = torch.empty(x.shape, device=x.device, dtype=torch.int8)
    call("qsync_quantize_with_scale", _ptr(x), _DT[x.dtype], x.numel(), _ptr(scale), _ptr(q),
         _stream())
    return q


def quantize_per_channel(w: torch.Tensor, transposed_f16: bool = False):
    """Per-output-channel (row) INT8 quantization of W [N, K]; optional FP16 W^T."""
    _req(w, "w", (torch.float32,))
    rows, cols = w.shape
    q = torch.empty_like(w, dtype=torch.int8)
    scales = torch.empty(rows, device=w.device, dtype=torch.float32)
    wt = torch.empty((cols, rows), device=w.device, dtype=torch.float16) if transposed_f16 else None
    call("qsync_quantize_per_channel", _ptr(w), rows, cols, _ptr(q), _ptr(scales), _ptr(wt),
         _stream())
    return q, scales, wt


# --------------------------------------------------------------------------- K9
def stochastic_round(x: torch.Tensor, q: float, zp: float, seed: int):
    """Device qsync::stochastic_round (indicator.cpp:176-193): returns (rounded int64, deq f64)."""
    _req(x, "x", (torch.float64,))
    r = torch.empty(x.shape, device=x.device, dtype=torch.int64)
    d = torch.empty(x.shape, device=x.device, dtype=torch.float64)
    call("qsync_stochastic_round_f64", _ptr(x), x.numel(), float(q), float(zp), int(seed), _ptr(r),
         _ptr(d), _stream())
    return r, d


def stochastic_round_float(x: torch.Tensor, e: int, k: int, seed: int) -> torch.Tensor:
    _req(x, "x", (torch.float64,))
    d = torch.empty(x.shape, device=x.device, dtype=torch.float64)
    call("qsync_stochastic_round_float_f64", _ptr(x), x.numel(), int(e), int(k), int(seed),
         _ptr(d), _stream())
    return d


def quantize_sr(x: torch.Tensor, scale: torch.Tensor, seed: int) -> torch.Tensor:
    _req(x, "x", (torch.float32,))
    q = torch.empty(x.shape, device=x.device, dtype=torch.int8)
    call("qsync_quantize_sr", _ptr(x), x.numel(), _ptr(scale), int(seed), _ptr(q), _stream())
    return q


def mt64_draws(seed: int, n: int, offset: int = 0, device="cuda") -> torch.Tensor:
    out = torch.empty(n, device=device, dtype=torch.int64)  # uint64 bits
    call("qsync_mt64_draws", int(seed), int(offset), int(n), _ptr(out), _stream())
    return out


# --------------------------------------------------------------------------- K3
def dequantize_per_tensor(q: torch.Tensor, scale: torch.Tensor) -> torch.Tensor:
    _req(q, "q", (torch.int8,))
    out = torch.empty(q.shape, device=q.device, dtype=torch.float32)
    call("qsync_dequantize_per_tensor", _ptr(q), q.numel(), _ptr(scale), _ptr(out), _stream())
    return out


def dequantize_per_channel(q: torch.Tensor, scales: torch.Tensor) -> torch.Tensor:
    _req(q, "q", (torch.int8,))
    out = torch.empty(q.shape, device=q.device, dtype=torch.float32)
    call("qsync_dequantize_per_channel", _ptr(q), q.shape[0], q.shape[1], _ptr(scales), _ptr(out),
         _stream())
    return out


# --------------------------------------------------------------------------- K4
def cast(x: torch.Tensor, dtype: torch.dtype, out=None) -> torch.Tensor:
    _req(x, "x", _DT_CAST)
    o = out if out is not None else torch.empty(x.shape, device=x.device, dtype=dtype)
    call("qsync_cast", _ptr(x), _DT_CAST[x.dtype], _ptr(o), _DT[dtype], x.numel(), _stream())
    return o


def cast_transpose(x: torch.Tensor, want_out: bool = True, want_t: bool = True,
                   want_colsum: bool = False, colsum_into: torch.Tensor | None = None):
    """[rows, cols] -> (FP16 copy, FP16 transpose [cols, pad8(rows)], FP32 column sums).

    With ``colsum_into`` the column sums are ADDED into that FP32 buffer (the
    bias gradient accumulated straight into its main_grad slot)."""
    _req(x, "x", (torch.float32, torch.float16))
    rows = x.shape[0]
    cols = x.numel() // max(rows, 1)
    o = torch.empty((rows, cols), device=x.device, dtype=torch.float16) if want_out else None
    t = _transposed(cols, rows, x.device) if want_t else None
    if colsum_into is not None:
        s, acc = colsum_into, 1
    else:
        s = torch.empty(cols, device=x.device, dtype=torch.float32) if want_colsum else None
        acc = 0
    call("qsync_cast_transpose", _ptr(x), _DT[x.dtype], rows, cols, _ptr(o), _ptr(t),
         t.shape[1] if t is not None else 0, _ptr(s), acc, _stream())
    return o, t, s


# --------------------------------------------------------------------------- K5
_ws = {}


def _stats_ws(device) -> torch.Tensor:
    key = (device.type, device.index)
    if key not in _ws:
        n = int(_lib.lib().qsync_stats_workspace_bytes())
        _ws[key] = torch.empty(n, device=device, dtype=torch.uint8)
    return _ws[key]


def tensor_stats(x: torch.Tensor, out=None) -> torch.Tensor:
    """float64[5] = {||x||^2, absmax, q, e, numel} (OpStats fields, profile.hpp:95-108)."""
    _req(x, "x", _DT)
    o = out if out is not None else torch.empty(5, device=x.device, dtype=torch.float64)
    call("qsync_tensor_stats", _ptr(x), _DT[x.dtype], x.numel(), _ptr(o), _ptr(_stats_ws(x.device)),
         _stream())
    return o


# --------------------------------------------------------------------------- K6/K7
# Optional per-launch timing (bench.py): a list that receives
# (kind, flops, start_event, end_event) for every GEMM launched while it is set.
GEMM_TIMER: list | None = None


def _timed(kind: str, flops: float):
    if GEMM_TIMER is None:
        return None
    # inside a CUDA-graph capture the events become event-record nodes of the graph
    ext = torch.cuda.is_current_stream_capturing()
    s = torch.cuda.Event(enable_timing=True, external=ext)
    e = torch.cuda.Event(enable_timing=True, external=ext)
    s.record()
    GEMM_TIMER.append((kind, flops, s, e))
    return e


def gemm_s8(a: torch.Tensor, b: torch.Tensor, scale_a=None, scale_b=None, bias=None,
            out_i32: bool = False, out_f32: bool = True, b_per_channel: bool = True,
            out=None):
    """C = A B^T on tcgen05 kind::i8.  Returns (c_i32 or None, c_f32 or None)."""
    _req(a, "a", (torch.int8,))
    _req(b, "b", (torch.int8,))
    M, K = a.shape
    N = b.shape[0]
    ci = torch.empty((M, N), device=a.device, dtype=torch.int32) if out_i32 else None
    cf = None
    if out_f32:
        cf = out if out is not None else torch.empty((M, N), device=a.device, dtype=torch.float32)
    ev = _timed("gemm_s8", 2.0 * M * N * K)
    call("qsync_gemm_s8", _ptr(a), _ptr(b), M, N, K, _ptr(ci), _ptr(cf), _ptr(scale_a),
         _ptr(scale_b), int(b_per_channel), _ptr(bias), _stream())
    if ev is not None:
        ev.record()
    return ci, cf


def gemm_f16(a: torch.Tensor, b: torch.Tensor, out_dtype=torch.float32, alpha: float = 1.0,
             alpha_dev=None, bias=None, out=None, accumulate: bool = False,
             a_mn: bool = False, b_mn: bool = False) -> torch.Tensor:
    """C = alpha * A B^T on tcgen05 kind::f16 (FP32 accumulators).

    A is [M, K] (or [K, M] with ``a_mn``); B is [N, K] (or [K, N] with ``b_mn``)."""
    _req(a, "a", (torch.float16, torch.bfloat16))
    _req(b, "b", (a.dtype,))
    if a_mn and not b_mn:
        raise QsyncError(4, "domain: MN-major A requires MN-major B")
    K, M = a.shape if a_mn else (a.shape[1], a.shape[0])
    N = b.shape[1] if b_mn else b.shape[0]
    c = out if out is not None else torch.empty((M, N), device=a.device, dtype=out_dtype)
    ev = _timed("gemm_f16", 2.0 * M * N * K)
    call("qsync_gemm_f16", _ptr(a), _ptr(b), _DT[a.dtype], M, N, K, _ptr(c), _DT[c.dtype],
         float(alpha), _ptr(alpha_dev), _ptr(bias), int(accumulate),
         (1 if a_mn else 0) | (2 if b_mn else 0), _stream())
    if ev is not None:
        ev.record()
    return c


_f32_ws: dict = {}
_f32_ws_retired: list = []


def gemm_f32(a: torch.Tensor, b: torch.Tensor, alpha: float = 1.0, alpha_dev=None, bias=None, out=None,
             accumulate: bool = False, a_mn: bool = False, b_mn: bool = False) -> torch.Tensor:
    """C = alpha * A B^T in FP32 on the tensor cores (3xTF32 split, FP32-level
    accuracy; qsync_gemm_f32).  Layouts as gemm_f16; FP32 output."""
    _req(a, "a", (torch.float32,))
    _req(b, "b", (torch.float32,))
    if a_mn and not b_mn:
        raise QsyncError(4, "domain: MN-major A requires MN-major B")
    K, M = a.shape if a_mn else (a.shape[1], a.shape[0])
    N = b.shape[1] if b_mn else b.shape[0]
    c = out if out is not None else torch.empty((M, N), device=a.device, dtype=torch.float32)
    nbytes = int(_lib.lib().qsync_gemm_f32_workspace_bytes(M, N, K))
    key = (a.device, torch.cuda.current_stream().cuda_stream)
    ws = _f32_ws.get(key)
    if ws is None or ws.numel() < nbytes:
        if ws is not None:  # kernels already enqueued (or captured) may still read it
            _f32_ws_retired.append(ws)
        ws = torch.empty(nbytes, device=a.device, dtype=torch.uint8)
        _f32_ws[key] = ws
    ev = _timed("gemm_f32", 2.0 * M * N * K)
    call("qsync_gemm_f32", _ptr(a), _ptr(b), M, N, K, _ptr(c), float(alpha), _ptr(alpha_dev), _ptr(bias),
         int(accumulate), (1 if a_mn else 0) | (2 if b_mn else 0), _ptr(ws), _stream())
    if ev is not None:
        ev.record()
    return c


# --------------------------------------------------------------------------- K8 conv
def conv_out_size(H, W, R, S, stride, pad, dil=(1, 1)):
    import ctypes as C
    P, Q = C.c_int64(0), C.c_int64(0)
    call("qsync_conv_out_size", H, W, R, S, stride[0], stride[1], pad[0], pad[1], dil[0], dil[1],
         C.byref(P), C.byref(Q))
    return P.value, Q.value


def im2col(x: torch.Tensor, R: int, S: int, stride, pad, dil=(1, 1), ld: int | None = None):
    """NHWC x (int8 / fp16) -> column matrix [N*P*Q, ld] (K = R*S*C, zero padded)."""
    _req(x, "x", (torch.int8, torch.float16, torch.bfloat16))
    N, H, W, Cc = x.shape
    P, Q = conv_out_size(H, W, R, S, stride, pad, dil)
    K = R * S * Cc
    align = 16 if x.dtype == torch.int8 else 8
    ld = ld or (K + align - 1) // align * align
    out = torch.empty((N * P * Q, ld), device=x.device, dtype=x.dtype)
    call("qsync_im2col", _ptr(x), _DT_CAST[x.dtype], N, H, W, Cc, R, S, stride[0], stride[1],
         pad[0], pad[1], dil[0], dil[1], _ptr(out), ld, _stream())
    return out, (P, Q)


def implicit_conv_ok(C: int, dtype: torch.dtype) -> bool:
    """Whether the implicit-GEMM forward applies: each (r,s) tap's channel run must
    be a whole number of 128-byte K-slices, or exactly half of one (64 bytes: two
    taps per slice, gathered by the cp.async lanes)."""
    return (C * (1 if dtype == torch.int8 else 2)) % 64 == 0


def conv_fwd_implicit(x: torch.Tensor, w2: torch.Tensor, R: int, S: int, stride, pad, scale_a=None,
                      scale_b=None, bias=None, out_dtype=torch.float32, b_per_channel: bool = True):
    """Implicit-GEMM Conv2d forward: x NHWC (int8 / fp16), w2 [Cout, R*S*C] (KRSC
    flattened) -> y [N*P*Q, Cout].  The column matrix is gathered tile by tile by
    the GEMM's producer warp, never materialised."""
    _req(x, "x", (torch.int8, torch.float16, torch.bfloat16))
    _req(w2, "w2", (x.dtype,))
    N, H, W, C = x.shape
    P, Q = conv_out_size(H, W, R, S, stride, pad)
    cout = w2.shape[0]
    y = torch.empty((N * P * Q, cout), device=x.device, dtype=out_dtype)
    ev = _timed("gemm_s8" if x.dtype == torch.int8 else "gemm_f16", 2.0 * N * P * Q * cout * R * S * C)
    call("qsync_conv_fwd_implicit", _ptr(x), _DT_CAST[x.dtype], N, H, W, C, R, S, stride[0], stride[1],
         pad[0], pad[1], _ptr(w2), cout, _ptr(y), _DT[out_dtype], _ptr(scale_a), _ptr(scale_b),
         int(b_per_channel), _ptr(bias), _stream())
    if ev is not None:
        ev.record()
    return y, (P, Q)


def implicit_dgrad_ok(C: int, cout: int, stride=(1, 1)) -> bool:
    """Whether qconv takes the implicit-GEMM dgrad: dY channel runs of 128 B,
    16-byte weight rows, and stride 1 -- a strided conv's dgrad is a fractionally
    strided gather (the cp.async lanes zero 3 of 4 taps at stride 2, measured
    slower than dY W + col2im), so it keeps the column path."""
    return cout % 64 == 0 and C % 8 == 0 and tuple(stride) == (1, 1)


def conv_set_impl(tma: bool) -> None:
    """Implicit-conv operand loads: TMA im2col mode (default) or the cp.async
    gather lanes (A/B and the strided dgrad, which TMA im2col cannot express)."""
    call("qsync_conv_set_impl", int(bool(tma)))


def implicit_wgrad_ok(C: int) -> bool:
    """Whether the implicit-GEMM wgrad applies (FP16 channel runs of 128 B)."""
    return C % 64 == 0


def conv_dgrad_implicit(dy: torch.Tensor, w: torch.Tensor, xshape, stride, pad,
                        out_dtype=torch.float32) -> torch.Tensor:
    """Implicit-GEMM Conv2d dgrad: dy NHWC [N,P,Q,Cout] FP16, w [Cout,R,S,C] FP16 ->
    dx NHWC [N,H,W,C] out_dtype.  dY taps are gathered by the GEMM's producer warp
    (no column-gradient matrix, no col2im)."""
    _req(dy, "dy", (torch.float16, torch.bfloat16))
    _req(w, "w", (dy.dtype,))
    N, H, W, C = xshape
    cout, R, S, _ = w.shape
    dx = torch.empty((N, H, W, C), device=dy.device, dtype=out_dtype)
    ev = _timed("gemm_f16", 2.0 * N * H * W * C * R * S * cout)
    call("qsync_conv_dgrad_implicit", _ptr(dy), _DT_CAST[dy.dtype], N, H, W, C, R, S, stride[0], stride[1],
         pad[0], pad[1], _ptr(w), cout, _ptr(dx), _DT[out_dtype], _stream())
    if ev is not None:
        ev.record()
    return dx


def conv_wgrad_implicit(x: torch.Tensor, dy: torch.Tensor, R: int, S: int, stride, pad, out=None,
                        accumulate: bool = False, alpha: float = 1.0, alpha_dev=None) -> torch.Tensor:
    """Implicit-GEMM Conv2d wgrad: x NHWC FP16 [N,H,W,C], dy [N*P*Q, Cout] FP16 ->
    dw FP32 [Cout, R*S*C] (+)= alpha * dY^T A, the column matrix A gathered from x
    by the GEMM's producer warp."""
    _req(x, "x", (torch.float16, torch.bfloat16))
    _req(dy, "dy", (x.dtype,))
    N, H, W, C = x.shape
    cout = dy.shape[-1]
    P, Q = conv_out_size(H, W, R, S, stride, pad)
    if out is None:
        out = (torch.zeros if accumulate else torch.empty)((cout, R * S * C), device=x.device,
                                                           dtype=torch.float32)
    ev = _timed("gemm_f16", 2.0 * N * P * Q * cout * R * S * C)
    call("qsync_conv_wgrad_implicit", _ptr(x), _DT_CAST[x.dtype], N, H, W, C, R, S, stride[0], stride[1],
         pad[0], pad[1], _ptr(dy), cout, _ptr(out), float(alpha), _ptr(alpha_dev), int(accumulate), _stream())
    if ev is not None:
        ev.record()
    return out


def col2im(dcol: torch.Tensor, xshape, R: int, S: int, stride, pad, dil=(1, 1)) -> torch.Tensor:
    """Adjoint of im2col: dx NHWC FP32 from the column gradient (FP32 or FP16)."""
    _req(dcol, "dcol", (torch.float32, torch.float16))
    N, H, W, Cc = xshape
    dx = torch.empty((N, H, W, Cc), device=dcol.device, dtype=torch.float32)
    call("qsync_col2im", _ptr(dcol), _DT[dcol.dtype], N, H, W, Cc, R, S, stride[0], stride[1],
         pad[0], pad[1], dil[0], dil[1], dcol.shape[1], _ptr(dx), _stream())
    return dx


# --------------------------------------------------------------------------- glue
def layernorm_fwd(a: torch.Tensor, b: torch.Tensor | None, gamma, beta, eps: float):
    """s = a + b, y = LN(s).  Returns (y, s, mean, rstd)."""
    _req(a, "a", (torch.float32,))
    cols = a.shape[-1]
    rows = a.numel() // cols
    y = torch.empty_like(a)
    s = torch.empty_like(a) if b is not None else None
    mean = torch.empty(rows, device=a.device, dtype=torch.float32)
    rstd = torch.empty(rows, device=a.device, dtype=torch.float32)
    bd = _DT[b.dtype] if b is not None else F32
    if b is not None:
        _req(b, "b", (torch.float32, torch.float16))
    call("qsync_layernorm_fwd", _ptr(a), _ptr(b), bd, _ptr(gamma), _ptr(beta), rows, cols,
         float(eps), _ptr(s), _ptr(y), _ptr(mean), _ptr(rstd), _stream())
    return y, (s if s is not None else a), mean, rstd


def layernorm_bwd(dy: torch.Tensor, s, mean, rstd, gamma, dgamma, dbeta) -> torch.Tensor:
    """dx of LN; dgamma / dbeta are ADDED into the given FP32 buffers."""
    _req(dy, "dy", (torch.float32,))
    cols = dy.shape[-1]
    rows = dy.numel() // cols
    dx = torch.empty_like(dy)
    call("qsync_layernorm_bwd", _ptr(dy), _ptr(s), _ptr(mean), _ptr(rstd), _ptr(gamma), rows, cols,
         _ptr(dx), _ptr(dgamma), _ptr(dbeta), _stream())
    return dx


# --------------------------------------------------------------------------- fused layer glue
ACT_NONE, ACT_GELU, ACT_DERIV = _lib.ACT_NONE, _lib.ACT_GELU, _lib.ACT_DERIV


def layernorm_fwd_ex(a, b, gamma, beta, eps: float, want_f16: bool = False,
                     want_absmax: bool = False, s_out: bool = True):
    """LN forward that also emits the next planned op's operand: FP16(y) and/or
    absmax(y) (device float[1]).  Returns (y, s, mean, rstd, y16, absmax)."""
    _req(a, "a", (torch.float32,))
    cols = a.shape[-1]
    rows = a.numel() // cols
    y = torch.empty_like(a)
    s = torch.empty_like(a) if (b is not None and s_out) else None
    mean = torch.empty(rows, device=a.device, dtype=torch.float32)
    rstd = torch.empty(rows, device=a.device, dtype=torch.float32)
    y16 = torch.empty(a.shape, device=a.device, dtype=torch.float16) if want_f16 else None
    am = torch.empty(1, device=a.device, dtype=torch.float32) if want_absmax else None
    bd = F32
    if b is not None:
        _req(b, "b", (torch.float32, torch.float16))
        bd = _DT[b.dtype]
    call("qsync_layernorm_fwd_ex", _ptr(a), _ptr(b), bd, _ptr(gamma), _ptr(beta), rows, cols,
         float(eps), _ptr(s), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(y16), _ptr(am), _stream())
    return y, (s if s is not None else a), mean, rstd, y16, am


def layernorm_fwd_quant(a, b, gamma, beta, eps: float, s_out: bool = True):
    """LN forward fused with the per-tensor INT8 quantizer of y (the input of an
    INT8-planned Linear).  Returns (y, s, mean, rstd, q, scale, q16): scale =
    device float[2] (s = absmax/127, absmax), q16 = FP16(q) for the wgrad."""
    _req(a, "a", (torch.float32,))
    cols = a.shape[-1]
    rows = a.numel() // cols
    y = torch.empty_like(a)
    s = torch.empty_like(a) if (b is not None and s_out) else None
    mean = torch.empty(rows, device=a.device, dtype=torch.float32)
    rstd = torch.empty(rows, device=a.device, dtype=torch.float32)
    q = torch.empty(a.shape, device=a.device, dtype=torch.int8)
    q16 = torch.empty(a.shape, device=a.device, dtype=torch.float16)
    sc = torch.empty(2, device=a.device, dtype=torch.float32)
    bd = F32
    if b is not None:
        _req(b, "b", (torch.float32, torch.float16))
        bd = _DT[b.dtype]
    call("qsync_layernorm_fwd_quant", _ptr(a), _ptr(b), bd, _ptr(gamma), _ptr(beta), rows, cols, float(eps),
         _ptr(s), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(q), _ptr(q16), _ptr(sc), _stream())
    return y, (s if s is not None else a), mean, rstd, q, sc, q16


def layernorm_bwd_ex(dy, s, mean, rstd, gamma, dgamma, dbeta, want_f16: bool = False,
                     colsum_into=None, out=None):
    """LN backward; also FP16(dx) and dx's column sums ADDED into ``colsum_into``.
    Returns (dx, dx16)."""
    _req(dy, "dy", (torch.float32,))
    cols = dy.shape[-1]
    rows = dy.numel() // cols
    dx = out if out is not None else torch.empty_like(dy)
    dx16 = torch.empty(dy.shape, device=dy.device, dtype=torch.float16) if want_f16 else None
    call("qsync_layernorm_bwd_ex", _ptr(dy), _ptr(s), _ptr(mean), _ptr(rstd), _ptr(gamma), rows,
         cols, _ptr(dx), _ptr(dgamma), _ptr(dbeta), _ptr(dx16), _ptr(colsum_into), _stream())
    return dx, dx16


def absmax_act(x: torch.Tensor, act: int = ACT_NONE, out=None) -> torch.Tensor:
    _req(x, "x", _DT)
    o = out if out is not None else torch.empty(1, device=x.device, dtype=torch.float32)
    call("qsync_absmax_act", _ptr(x), _DT[x.dtype], x.numel(), int(act), _ptr(o), _stream())
    return o


def quantize_act(x: torch.Tensor, absmax: torch.Tensor, act: int = ACT_NONE, want_dact: bool = False,
                 want_q16: bool = False):
    """q = sat(rint(act(x) / s)), s = absmax/127 from a device absmax.
    Returns (q, s[1]) [+ act'(x) FP16 with ``want_dact``] [+ FP16(q) with ``want_q16``]."""
    _req(x, "x", _DT)
    q = torch.empty(x.shape, device=x.device, dtype=torch.int8)
    s = torch.empty(1, device=x.device, dtype=torch.float32)
    d = torch.empty(x.shape, device=x.device, dtype=torch.float16) if want_dact else None
    h = torch.empty(x.shape, device=x.device, dtype=torch.float16) if want_q16 else None
    call("qsync_quantize_act_ex", _ptr(x), _DT[x.dtype], x.numel(), int(act), _ptr(absmax), _ptr(q),
         _ptr(s), _ptr(d), _ptr(h), _stream())
    out = (q, s) + ((d,) if want_dact else ()) + ((h,) if want_q16 else ())
    return out


def gelu_absmax_store(x: torch.Tensor, want_dact: bool = True):
    """(absmax[1], y = GELU(x) in x's dtype, GELU'(x) FP16 or None) from one erf per element."""
    _req(x, "x", (torch.float32, torch.float16))
    am = torch.empty(1, device=x.device, dtype=torch.float32)
    y = torch.empty_like(x)
    d = torch.empty(x.shape, device=x.device, dtype=torch.float16) if want_dact else None
    call("qsync_gelu_absmax_store", _ptr(x), _DT[x.dtype], x.numel(), _ptr(am), _ptr(y), _ptr(d), _stream())
    return am, y, d


def act_cast(x: torch.Tensor, dtype: torch.dtype, act: int = ACT_NONE, out=None, want_dact: bool = False):
    """act(x) as dtype; with ``want_dact`` returns (y, act'(x) FP16)."""
    _req(x, "x", (torch.float32, torch.float16))
    o = out if out is not None else torch.empty(x.shape, device=x.device, dtype=dtype)
    d = torch.empty(x.shape, device=x.device, dtype=torch.float16) if want_dact else None
    call("qsync_act_cast", _ptr(x), _DT[x.dtype], _ptr(o), _DT[dtype], x.numel(), int(act), _ptr(d),
         _stream())
    return (o, d) if want_dact else o


def act_bwd_colsum(dy: torch.Tensor, h: torch.Tensor | None, act: int = ACT_NONE,
                   out_dtype: torch.dtype | None = torch.float16, colsum_into=None):
    """g = dy * act'(h) as out_dtype (None: no output), column sums ADDED into ``colsum_into``."""
    _req(dy, "dy", (torch.float32, torch.float16, torch.bfloat16))
    if h is not None:
        _req(h, "h", (torch.float32, torch.float16))
    cols = dy.shape[-1]
    rows = dy.numel() // cols
    o = torch.empty(dy.shape, device=dy.device, dtype=out_dtype) if out_dtype is not None else None
    call("qsync_act_bwd_colsum", _ptr(dy), _DT[dy.dtype], _ptr(h), _DT[h.dtype] if h is not None else F32,
         rows, cols, int(act), _ptr(o), _DT[out_dtype] if out_dtype is not None else F32,
         _ptr(colsum_into), _stream())
    return o


def gemm_s8_ex(a: torch.Tensor, b: torch.Tensor, scale_a, scale_b, bias=None,
               out_dtype=torch.float32, b_per_channel: bool = True, out=None) -> torch.Tensor:
    """INT8 GEMM + dequant epilogue written as out_dtype (F32 / F16)."""
    _req(a, "a", (torch.int8,))
    _req(b, "b", (torch.int8,))
    M, K = a.shape
    N = b.shape[0]
    c = out if out is not None else torch.empty((M, N), device=a.device, dtype=out_dtype)
    ev = _timed("gemm_s8", 2.0 * M * N * K)
    call("qsync_gemm_s8_ex", _ptr(a), _ptr(b), M, N, K, _ptr(c), _DT[c.dtype], _ptr(scale_a),
         _ptr(scale_b), int(b_per_channel), _ptr(bias), _stream())
    if ev is not None:
        ev.record()
    return c


def gemm_gelu(a: torch.Tensor, b: torch.Tensor, scale_a=None, scale_b=None, bias=None,
              g_dtype=torch.float32, b_per_channel: bool = True):
    """FF1 with its GELU in the epilogue: (absmax[1], g = GELU(y) as g_dtype,
    GELU'(y) FP16) where y is what gemm_s8_ex (INT8 a/b, FP32 y) or gemm_f16
    (FP16 a/b, FP16 y) would return -- bit-identical to that GEMM followed by
    gelu_absmax_store / act_cast(ACT_GELU, want_dact=True)."""
    _req(a, "a", (torch.int8, torch.float16, torch.bfloat16))
    _req(b, "b", (a.dtype,))
    M, K = a.shape
    N = b.shape[0]
    g = torch.empty((M, N), device=a.device, dtype=g_dtype)
    d = torch.empty((M, N), device=a.device, dtype=torch.float16)
    am = torch.empty(1, device=a.device, dtype=torch.float32)
    ev = _timed("gemm_s8" if a.dtype == torch.int8 else "gemm_f16", 2.0 * M * N * K)
    call("qsync_gemm_gelu", _ptr(a), _ptr(b), _DT_CAST[a.dtype], M, N, K, _ptr(scale_a), _ptr(scale_b),
         int(b_per_channel), _ptr(bias), _ptr(g), _DT[g_dtype], _ptr(d), _ptr(am), _stream())
    if ev is not None:
        ev.record()
    return am, g, d


def gemm_s8_ymax(a: torch.Tensor, b: torch.Tensor, scale_a, scale_b, bias=None, b_per_channel: bool = True):
    """(y FP32 as gemm_s8_ex, ymax[1] = max(0, max y))."""
    _req(a, "a", (torch.int8,))
    _req(b, "b", (torch.int8,))
    M, K = a.shape
    N = b.shape[0]
    c = torch.empty((M, N), device=a.device, dtype=torch.float32)
    ym = torch.empty(1, device=a.device, dtype=torch.float32)
    ev = _timed("gemm_s8", 2.0 * M * N * K)
    call("qsync_gemm_s8_ymax", _ptr(a), _ptr(b), M, N, K, _ptr(c), _ptr(scale_a), _ptr(scale_b),
         int(b_per_channel), _ptr(bias), _ptr(ym), _stream())
    if ev is not None:
        ev.record()
    return c, ym


def gelu_quantize(h: torch.Tensor, hmax: torch.Tensor, want_dact: bool = True, want_q16: bool = True):
    """FF2's INT8 operand from FF1's FP32 output in one pass (qsync_gelu_quantize):
    (q, s[1], GELU'(h) FP16 or None, FP16(q) or None) == quantize_act(gelu(h))."""
    _req(h, "h", (torch.float32,))
    q = torch.empty(h.shape, device=h.device, dtype=torch.int8)
    s = torch.empty(2, device=h.device, dtype=torch.float32)
    d = torch.empty(h.shape, device=h.device, dtype=torch.float16) if want_dact else None
    h16 = torch.empty(h.shape, device=h.device, dtype=torch.float16) if want_q16 else None
    call("qsync_gelu_quantize", _ptr(h), h.numel(), _ptr(hmax), _ptr(q), _ptr(h16), _ptr(d), _ptr(s), _stream())
    return q, s[:1], d, h16


def gelu_fp32_check():
    """(monotonicity violations above 0.1701 over float32 [0, 16], max |gelu| for h < 0)."""
    out = torch.zeros(2, dtype=torch.int32, device="cuda")
    call("qsync_gelu_fp32_check", _ptr(out))
    v = out.cpu()
    return int(v[0]), float(v[1:2].view(torch.float32)[0])


def zero_(t: torch.Tensor) -> torch.Tensor:
    """t.zero_() on this library's kernel (16-byte stores)."""
    if t.numel():
        call("qsync_zero", _ptr(t), t.numel() * t.element_size(), _stream())
    return t


def cls_head_fwd(x: torch.Tensor, wp, bp, wc, bc, labels):
    """(loss[1], pooled [B, H], probs [B, C]) of the pooler + classifier + mean CE
    on x [B, S, H] FP32 (qsync_cls_head_fwd)."""
    _req(x, "x", (torch.float32,))
    B, S, H = x.shape
    C = wc.shape[0]
    pooled = torch.empty((B, H), device=x.device, dtype=torch.float32)
    probs = torch.empty((B, C), device=x.device, dtype=torch.float32)
    loss = torch.empty(1, device=x.device, dtype=torch.float32)
    call("qsync_cls_head_fwd", _ptr(x), B, S, H, _ptr(wp), _ptr(bp), _ptr(wc), _ptr(bc), C, _ptr(labels),
         _ptr(pooled), _ptr(probs), _ptr(loss), _stream())
    return loss, pooled, probs


def cls_head_bwd(x, wp, wc, labels, pooled, probs, dloss, dwp, dbp, dwc, dbc):
    """dx [B, S, H]; ADDS the weight / bias gradients into dwp, dbp, dwc, dbc."""
    B, S, H = x.shape
    dpre = torch.empty((9, B, H), device=x.device, dtype=torch.float32)  # dpre + 8 split partials
    dx = torch.empty_like(x)
    call("qsync_cls_head_bwd", _ptr(x), B, S, H, _ptr(wp), _ptr(wc), wc.shape[0], _ptr(labels), _ptr(pooled),
         _ptr(probs), _ptr(dloss), _ptr(dwp), _ptr(dbp), _ptr(dwc), _ptr(dbc), _ptr(dpre), _ptr(dx), _stream())
    return dx


def embed_layernorm_fwd(tokens, word, pos, typ, gamma, beta, eps: float, want_f16: bool = False,
                        want_absmax: bool = False):
    """y = LN(word[tok] + pos[s] + typ[0]) for tokens [B, S] (int64).
    Returns (y [B*S, H], s, mean, rstd, y16, absmax)."""
    _req(tokens, "tokens", (torch.int64,))
    B, S = tokens.shape
    H = word.shape[1]
    rows = B * S
    dev = word.device
    y = torch.empty((rows, H), device=dev, dtype=torch.float32)
    s = torch.empty_like(y)
    mean = torch.empty(rows, device=dev, dtype=torch.float32)
    rstd = torch.empty(rows, device=dev, dtype=torch.float32)
    y16 = torch.empty((rows, H), device=dev, dtype=torch.float16) if want_f16 else None
    am = torch.empty(1, device=dev, dtype=torch.float32) if want_absmax else None
    call("qsync_embed_layernorm_fwd", _ptr(tokens), rows, S, _ptr(word), _ptr(pos), _ptr(typ), _ptr(gamma),
         _ptr(beta), H, float(eps), _ptr(s), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(y16), _ptr(am), _stream())
    return y, s, mean, rstd, y16, am


def embed_layernorm_fwd_quant(tokens, word, pos, typ, gamma, beta, eps: float):
    """embed_layernorm_fwd fused with the INT8 quantizer of y (layernorm_fwd_quant).
    Returns (y [B*S, H], s, mean, rstd, q, scale float[2], q16)."""
    _req(tokens, "tokens", (torch.int64,))
    B, S = tokens.shape
    H = word.shape[1]
    rows = B * S
    dev = word.device
    y = torch.empty((rows, H), device=dev, dtype=torch.float32)
    s = torch.empty_like(y)
    mean = torch.empty(rows, device=dev, dtype=torch.float32)
    rstd = torch.empty(rows, device=dev, dtype=torch.float32)
    q = torch.empty((rows, H), device=dev, dtype=torch.int8)
    q16 = torch.empty((rows, H), device=dev, dtype=torch.float16)
    sc = torch.empty(2, device=dev, dtype=torch.float32)
    call("qsync_embed_layernorm_fwd_quant", _ptr(tokens), rows, S, _ptr(word), _ptr(pos), _ptr(typ), _ptr(gamma),
         _ptr(beta), H, float(eps), _ptr(s), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(q), _ptr(q16), _ptr(sc),
         _stream())
    return y, s, mean, rstd, q, sc, q16


def embed_layernorm_bwd(dy, s, mean, rstd, gamma, tokens, dgamma, dbeta, dword, dpos, dtyp) -> None:
    """Backward of embed_layernorm_fwd; every gradient is ADDED into its buffer."""
    _req(dy, "dy", (torch.float32,))
    B, S = tokens.shape
    call("qsync_embed_layernorm_bwd", _ptr(dy), _ptr(s), _ptr(mean), _ptr(rstd), _ptr(gamma), _ptr(tokens),
         B * S, S, dy.shape[-1], _ptr(dgamma), _ptr(dbeta), _ptr(dword), _ptr(dpos), _ptr(dtyp), _stream())


def attention_fwd(qkv: torch.Tensor, scale: float | None = None, want_absmax: bool = False):
    """Attention core on packed QKV [B, S, 3, H, D] FP16 -> (out [B, S, H, D] FP16,
    lse [B, H, S] FP32, absmax(out) device float[1] or None)."""
    _req(qkv, "qkv", (torch.float16,))
    B, S, _, H, D = qkv.shape
    scale = D ** -0.5 if scale is None else scale
    out = torch.empty((B, S, H, D), device=qkv.device, dtype=torch.float16)
    lse = torch.empty((B, H, S), device=qkv.device, dtype=torch.float32)
    am = torch.empty(1, device=qkv.device, dtype=torch.float32) if want_absmax else None
    call("qsync_attention_fwd", _ptr(qkv), B, S, H, D, float(scale), _ptr(out), _ptr(lse), _ptr(am), _stream())
    return out, lse, am


def attention_fwd_quant(qkv: torch.Tensor, scale: float | None = None, want_q16: bool = True):
    """Attention core for an INT8 O projection: (out, lse, q [B*S, H*D] int8,
    s[1] scale, q16 FP16 grid values or None) -- out / lse as attention_fwd, q /
    s / q16 as quantize_act(out, absmax(out)), from one kernel when it fits."""
    _req(qkv, "qkv", (torch.float16,))
    B, S, _, H, D = qkv.shape
    scale = D ** -0.5 if scale is None else scale
    out = torch.empty((B, S, H, D), device=qkv.device, dtype=torch.float16)
    lse = torch.empty((B, H, S), device=qkv.device, dtype=torch.float32)
    q = torch.empty((B * S, H * D), device=qkv.device, dtype=torch.int8)
    q16 = torch.empty((B * S, H * D), device=qkv.device, dtype=torch.float16) if want_q16 else None
    qs = torch.empty(2, device=qkv.device, dtype=torch.float32)
    call("qsync_attention_fwd_quant", _ptr(qkv), B, S, H, D, float(scale), _ptr(out), _ptr(lse), _ptr(q), _ptr(q16),
         _ptr(qs), _stream())
    return out, lse, q, qs[:1], q16


def attention_bwd(qkv: torch.Tensor, out: torch.Tensor, dout: torch.Tensor, lse: torch.Tensor,
                  scale: float | None = None) -> torch.Tensor:
    """dQKV (packed like qkv) of the attention core."""
    _req(qkv, "qkv", (torch.float16,))
    _req(dout, "dout", (torch.float16,))
    B, S, _, H, D = qkv.shape
    scale = D ** -0.5 if scale is None else scale
    dqkv = torch.empty_like(qkv)
    call("qsync_attention_bwd", _ptr(qkv), _ptr(out), _ptr(dout), _ptr(lse), B, S, H, D, float(scale),
         _ptr(dqkv), _stream())
    return dqkv


def sm_count() -> int:
    return int(_lib.lib().qsync_device_sm_count())


# --------------------------------------------------------------------------- FP8 rung
def quantize_fp8(x: torch.Tensor):
    """Per-tensor E4M3: s = absmax/448, q = e4m3(x / s).  Returns (q float8_e4m3fn, s[1])."""
    _req(x, "x", _DT)
    am = absmax(x)
    q = torch.empty(x.shape, device=x.device, dtype=torch.float8_e4m3fn)
    s = torch.empty(1, device=x.device, dtype=torch.float32)
    call("qsync_quantize_fp8", _ptr(x), _DT[x.dtype], x.numel(), _ptr(am), _ptr(q), _ptr(s), _stream())
    return q, s


def quantize_fp8_rows(w: torch.Tensor):
    """Per-row (output channel) E4M3 of W [N, K]: returns (q, scales[N])."""
    _req(w, "w", (torch.float32,))
    q = torch.empty(w.shape, device=w.device, dtype=torch.float8_e4m3fn)
    s = torch.empty(w.shape[0], device=w.device, dtype=torch.float32)
    call("qsync_quantize_fp8_rows", _ptr(w), w.shape[0], w.shape[1], _ptr(q), _ptr(s), _stream())
    return q, s


def gemm_f8(a: torch.Tensor, b: torch.Tensor, scale_a, scale_b, bias=None, out_dtype=torch.float32,
            b_per_channel: bool = True, out=None) -> torch.Tensor:
    """C = (A B^T) * scale_a * scale_b[n] + bias on tcgen05 kind::f8f6f4 (E4M3, FP32 accumulation)."""
    _req(a, "a", (torch.float8_e4m3fn,))
    _req(b, "b", (torch.float8_e4m3fn,))
    M, K = a.shape
    N = b.shape[0]
    c = out if out is not None else torch.empty((M, N), device=a.device, dtype=out_dtype)
    ev = _timed("gemm_f8", 2.0 * M * N * K)
    call("qsync_gemm_f8", _ptr(a), _ptr(b), M, N, K, _ptr(c), _DT[c.dtype], _ptr(scale_a), _ptr(scale_b),
         int(b_per_channel), _ptr(bias), _stream())
    if ev is not None:
        ev.record()
    return c


def launch_count() -> int:
    """Kernels launched by libqsync_b200 so far in this process."""
    return int(_lib.lib().qsync_launch_count())


def force_splitk(ks: int) -> None:
    """Bench hook: pin the split-K factor of accumulating GEMMs (0 = heuristic)."""
    call("qsync_gemm_force_splitk", int(ks))


def set_streamk(mode: int) -> None:
    """Stream-K scheduling of the plain GEMMs: -1 = never (the tile schedule,
    default: measured faster at the step shapes), 0 = cost model, 1 = wherever
    eligible."""
    call("qsync_gemm_set_streamk", int(mode))


def set_dual_issue(on: bool) -> None:
    """Two MMA issuers for 192-wide single-unit-per-CTA GEMMs (default on)."""
    call("qsync_gemm_set_dual", int(bool(on)))


def force_cta(cta: int) -> None:
    """Test hook: 1 = single-CTA tiles, 2 = CTA-pair (cta_group::2) tiles, 0 = cost model."""
    call("qsync_gemm_force_cta", int(cta))


def force_tile_n(bn: int) -> None:
    """Test hook: pin the GEMM tile N (0 = heuristic)."""
    call("qsync_gemm_force_tile_n", int(bn))


# --------------------------------------------------------------------------- C1
class Communicator:
    """One NCCL communicator of this rank through the C ABI (``qsync_comm_*``):
    the data-parallel gradient exchange of the training step.  ``group`` is any
    initialised torch.distributed process group (gloo or nccl) used once, to
    broadcast rank 0's communicator id -- host plumbing only; the buckets go
    through ``allreduce_bucket`` (ncclAllReduce on the caller's stream)."""

    def __init__(self, world: int, rank: int, group=None, comm_id: bytes | None = None):
        import ctypes as C
        self._C = C
        if comm_id is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                call("qsync_comm_unique_id", C.addressof(buf))
            if world > 1:
                import torch.distributed as dist
                obj = [bytes(buf) if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                comm_id = obj[0]
            else:
                comm_id = bytes(buf)
        idbuf = (C.c_uint8 * 128).from_buffer_copy(comm_id)
        h = C.c_void_p()
        call("qsync_comm_init", C.byref(h), int(world), int(rank), C.addressof(idbuf))
        self.handle = h
        self.world, self.rank = int(world), int(rank)

    def info(self) -> tuple[int, int, int]:
        C = self._C
        n, r, d = C.c_int(), C.c_int(), C.c_int()
        call("qsync_comm_info", self.handle, C.byref(n), C.byref(r), C.byref(d))
        return n.value, r.value, d.value

    def allreduce_bucket(self, buf: torch.Tensor, average: bool = True) -> None:
        """In-place FP32 all-reduce (mean over ranks by default) on the current stream."""
        _req(buf, "bucket", (torch.float32,))
        call("qsync_allreduce_bucket", self.handle, _ptr(buf), buf.numel(), int(average), _stream())

    def close(self) -> None:
        if self.handle is not None and self.handle.value:
            call("qsync_comm_destroy", self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter teardown
            pass


def nccl_version() -> int:
    """Version of the NCCL library the C ABI resolved (e.g. 22809), -1 if none."""
    return int(_lib.lib().qsync_comm_nccl_version())
