"""Layer-fused execution of the planned encoder layer, and the fused optimizer.

The per-operator path (``qlinear.py``) runs each planned Linear as its own
autograd op with the glue (cast, GELU, residual add, LayerNorm) as separate
kernels between them.  Here one autograd Function owns a whole encoder layer,
so the glue folds into the kernels that already touch each tensor:

forward, per planned op P (INT8 / FP16 / FP32; precision.hpp:12):
  * the LayerNorm that produces an op's input also emits that op's operand
    format: FP16(y) for an FP16 op, absmax(y) for an INT8 op (its per-tensor
    quantizer is then one pass) -- ``layernorm_fwd_ex``;
  * an INT8 QKV projection writes its dequantized output as FP16 straight from
    the GEMM epilogue; the attention core (FP16) is this
    package's kernel (csrc/attn.cu), reading the packed QKV as the projection
    wrote it and emitting absmax(out) for an INT8 O projection;
  * GELU is applied inside the FF2 operand kernel: absmax(gelu(h)) then
    quantize(gelu(h)) for INT8, cast(gelu(h)) for FP16 -- the FP32 GELU output
    is never materialised;
  * weights are read in the plan's format from copies the optimizer emitted
    when it last updated them (``FusedAdamW``): per-channel INT8 W^ + scales
    and FP16 W.
backward (cost_mapper.cpp:13-15: FP16 for INT8/FP16 ops, wgrad FP32 :48-50):
  * LayerNorm backward also emits FP16(dx) (the next op's dY) and dx's column
    sums (that op's bias gradient);
  * GELU backward is fused with FF1's FP16 dY cast and bias column sums, and
    reads GELU'(h) (FP16) that FF2's operand kernel stored in the forward;
  * the dgrad of the op that reads the residual stream is reduce-added by the
    GEMM epilogue (TMA reduce-add) into the LayerNorm-backward output, which is
    the residual gradient: no separate add;
  * wgrad (and bias) accumulate into the flat FP32 gradient buffer
    (``main_grad``); wgrad GEMMs run on the side stream.

Numerics are those of the per-operator path (same kernels, same scale rules):
the INT8 quantized operands and int32 GEMM accumulators are bit-identical;
FP16 paths differ only where a value is now rounded once instead of twice.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import ops
from . import qlinear as _ql
from ._lib import call
from .qlinear import FP16, FP32, INT8

_p = lambda t: None if t is None else t.data_ptr()  # noqa: E731


# =============================================================================== optimizer
class _Seg(C.Structure):
    """Mirror of qsync_adamw_seg (include/qsync_b200.h)."""
    _fields_ = [("p", C.c_void_p), ("g", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p),
                ("w16", C.c_void_p), ("wq", C.c_void_p), ("wscale", C.c_void_p),
                ("rows", C.c_int64), ("cols", C.c_int64)]


class FusedAdamW:
    """AdamW on FP32 master weights (torch.optim.AdamW semantics, decoupled
    decay) in ONE kernel over all parameters, which also re-emits the planned
    Linears' weight copies (FP16 W; per-channel INT8 W^ + scales) from the
    updated weights -- ``qsync_adamw_step``.  Gradients are read from each
    parameter's ``main_grad`` (the flat FP32 buffer)."""

    def __init__(self, params, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 1e-2):
        self.params = [p for p in params if p.requires_grad]
        self.lr, self.betas, self.eps, self.wd = lr, betas, eps, weight_decay
        dev = self.params[0].device
        self.m = [torch.zeros_like(p) for p in self.params]
        self.v = [torch.zeros_like(p) for p in self.params]
        self.step_t = torch.zeros(1, dtype=torch.int64, device=dev)
        self._prep: dict[int, object] = {}  # id(weight) -> QLinear
        self._build()

    def attach(self, qlinears) -> None:
        """(Re)allocate the weight copies each planned Linear's precision needs
        and compute them from the current weights."""
        self._prep = {}
        for m in qlinears:
            w = m.weight
            m.w16 = m.wq = m.ws = None
            if m.precision in (INT8, FP16):
                m.w16 = torch.empty(w.shape, device=w.device, dtype=torch.float16)
            if m.precision == INT8:
                m.wq = torch.empty(w.shape, device=w.device, dtype=torch.int8)
                m.ws = torch.empty(w.shape[0], device=w.device, dtype=torch.float32)
            if m.w16 is not None:
                self._prep[id(w)] = m
        self._build()
        self.prepare()

    def _build(self) -> None:
        segs = (_Seg * len(self.params))()
        starts = [0]
        for i, p in enumerate(self.params):
            g = getattr(p, "main_grad", None)
            if g is None:
                g = p.grad if p.grad is not None else torch.zeros_like(p)
                p.grad = g
            rows = p.shape[0] if p.dim() == 2 else 1
            cols = p.numel() // rows
            mod = self._prep.get(id(p))
            s = segs[i]
            s.p, s.g, s.m, s.v = p.data_ptr(), g.data_ptr(), self.m[i].data_ptr(), self.v[i].data_ptr()
            s.w16 = _p(getattr(mod, "w16", None)) if mod is not None else None
            s.wq = _p(getattr(mod, "wq", None)) if mod is not None else None
            s.wscale = _p(getattr(mod, "ws", None)) if mod is not None else None
            s.rows, s.cols = rows, cols
            starts.append(starts[-1] + rows)
        self._index = {id(p): i for i, p in enumerate(self.params)}
        self._row_start = starts
        raw = np.frombuffer(bytes(segs), dtype=np.uint8).copy()
        dev = self.params[0].device
        self._segs = torch.from_numpy(raw).to(dev)
        self._starts = torch.tensor(starts, dtype=torch.int64, device=dev)
        self._nseg = len(self.params)
        self._rows = starts[-1]

    def _launch(self, update: int) -> None:
        call("qsync_adamw_step", self._segs.data_ptr(), self._nseg, self._starts.data_ptr(),
             self._rows, self.step_t.data_ptr(), float(self.lr), float(self.betas[0]),
             float(self.betas[1]), float(self.eps), float(self.wd), int(update),
             torch.cuda.current_stream().cuda_stream)

    def step(self) -> None:
        self._launch(1)

    def rows_of(self, params) -> tuple[int, int]:
        """Global row range [begin, end) covering ``params`` (contiguous in the
        optimizer's parameter order, as a gradient bucket is)."""
        idx = [self._index[id(p)] for p in params if id(p) in self._index]
        if not idx:
            return 0, 0
        return self._row_start[min(idx)], self._row_start[max(idx) + 1]

    def step_range(self, r0: int, r1: int) -> None:
        """Update rows [r0, r1) now (bucket-wise optimizer); no step advance."""
        if r1 > r0:
            call("qsync_adamw_step_range", self._segs.data_ptr(), self._nseg, self._starts.data_ptr(), int(r0),
                 int(r1), self.step_t.data_ptr(), float(self.lr), float(self.betas[0]), float(self.betas[1]),
                 float(self.eps), float(self.wd), 1, torch.cuda.current_stream().cuda_stream)

    def advance(self) -> None:
        """Advance the device step counter once every range of the step is enqueued."""
        call("qsync_adamw_advance", self.step_t.data_ptr(), torch.cuda.current_stream().cuda_stream)

    def prepare(self) -> None:
        """Recompute the weight copies from the current weights (no update)."""
        if self._prep:
            self._launch(0)
            for m in self._prep.values():
                m._wver = m.weight._version

    def refresh_if_stale(self) -> None:
        """Re-emit the copies when a weight changed OUTSIDE this optimizer since
        they were written (load_state_dict, a DP broadcast, manual edits bump the
        tensor version; the update kernel writes weights and copies together and
        leaves the version alone), so the forward never runs on stale copies."""
        if any(getattr(m, "_wver", None) != m.weight._version for m in self._prep.values()):
            self.prepare()


# =============================================================================== profiling marks
# Operator-region marks for the fused-implementation profiler
# (profiler.measure_fused_costs): REGION(kind, op) is called where the device work
# of (kind, op) begins -- kind "fwd" / "bwd" / "cast" (an op's input conversion)
# / "opt" -- and each region ends at the next mark.  None in training: no cost.
REGION = None


def _mark(kind: str, op: str) -> None:
    if REGION is not None:
        REGION(kind, op)


# =============================================================================== layer
def _operand(x, aux, prec):
    """The planned op's input operand (and what its backward keeps)."""
    if isinstance(aux, tuple):  # produced by the upstream kernel (LayerNorm + quantizer)
        assert prec == INT8 and aux[0] == "i8"
        return aux
    if prec == INT8:
        if aux is not None and aux.dtype == torch.float32 and aux.numel() == 1:
            # the quantizer also writes FP16(q) for the wgrad (no cast kernel there)
            xq, s, x16 = ops.quantize_act(x, aux, want_q16=True)
            return ("i8", xq, s, x16)
        xq, sc, _ = ops.quantize_per_tensor(x)
        return ("i8", xq, sc[:1])
    if prec == FP16:
        if x.dtype == torch.float16:
            return ("f16", x, None)
        if aux is not None and aux.dtype == torch.float16:
            return ("f16", aux, None)
        return ("f16", ops.cast(x, torch.float16), None)
    return ("f32", x.float() if x.dtype != torch.float32 else x, None)


def _weights(m):
    """(wq, ws, w16) of a planned Linear: the optimizer-emitted copies when
    present and current, else made now (standalone use, or the weight changed
    outside the optimizer since the copies were written)."""
    if getattr(m, "_wver", None) is not None and m._wver != m.weight._version:
        with torch.no_grad():
            if getattr(m, "wq", None) is not None:
                wq, ws, _ = ops.quantize_per_channel(m.weight.detach())
                m.wq.copy_(wq)
                m.ws.copy_(ws)
            if getattr(m, "w16", None) is not None:
                m.w16.copy_(ops.cast(m.weight.detach(), torch.float16))
        m._wver = m.weight._version
    if m.precision == INT8:
        if getattr(m, "wq", None) is not None:
            return m.wq, m.ws, m.w16
        wq, ws, _ = ops.quantize_per_channel(m.weight.detach())
        return wq, ws, ops.cast(m.weight.detach(), torch.float16)
    if m.precision == FP16:
        if getattr(m, "w16", None) is not None:
            return None, None, m.w16
        return None, None, ops.cast(m.weight.detach(), torch.float16)
    return None, None, None


def _linear_fwd(m, opnd, out_dtype=None):
    kind, x, s = opnd[:3]
    w, b = m.weight, m.bias
    bias = b.detach() if b is not None else None
    wq, ws, w16 = _weights(m)
    if kind == "i8":
        y = ops.gemm_s8_ex(x, wq, s, ws, bias, out_dtype=out_dtype or torch.float32)
    elif kind == "f16":
        y = ops.gemm_f16(x, w16, out_dtype=torch.float16, bias=bias)
    else:  # FP32 plan: tensor cores through the 3xTF32 split (FP32-level accuracy)
        y = ops.gemm_f32(x, w.detach(), bias=bias)
    return y, w16


# INT8 FF1 -> INT8 FF2: FF1's GEMM reduces max(h), then one pass builds FF2's
# operand (qsync_gemm_s8_ymax + qsync_gelu_quantize).  A/B: ab_step onepass=1,0.
GELU_ONE_PASS = True

# INT8 O projection: its operand quantized inside the attention kernel
# (qsync_attention_fwd_quant) instead of a quantize_act pass over the output.
# Off: bit-identical but ~2 us per layer slower (the grid barrier waits for the
# slowest (batch, head) block and holds the dependents' launch; the separate
# one-pass quantizer reads the 3 MB output from L2 under PDL).  ab_step attnq=1,0:
# int8 plan 4.71 vs 4.69 ms, mixed 4.52 vs 4.49.
ATTN_QUANT = False

# INT8 FF2 operand from h: absmax(gelu(h)) then quantize(gelu(h)) with GELU'
# (GELU evaluated twice, g never stored: 162 MB moved at [4096, 3072] FP32 h)
# instead of gelu_absmax_store + a quantize of the stored g (212 MB).  Off:
# measured slower even with the one-exponential GELU (tools/ab_step.py
# ff2recompute=1,0: int8 plan 5.19 vs 5.03 ms, mixed 4.95 vs 4.87).
FF2_INT8_RECOMPUTE = False

# GELU in FF1's GEMM epilogue (qsync_gemm_gelu) instead of the GELU-applying FF2
# operand kernel after a plain GEMM.  Off: measured SLOWER (tools/ab_step.py
# ff1gelu=1,0 on one B200: int8 plan 5.48 vs 5.00 ms, fp16 4.99 vs 4.66, mixed
# 5.27 vs 4.87; 128/192-wide tiles no better).  The erf GELU + GELU' is ~45
# instructions per element; in the epilogue it runs on 8 warps per SM and stalls
# the tile pipeline, where the standalone kernel spreads it over full occupancy.
FF1_GELU_EPILOGUE = False


def _ff1_gelu(m, opnd, g_dtype):
    """FF1 (INT8 / FP16 operand) with GELU in the GEMM epilogue: (absmax(g), g,
    GELU'(h) FP16, w16) -- ops.gemm_gelu."""
    kind, x, s = opnd[:3]
    bias = m.bias.detach() if m.bias is not None else None
    wq, ws, w16 = _weights(m)
    if kind == "i8":
        am, g, gp = ops.gemm_gelu(x, wq, s, ws, bias, g_dtype=g_dtype)
    else:
        am, g, gp = ops.gemm_gelu(x, w16, bias=bias, g_dtype=g_dtype)
    return am, g, gp, w16


# Side-stream wgrad GEMMs launched with programmatic dependent launch (each
# follows an event wait on the main stream).  A/B: tools/ab_step.py wgradpdl=1,0.
WGRAD_PDL = True

# Persistent-grid cap for the side-stream wgrad GEMMs (0 = all SMs): leaves SMs
# to the critical-path chain on the main stream.  Set by TrainStep / tools.
WGRAD_CTAS = 0


def _call_cap(n):
    call("qsync_gemm_set_max_ctas", int(n))


def _wgrad(m, dy16_or_32, opnd, side):
    """wgrad of one planned op into weight.main_grad (FP32, accumulate)."""
    kind, x, s = opnd[:3]
    mw = m.weight.main_grad
    if kind == "i8":  # FP16 copy of the INT8 grid values (exact), from the quantizer when it wrote one
        x16 = opnd[3] if len(opnd) > 3 else ops.cast(x, torch.float16)
    else:
        x16 = x

    def run():
        if side is not None and WGRAD_CTAS:
            _call_cap(WGRAD_CTAS)
        if side is not None and not WGRAD_PDL:
            call("qsync_gemm_set_pdl", 0)
        try:
            if kind == "f32":  # training-device FP32 wgrad: 3xTF32 on the tensor cores
                ops.gemm_f32(dy16_or_32.float().contiguous(), x16, out=mw, accumulate=True, a_mn=True,
                             b_mn=True)
            else:
                ops.gemm_f16(dy16_or_32, x16, alpha_dev=s, out=mw, accumulate=True, a_mn=True, b_mn=True)
        finally:
            if side is not None and WGRAD_CTAS:
                _call_cap(0)
            if side is not None and not WGRAD_PDL:
                call("qsync_gemm_set_pdl", 1)

    if side is not None:
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            run()
        for t in (dy16_or_32, x16, s):
            if t is not None:
                t.record_stream(side)
    else:
        run()


def _dgrad(m, dy, w16, out_dtype, acc_into=None):
    """dgrad of one planned op: FP16 GEMM (INT8/FP16 ops) or FP32 (FP32 op);
    with ``acc_into`` the result is ADDED into that FP32 buffer."""
    if m.precision == FP32:  # 3xTF32 on the tensor cores (FP32-level accuracy)
        dyf = dy.float().contiguous()
        if acc_into is not None:
            return ops.gemm_f32(dyf, m.weight.detach(), out=acc_into, accumulate=True, b_mn=True)
        d = ops.gemm_f32(dyf, m.weight.detach(), b_mn=True)
        return d if out_dtype == torch.float32 else d.to(out_dtype)
    if acc_into is not None:
        return ops.gemm_f16(dy, w16, out=acc_into, accumulate=True, b_mn=True)
    return ops.gemm_f16(dy, w16, out_dtype=out_dtype, b_mn=True)


def _bias_main_grad(m):
    return m.bias.main_grad if m.bias is not None else None


def _need_aux(prec):
    return (prec == FP16, prec == INT8)


class _FusedLayerFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x0, aux0, layer, next_prec):
        L = layer
        B, S, H = x0.shape
        nh = L.cfg.heads
        M = B * S
        x0f = x0.reshape(M, H)
        pq, po, p1, p2 = L.qkv.precision, L.o.precision, L.ff1.precision, L.ff2.precision
        # --- QKV projection -> FP16 packed QKV for the attention core
        pre = L.qkv.name.rsplit(".", 1)[0]
        _mark("cast", L.qkv.name)
        op_qkv = _operand(x0f, aux0, pq)
        _mark("fwd", L.qkv.name)
        qkv, w16_qkv = _linear_fwd(L.qkv, op_qkv, out_dtype=torch.float16)
        if qkv.dtype != torch.float16:
            qkv = ops.cast(qkv, torch.float16)
        qkv5 = qkv.view(B, S, 3, nh, H // nh)
        scale = (H // nh) ** -0.5
        # Attention core (FP16, csrc/attn.cu); it also emits absmax(out) when the
        # O projection is INT8, so that op's quantizer is one pass.
        _mark("fwd", pre + ".attn")
        if po == INT8 and ATTN_QUANT:
            # the attention kernel also quantizes its output for the INT8 O
            # projection (grid barrier on absmax): no separate quantizer pass
            a, lse, aq, as_, aq16 = ops.attention_fwd_quant(qkv5, scale)
            a2 = a.reshape(M, H)
            _mark("cast", L.o.name)
            op_o = ("i8", aq, as_, aq16)
        else:
            a, lse, a_am = ops.attention_fwd(qkv5, scale, want_absmax=po == INT8)
            a2 = a.reshape(M, H)
            # --- output projection + residual LayerNorm (emits FF1's operand)
            _mark("cast", L.o.name)
            op_o = _operand(a2, a_am, po)
        _mark("fwd", L.o.name)
        yo, w16_o = _linear_fwd(L.o, op_o)
        f16, am = _need_aux(p1)
        _mark("fwd", pre + ".ln1")
        if am:  # INT8 FF1: LayerNorm and its per-tensor quantizer in one kernel
            x1, s1, mean1, rstd1, q1, sc1, q1_16 = ops.layernorm_fwd_quant(
                x0f, yo, L.ln1.weight.detach(), L.ln1.bias.detach(), L.ln1.eps)
            aux1 = ("i8", q1, sc1[:1], q1_16)
        else:
            x1, s1, mean1, rstd1, x1_16, _ = ops.layernorm_fwd_ex(
                x0f, yo, L.ln1.weight.detach(), L.ln1.bias.detach(), L.ln1.eps, f16, False)
            aux1 = x1_16 if f16 else None
        # --- FF1 -> GELU: in FF1's GEMM epilogue (INT8 / FP16 FF1), else folded
        # into FF2's operand kernel; either way GELU'(h) is stored in FP16 for the
        # backward, which then needs no transcendental (dh = dg * GELU'(h)).
        _mark("cast", L.ff1.name)
        op_1 = _operand(x1, aux1, p1)
        _mark("fwd", L.ff1.name)
        h = None
        hmax = None
        if FF1_GELU_EPILOGUE and op_1[0] in ("i8", "f16") and L.ff1.weight.shape[0] % 8 == 0:
            # g in the dtype the FF2 operand kernel reads, GELU'(h) and absmax(g),
            # bit-identical to the GEMM + operand kernel below; h is never stored.
            h_dtype = torch.float32 if op_1[0] == "i8" else torch.float16
            gdt = h_dtype if p2 == INT8 else (torch.float16 if p2 == FP16 else torch.float32)
            gam, g_act, gp, w16_1 = _ff1_gelu(L.ff1, op_1, gdt)
        elif op_1[0] == "i8" and p2 == INT8 and GELU_ONE_PASS:
            # INT8 FF1 -> INT8 FF2: the GEMM also reduces max(h), then one pass
            # quantizes gelu(h) (no GELU(h) stored, no absmax pass; bit-identical)
            wq1, ws1, w16_1 = _weights(L.ff1)
            h, hmax = ops.gemm_s8_ymax(op_1[1], wq1, op_1[2], ws1,
                                       L.ff1.bias.detach() if L.ff1.bias is not None else None)
            h_dtype = h.dtype
        else:
            h, w16_1 = _linear_fwd(L.ff1, op_1)
            h_dtype = h.dtype
        _mark("fwd", pre + ".gelu")
        if p2 == INT8 and hmax is not None:
            gq, gs, gp, g16 = ops.gelu_quantize(h, hmax)
            op_2 = ("i8", gq, gs, g16)
        elif p2 == INT8:
            if h is not None and FF2_INT8_RECOMPUTE:
                # two reads of h, GELU evaluated in both (absmax, then quantize +
                # GELU' + FP16 q): g is never stored (bit-identical q, s, GELU')
                gam = ops.absmax_act(h, ops.ACT_GELU)
                gq, gs, gp, g16 = ops.quantize_act(h, gam, ops.ACT_GELU, want_dact=True, want_q16=True)
            else:
                if h is not None:
                    # one GELU evaluation: g (and GELU') stored with the absmax pass
                    gam, g_act, gp = ops.gelu_absmax_store(h)
                # the quantizer is then a pure streaming pass over g (bit-identical q, s)
                gq, gs, g16 = ops.quantize_act(g_act, gam, want_q16=True)
                del g_act
            op_2 = ("i8", gq, gs, g16)
        elif p2 == FP16:
            if h is not None:
                g_act, gp = ops.act_cast(h, torch.float16, ops.ACT_GELU, want_dact=True)
            op_2 = ("f16", g_act, None)
        else:
            if h is not None:
                g_act, gp = ops.act_cast(h, torch.float32, ops.ACT_GELU, want_dact=True)
            op_2 = ("f32", g_act, None)
        _mark("fwd", L.ff2.name)
        f, w16_2 = _linear_fwd(L.ff2, op_2)
        f16n, amn = _need_aux(next_prec)
        _mark("fwd", pre + ".ln2")
        none = torch.empty(0, device=x0.device)
        if amn:  # the next layer's INT8 QKV operand straight out of LN2
            x2, s2, mean2, rstd2, q2, sc2, q2_16 = ops.layernorm_fwd_quant(
                x1, f, L.ln2.weight.detach(), L.ln2.bias.detach(), L.ln2.eps)
            auxes = (q2, sc2, q2_16)
        else:
            x2, s2, mean2, rstd2, x2_16, _ = ops.layernorm_fwd_ex(
                x1, f, L.ln2.weight.detach(), L.ln2.bias.detach(), L.ln2.eps, f16n, False)
            auxes = (x2_16 if f16n else none, none, none)

        ctx.layer = L
        ctx.ops_ = (op_qkv, op_o, op_1, op_2)
        ctx.w16 = (w16_qkv, w16_o, w16_1, w16_2)
        ctx.attn = (qkv5, a, lse, scale)
        ctx.ln = (s1, mean1, rstd1, s2, mean2, rstd2)
        ctx.h = (h_dtype, gp)  # GELU'(h) is all the backward needs of h
        ctx.shape = (B, S, H)
        out = x2.view(B, S, H)
        ctx.mark_non_differentiable(*auxes)
        ctx.set_materialize_grads(False)  # no zero-filled gradient for the aux outputs
        return (out,) + auxes

    @staticmethod
    def backward(ctx, dx2, _daux, _ds, _d16):
        L = ctx.layer
        B, S, H = ctx.shape
        M = B * S
        op_qkv, op_o, op_1, op_2 = ctx.ops_
        w16_qkv, w16_o, w16_1, w16_2 = ctx.w16
        qkv5, a, lse, scale = ctx.attn
        s1, mean1, rstd1, s2, mean2, rstd2 = ctx.ln
        h_dtype, gp = ctx.h
        side = _ql.WGRAD_STREAM
        dx2 = dx2.reshape(M, H).contiguous()
        if dx2.dtype != torch.float32:
            dx2 = dx2.float()
        # --- LN2 backward -> FF2's dY (FP16) + ff2 bias grad
        p2 = L.ff2.precision
        pre = L.qkv.name.rsplit(".", 1)[0]
        _mark("bwd", pre + ".ln2")
        ds2, ds2_16 = ops.layernorm_bwd_ex(dx2, s2, mean2, rstd2, L.ln2.weight.detach(),
                                           L.ln2.weight.main_grad, L.ln2.bias.main_grad,
                                           want_f16=p2 != FP32, colsum_into=_bias_main_grad(L.ff2))
        dy2 = ds2_16 if p2 != FP32 else ds2
        # FF2's FP16 backward kernel emits its input gradient in FP16 (as the
        # reference's FP16 op does before the cast back), halving dG's traffic
        _mark("bwd", L.ff2.name)
        dg = _dgrad(L.ff2, dy2, w16_2, torch.float16 if p2 != FP32 else h_dtype)
        _wgrad(L.ff2, dy2, op_2, side if p2 != FP32 else None)
        # --- GELU backward fused with FF1's dY cast + ff1 bias grad
        p1 = L.ff1.precision
        _mark("bwd", pre + ".gelu")
        dh = ops.act_bwd_colsum(dg, gp, ops.ACT_DERIV,
                                out_dtype=torch.float16 if p1 != FP32 else torch.float32,
                                colsum_into=_bias_main_grad(L.ff1))
        # FF1 dgrad reduce-added into ds2: ds2 becomes d(x1) = residual + FF1 paths
        _mark("bwd", L.ff1.name)
        _dgrad(L.ff1, dh, w16_1, torch.float32, acc_into=ds2)
        _wgrad(L.ff1, dh, op_1, side if p1 != FP32 else None)
        # --- LN1 backward -> O's dY + o bias grad
        po = L.o.precision
        _mark("bwd", pre + ".ln1")
        ds1, ds1_16 = ops.layernorm_bwd_ex(ds2, s1, mean1, rstd1, L.ln1.weight.detach(),
                                           L.ln1.weight.main_grad, L.ln1.bias.main_grad,
                                           want_f16=po != FP32, colsum_into=_bias_main_grad(L.o))
        dyo = ds1_16 if po != FP32 else ds1
        _mark("bwd", L.o.name)
        da = _dgrad(L.o, dyo, w16_o, torch.float16)
        _wgrad(L.o, dyo, op_o, side if po != FP32 else None)
        # --- attention core backward (FP16) -> packed dQKV
        _mark("bwd", pre + ".attn")
        dqkv = ops.attention_bwd(qkv5, a, da.view(a.shape), lse, scale)
        dqkv2 = dqkv.view(M, 3 * H)
        # --- QKV backward: bias grad (column sums), dgrad reduce-added into ds1
        pq = L.qkv.precision
        _mark("bwd", L.qkv.name)
        mb = _bias_main_grad(L.qkv)
        if pq == FP32:
            dq32 = dqkv2.float()
            if mb is not None:
                mb.add_(dq32.sum(0))
            _dgrad(L.qkv, dq32, None, torch.float32, acc_into=ds1)
            _wgrad(L.qkv, dq32, op_qkv, None)
        else:
            if mb is not None:
                ops.act_bwd_colsum(dqkv2, None, ops.ACT_NONE, out_dtype=None, colsum_into=mb)
            _dgrad(L.qkv, dqkv2, w16_qkv, torch.float32, acc_into=ds1)
            _wgrad(L.qkv, dqkv2, op_qkv, side)
        if _ql.GRAD_READY is not None:
            _ql.GRAD_READY(list(L.parameters()))
        return ds1.view(B, S, H), None, None, None


def fused_layer(layer, x, aux, next_prec):
    """Run one EncoderLayer through the layer-fused Function.  Returns (x, aux)
    where aux is the next planned op's operand hint (FP16 copy or absmax)."""
    from .glue import pack_aux
    out, aux2, s2, q16 = _FusedLayerFn.apply(x, aux, layer, next_prec)
    return out, pack_aux(aux2, s2, q16)
