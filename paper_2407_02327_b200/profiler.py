"""Profiler: measure the hot path on the B200 and emit a QSync ProfileBundle.

The reference planner consumes measured costs (README "Profile bundle
schema"); this module produces them from this package's kernels, in the exact
schema `bundle_from_json` validates (profile.cpp:283-413):

* ``graph``        -- the BERT-base operator DAG: adjustable Linears (INT8/FP16/FP32),
                      dependent GELU, fixed embeddings / attention core / LayerNorm /
                      loss; residual edges included (depth = longest path, graph.cpp:178-183).
* ``op_costs``     -- per (op, precision): ``pure_cost_ns`` = measured fwd + bwd time of
                      the op's kernels on the device (CUDA events), ``fwd_fraction``
                      measured, ``memory_bytes`` = the bytes that precision keeps
                      resident (weights, low-precision copies, saved operands, output).
* ``cast_samples`` -- measured K2/K3/K4 latencies over tensor sizes for every key
                      ``required_cast_keys`` asks for (quantize includes the absmax pass).
* ``tensor_stats`` -- per training step, per adjustable op, the K5 device statistics of
                      the input activation, weight and incoming gradient (OpStats fields).
* ``devices``      -- the DP ranks (a training device + a memory-capped inference device).

The reference's ``plan`` (cli.cpp:116-136) then turns the bundle into per-rank plans
that ``train_step.load_plan`` applies.
"""
from __future__ import annotations

import json
import math
import statistics

import torch
import torch.nn.functional as F

from . import ops, qlinear
from .qlinear import FP16, FP32, INT8, QLinear
from .train_step import BertConfig, BertEncoderStack

_PREC_BYTES = {INT8: 1, FP16: 2, FP32: 4}


# ----------------------------------------------------------------------------- timing
def _time_ns(fn, reps: int = 10) -> int:
    """Median device time of fn() (CUDA events; a device spin keeps launches queued)."""
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        torch.cuda._sleep(2_000_000)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e6)
    return max(1, int(statistics.median(times)))


def _graph_time_ns(fn, n: int = 20, reps: int = 3) -> int:
    """Per-call device time of fn() launched n times back-to-back inside a CUDA
    graph (as in the train step: no launch gaps), best of reps."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e6 / n)
    return max(1, int(best))


def graph_step_ms(cfg: BertConfig, batch: int, plan: dict, steps: int = 20) -> float:
    """The train step as the bench runs it (one CUDA graph, wgrad side stream)."""
    from .train_step import TrainStep
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(plan)
    st = TrainStep(m, batch=batch, graph=True)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        st()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del st, m
    torch.cuda.empty_cache()
    return ms


def graph_fwd_ms(cfg: BertConfig, batch: int, plan: dict, steps: int = 20) -> float:
    """The forward pass of the fused train step alone, as one CUDA graph (the
    forward has no side-stream overlap; used to calibrate forward and backward
    regions separately)."""
    from .train_step import TrainStep
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(plan)
    st = TrainStep(m, batch=batch, graph=False)  # fused layers + the optimizer's prepared weight copies
    tok, lab = st.tokens.random_(0, cfg.vocab), st.labels
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            m(tok, lab)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        m(tok, lab)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del g, st, m
    torch.cuda.empty_cache()
    return ms


# ----------------------------------------------------------------------------- graph
def bert_graph(cfg: BertConfig, batch: int) -> dict:
    T, H, Fh = batch * cfg.seq, cfg.hidden, cfg.ffn
    nodes, edges = [], []

    def node(i, kind, out, sub, prec, w=0):
        nodes.append({"id": i, "kind": kind, "output_numel": out, "subgraph_id": sub,
                      "supported_precisions": prec, "has_weight": w > 0, "weight_numel": w})

    all3 = [INT8, FP16, FP32]
    node("embed", "fixed", T * H, "embed", [FP32])
    prev = "embed"
    for i in range(cfg.layers):
        L = f"layer{i}"
        node(f"{L}.qkv", "adjustable", T * 3 * H, L, all3, 3 * H * H)
        node(f"{L}.attn", "fixed", T * H, L, [FP32])
        node(f"{L}.o", "adjustable", T * H, L, all3, H * H)
        node(f"{L}.ln1", "fixed", T * H, L, [FP32])
        node(f"{L}.ff1", "adjustable", T * Fh, L, all3, Fh * H)
        node(f"{L}.gelu", "dependent", T * Fh, L, [FP16, FP32])
        node(f"{L}.ff2", "adjustable", T * H, L, all3, H * Fh)
        node(f"{L}.ln2", "fixed", T * H, L, [FP32])
        edges += [[prev, f"{L}.qkv"], [f"{L}.qkv", f"{L}.attn"], [f"{L}.attn", f"{L}.o"],
                  [f"{L}.o", f"{L}.ln1"], [prev, f"{L}.ln1"],           # residual
                  [f"{L}.ln1", f"{L}.ff1"], [f"{L}.ff1", f"{L}.gelu"], [f"{L}.gelu", f"{L}.ff2"],
                  [f"{L}.ff2", f"{L}.ln2"], [f"{L}.ln1", f"{L}.ln2"]]  # residual
        prev = f"{L}.ln2"
    node("pooler", "adjustable", batch * H, "head", all3, H * H)
    node("loss", "fixed", batch, "head", [FP32])
    edges += [[prev, "pooler"], ["pooler", "loss"]]
    return {"nodes": nodes, "edges": edges,
            "assignment": {n["id"]: FP32 for n in nodes}}


# ----------------------------------------------------------------------------- op costs
def linear_memory_bytes(precision: str, M: int, N: int, K: int) -> int:
    """Bytes an op keeps resident at a precision: FP32 master weight + its FP32
    gradient + AdamW moments, the precision's operand copies, the operand saved
    for backward, and the output (graph.hpp:38-40 output format)."""
    # What the op itself keeps resident between forward and backward: the FP32
    # master weight, its FP32 gradient and the two AdamW moments, plus the
    # operands saved for backward.  (Its output is the consumer's saved input.)
    W = N * K
    base = 4 * W * 4
    if precision == INT8:
        return base + M * K * 1            # Xq (int8); W16 is recomputed in backward
    if precision == FP16:
        return base + M * K * 2 + W * 2    # X16, W16
    return base + M * K * 4                # X


def measure_linear(M: int, N: int, K: int, precision: str, reps: int = 10) -> dict:
    """``pure_cost_ns`` = the operator's compute kernels only (OpCostEntry,
    profile.hpp:72-76): for INT8/FP16 the fwd GEMM + dgrad + wgrad GEMMs, timed
    per launch with CUDA events; the casts around them (quantize, FP16 casts,
    dequant) are the cast model's job (cost_mapper.cpp:30-53)."""
    lin = QLinear(K, N, "probe", precision=precision).cuda()
    x = torch.randn(M, K, device="cuda", requires_grad=True)
    dy = torch.randn(M, N, device="cuda").to(qlinear.output_dtype(precision))

    def fwd_bwd():
        y = lin(x)
        y.backward(dy)
        lin.weight.grad = None
        lin.bias.grad = None
        x.grad = None

    if precision == FP32:
        def fwd():
            with torch.no_grad():
                lin(x)
        f = _time_ns(fwd, reps)
        t = _time_ns(fwd_bwd, reps)
    else:
        fwd_bwd()
        fs, ts = [], []
        for _ in range(reps):
            ops.GEMM_TIMER = []
            torch.cuda._sleep(5_000_000)
            fwd_bwd()
            torch.cuda.synchronize()
            rec, ops.GEMM_TIMER = ops.GEMM_TIMER, None
            times = [s_.elapsed_time(e_) * 1e6 for _, _, s_, e_ in rec]
            fs.append(times[0])
            ts.append(sum(times))
        f, t = int(statistics.median(fs)), int(statistics.median(ts))
    return {"pure_cost_ns": max(t, f + 1), "fwd_fraction": min(1.0, f / max(t, f + 1)),
            "memory_bytes": linear_memory_bytes(precision, M, N, K)}


def measure_glue(cfg: BertConfig, batch: int, reps: int = 10) -> dict:
    """Costs of the fixed / dependent operators (their FP32 or FP16 kernels)."""
    from .glue import AddLayerNorm, attention
    T, H, Fh = batch * cfg.seq, cfg.hidden, cfg.ffn
    out = {}
    qkv = torch.randn(batch, cfg.seq, 3, cfg.heads, H // cfg.heads, device="cuda",
                      dtype=torch.float16, requires_grad=True)
    g = torch.randn(batch, cfg.seq, cfg.heads, H // cfg.heads, device="cuda", dtype=torch.float16)

    def attn():
        attention(qkv).backward(g)
    t = _time_ns(attn, reps)
    out["attn"] = {FP32: {"pure_cost_ns": t, "fwd_fraction": 1.0 / 3.0,
                          "memory_bytes": T * 3 * H * 2 + T * H * 2}}
    ln = AddLayerNorm(H).cuda()
    a = torch.randn(T, H, device="cuda", requires_grad=True)
    b = torch.randn(T, H, device="cuda", requires_grad=True)
    gy = torch.randn(T, H, device="cuda")

    def lnfb():
        ln(a, b).backward(gy)
    t = _time_ns(lnfb, reps)
    out["ln"] = {FP32: {"pure_cost_ns": t, "fwd_fraction": 1.0 / 3.0,
                        "memory_bytes": T * H * 4 * 2 + 2 * H * 4 * 4}}
    out["gelu"] = {}
    for p, dt in ((FP32, torch.float32), (FP16, torch.float16)):
        xg = torch.randn(T, Fh, device="cuda", dtype=dt, requires_grad=True)
        gg = torch.randn(T, Fh, device="cuda", dtype=dt)

        def gelu(xg=xg, gg=gg):
            F.gelu(xg).backward(gg)
        out["gelu"][p] = {"pure_cost_ns": _time_ns(gelu, reps), "fwd_fraction": 1.0 / 3.0,
                          "memory_bytes": T * Fh * _PREC_BYTES[p] * 2}
    emb = torch.nn.Embedding(cfg.vocab, H).cuda()
    tok = torch.randint(0, cfg.vocab, (batch, cfg.seq), device="cuda")
    ge = torch.randn(batch, cfg.seq, H, device="cuda")

    def embed():
        emb(tok).backward(ge)
    out["embed"] = {FP32: {"pure_cost_ns": _time_ns(embed, reps), "fwd_fraction": 1.0 / 3.0,
                           "memory_bytes": cfg.vocab * H * 4 * 4 + T * H * 4}}
    cls = torch.nn.Linear(H, cfg.num_labels).cuda()
    pooled = torch.randn(batch, H, device="cuda", requires_grad=True)
    lab = torch.randint(0, cfg.num_labels, (batch,), device="cuda")

    def loss():
        F.cross_entropy(cls(pooled), lab).backward()
    out["loss"] = {FP32: {"pure_cost_ns": _time_ns(loss, reps), "fwd_fraction": 1.0 / 3.0,
                          "memory_bytes": H * cfg.num_labels * 16 + batch * H * 4}}
    return out


def measure_op_costs(cfg: BertConfig, batch: int, reps: int = 10) -> dict:
    T, H, Fh = batch * cfg.seq, cfg.hidden, cfg.ffn
    shapes = {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, Fh, H), "ff2": (T, H, Fh)}
    per_shape = {k: {p: measure_linear(*s, p, reps) for p in (INT8, FP16, FP32)}
                 for k, s in shapes.items()}
    pooler = {p: measure_linear(batch, H, H, p, reps) for p in (INT8, FP16, FP32)}
    glue = measure_glue(cfg, batch, reps)
    costs = {"embed": glue["embed"], "pooler": pooler, "loss": glue["loss"]}
    for i in range(cfg.layers):
        L = f"layer{i}"
        for k in shapes:
            costs[f"{L}.{k}"] = per_shape[k]
        costs[f"{L}.attn"] = glue["attn"]
        costs[f"{L}.ln1"] = glue["ln"]
        costs[f"{L}.ln2"] = glue["ln"]
        costs[f"{L}.gelu"] = glue["gelu"]
    return costs


# ----------------------------------------------------------------------------- fused step
def _region_times(st, reps: int) -> dict:
    """Device time per (kind, op) region of one eager fused step (fused.REGION
    marks; single stream, launches queued behind a device spin), median of reps."""
    from . import fused
    runs = []
    for _ in range(reps):
        marks = []

        def hook(kind, op, marks=marks):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((kind, op, e))

        torch.cuda.synchronize()
        torch.cuda._sleep(400_000_000)  # the whole step is enqueued before it runs
        fused.REGION = hook
        try:
            st()
        finally:
            fused.REGION = None
        torch.cuda.synchronize()
        t: dict = {}
        for (k, o, e0), (_, _, e1) in zip(marks, marks[1:]):
            t[(k, o)] = t.get((k, o), 0.0) + e0.elapsed_time(e1) * 1e6
        runs.append(t)
    keys = set().union(*runs)
    return {k: statistics.median(r.get(k, 0.0) for r in runs) for k in keys}


def _param_numel(cfg: BertConfig) -> dict:
    """Parameters the optimizer updates per graph node: (planned weight numel, other numel)."""
    H, Fh = cfg.hidden, cfg.ffn
    out = {"embed": (0, (cfg.vocab + cfg.max_pos + cfg.type_vocab) * H + 2 * H),
           "pooler": (H * H, H), "loss": (0, H * cfg.num_labels + cfg.num_labels)}
    for i in range(cfg.layers):
        L = f"layer{i}"
        for k, (n, kk) in {"qkv": (3 * H, H), "o": (H, H), "ff1": (Fh, H), "ff2": (H, Fh)}.items():
            out[f"{L}.{k}"] = (n * kk, n)
        out[f"{L}.ln1"] = (0, 2 * H)
        out[f"{L}.ln2"] = (0, 2 * H)
    return out


# AdamW bytes per parameter (read p, g, m, v; write p, m, v) plus the weight
# copies the optimizer emits for the planned precision (w16; INT8 also wq).
_OPT_BYTES = {FP32: 28, FP16: 30, INT8: 31}


def measure_fused_costs(cfg: BertConfig, batch: int, reps: int = 5, calibrate: bool = True) -> dict:
    """Per-operator costs of the layer-fused training step as it executes
    (fused.py), for the bundle's ``op_costs``:

    * one eager step per uniform plan (INT8, FP16, FP32) with the wgrad GEMMs on the
      main stream, device time split at the operator-region marks;
    * ``pure_cost_ns`` = the op's fwd + bwd regions plus its parameters' share of
      the gradient zeroing + AdamW step (by bytes the optimizer moves for them: the
      reference models no optimizer time, replayer.cpp:64-73 with a zero-duration
      event, cost_mapper.cpp:127-130);
    * an op's input conversion ("cast" region: the INT8 quantizer) is the cast
      model's, see ``measure_fused_cast_samples``;
    * GELU (dependent) -- FP16 from the FP16 plan, FP32 from the cheaper of the
      INT8 plan (GELU fused with FF2's quantizer) and the FP32 plan;
    * ``calibrate``: the eager single-stream regions are scaled by (graph step time /
      their sum) of the same plan, so each op is charged its share of the step as the
      bench runs it -- the wgrad GEMMs overlapping the main stream and PDL-chained
      kernels, which the reference's sequential per-device model cannot express.
      The uniform plans' predictions then match by construction; a mixed plan is
      predicted from them plus the cast model (``last_diag`` keeps the factors).
    """
    from .train_step import TrainStep, uniform_plan
    T, H = batch * cfg.seq, cfg.hidden
    Fh = cfg.ffn
    per = {}
    for p in (INT8, FP16, FP32):
        torch.manual_seed(0)
        m = BertEncoderStack(cfg).cuda()
        m.apply_plan(uniform_plan(cfg, p) if p != FP32 else {})
        st = TrainStep(m, batch=batch, graph=False, overlap_wgrad=False)
        st.tokens.random_(0, cfg.vocab)
        for _ in range(3):
            st()
        per[p] = _region_times(st, reps)
        del st, m
        torch.cuda.empty_cache()
    diag = {}
    for p in (INT8, FP16, FP32):
        # Forward and backward calibrated separately: only the backward overlaps
        # (wgrad side stream) -- one factor over-shrank the forward regions and
        # over-predicted the backward ones.  fwd + cast regions -> the graphed
        # forward; bwd + opt regions -> the rest of the graphed step.
        plan = uniform_plan(cfg, p) if p != FP32 else {}
        tot = sum(per[p].values())
        tot_f = sum(v for (k, _), v in per[p].items() if k in ("fwd", "cast"))
        graph_ns = graph_step_ms(cfg, batch, plan) * 1e6
        fwd_ns = graph_fwd_ms(cfg, batch, plan) * 1e6
        sf = fwd_ns / tot_f if calibrate and tot_f > 0 else 1.0
        sb = (graph_ns - fwd_ns) / (tot - tot_f) if calibrate and tot > tot_f else 1.0
        diag[p] = {"eager_regions_ms": tot / 1e6, "graph_step_ms": graph_ns / 1e6, "graph_fwd_ms": fwd_ns / 1e6,
                   "scale_fwd": sf, "scale_bwd": sb, "scale": graph_ns / tot if tot else 1.0}
        per[p] = {k: v * (sf if k[0] in ("fwd", "cast") else sb) for k, v in per[p].items()}
    measure_fused_costs.last_diag = diag
    for p in per:  # the pooler is costed from its kernels (measure_linear); its autograd
        # backward region stays with the head's, as before the head had marks
        per[p][("bwd", "loss")] = per[p].get(("bwd", "loss"), 0.0) + per[p].pop(("bwd", "pooler"), 0.0)
    numel = _param_numel(cfg)

    def opt_share(op, p):
        t = per[p]
        t_opt = t.get(("opt", "optimizer"), 0.0) + t.get(("opt", "zero"), 0.0)
        total = sum(w * _OPT_BYTES[p] + b * _OPT_BYTES[FP32] for w, b in numel.values())
        w, b = numel.get(op, (0, 0))  # (attention, GELU: no parameters)
        return t_opt * (w * _OPT_BYTES[p] + b * _OPT_BYTES[FP32]) / total

    def entry(op, p, mem):
        fwd = per[p].get(("fwd", op), 0.0)
        bwd = per[p].get(("bwd", op), 0.0) + opt_share(op, p)
        tot = max(1, int(round(fwd + bwd)))
        return {"pure_cost_ns": tot, "fwd_fraction": min(1.0, fwd / tot), "memory_bytes": mem}

    costs = {}
    shapes = {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, Fh, H), "ff2": (T, H, Fh)}
    pooler = {p: measure_linear(batch, H, H, p) for p in (INT8, FP16, FP32)}
    for p in pooler:
        pooler[p]["pure_cost_ns"] += int(opt_share("pooler", p))
    costs["pooler"] = pooler
    med = statistics.median

    def fixed(op, mem):
        # The FP32 plan's region: in the INT8 / FP16 plans a fixed op's region
        # also holds the conversion of its output for the next planned op
        # (LayerNorm + quantizer / FP16 copy, attention + quantizer), which the
        # cast model charges at that precision boundary.
        e = entry(op, FP32, mem)
        return {FP32: {"pure_cost_ns": e["pure_cost_ns"], "fwd_fraction": e["fwd_fraction"], "memory_bytes": mem}}

    costs["embed"] = fixed("embed", cfg.vocab * H * 4 * 4 + T * H * 4)
    loss = fixed("loss", H * cfg.num_labels * 16 + batch * H * 4)
    # the head's regions also hold the pooler's kernels, costed above from its own
    loss[FP32]["pure_cost_ns"] = max(1, loss[FP32]["pure_cost_ns"] - pooler[FP32]["pure_cost_ns"])
    costs["loss"] = loss
    for i in range(cfg.layers):
        L = f"layer{i}"
        for k, (M, N, K) in shapes.items():
            costs[f"{L}.{k}"] = {p: entry(f"{L}.{k}", p, linear_memory_bytes(p, M, N, K))
                                 for p in (INT8, FP16, FP32)}
        costs[f"{L}.attn"] = fixed(f"{L}.attn", T * 3 * H * 2 + T * H * 2)
        costs[f"{L}.ln1"] = fixed(f"{L}.ln1", T * H * 4 * 2 + 2 * H * 4 * 4)
        costs[f"{L}.ln2"] = fixed(f"{L}.ln2", T * H * 4 * 2 + 2 * H * 4 * 4)
        g16 = entry(f"{L}.gelu", FP16, T * Fh * 2 * 2)
        g32 = min((entry(f"{L}.gelu", p, T * Fh * 4 * 2) for p in (INT8, FP32)),
                  key=lambda e: e["pure_cost_ns"])
        costs[f"{L}.gelu"] = {FP16: g16, FP32: g32}
    return costs


def measure_fused_cast_samples(cfg: BertConfig, rows=(512, 1024, 2048, 4096, 8192)):
    """Cast samples of the fused implementation, where a conversion is not a
    kernel of its own but part of its producer or consumer:

    * FP32 -> FP16 (float_to_float): the producing LayerNorm also writes FP16(y)
      -- the extra time of ``layernorm_fwd_ex`` with the copy over without;
    * FP16 -> FP32: an FP32 LayerNorm reads the FP16 producer directly -- the extra
      time of the FP16 input over an FP32 one (clamped at 1 ns);
    * FP32 / FP16 -> INT8 (quantize_fixed): the single-pass quantizer with the
      absmax the producer already wrote (``quantize_act``);
    * INT8 -> FP32 (dequantize_fixed): folded into the GEMM epilogues (the INT8
      GEMM and the wgrad write FP32) -- the extra time of the FP32 over the FP16
      epilogue of the INT8 GEMM, clamped at 1 ns.
    Each is timed back-to-back inside a CUDA graph, as the train step runs it.
    """
    H = cfg.hidden
    samples = []
    g = torch.rand(H, device="cuda") + 0.5
    be = torch.randn(H, device="cuda")
    w8 = torch.randint(-127, 128, (H, H), dtype=torch.int8, device="cuda")
    sw = torch.rand(H, device="cuda") * 0.01
    for r in rows:
        n = r * H
        a = torch.randn(r, H, device="cuda")
        b32 = torch.randn(r, H, device="cuda")
        b16 = b32.half()
        am = torch.tensor([4.0], device="cuda")
        x8 = torch.randint(-127, 128, (r, H), dtype=torch.int8, device="cuda")
        sa = torch.tensor([0.01], device="cuda")
        def t(fn):  # best of 5 graph timings: the marginal costs are differences of near-equal times
            return min(_graph_time_ns(fn) for _ in range(5))
        plain = t(lambda: ops.layernorm_fwd_ex(a, b32, g, be, 1e-12, False, False))
        with16 = t(lambda: ops.layernorm_fwd_ex(a, b32, g, be, 1e-12, True, False))
        in16 = t(lambda: ops.layernorm_fwd_ex(a, b16, g, be, 1e-12, False, False))
        q32 = t(lambda: ops.quantize_act(a, am))
        q16 = t(lambda: ops.quantize_act(b16, am))
        e32 = t(lambda: ops.gemm_s8_ex(x8, w8, sa, sw, None, out_dtype=torch.float32))
        e16 = t(lambda: ops.gemm_s8_ex(x8, w8, sa, sw, None, out_dtype=torch.float16))
        for src, dst, scheme, ns in ((FP32, FP16, "float_to_float", with16 - plain),
                                     (FP16, FP32, "float_to_float", in16 - plain),
                                     (FP32, INT8, "quantize_fixed", q32),
                                     (FP16, INT8, "quantize_fixed", q16),
                                     (INT8, FP32, "dequantize_fixed", e32 - e16)):
            samples.append({"src": src, "dst": dst, "scheme": scheme, "numel": n,
                            "measured_ns": max(1, int(ns))})
    return samples


def fit_cast(samples: list) -> tuple[float, float]:
    """(a, b) of the reference's cast model for one key: OLS a*numel + b, a < 0 ->
    flat mean, b < 0 -> refit through the origin (profile.cpp:33-83)."""
    xs = [float(x) for x, _ in samples]
    ys = [float(y) for _, y in samples]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    a = sxy / sxx
    b = my - a * mx
    if a < 0:
        a, b = 0.0, my
    if b < 0:
        sxx0 = sum(x * x for x in xs)
        sxy0 = sum(x * y for x, y in zip(xs, ys))
        a, b = (max(0.0, sxy0 / sxx0) if sxx0 > 0 else 0.0), 0.0
    return a, b


def net_weight_casts(cfg: BertConfig, costs: dict, cast_samples: list) -> dict:
    """The fused step converts weights inside the optimizer (w16 / wq emitted with
    the update), and that time is already in each op's optimizer share.  The
    reference's cost mapper adds a weight cast FP32 -> k on every weighted op's
    forward event (cost_mapper.cpp:42-43), so the entry is stored net of it: the
    op's forward share is reduced by exactly the cast model's prediction."""
    keys = {}
    for smp in cast_samples:
        keys.setdefault((smp["src"], smp["dst"]), []).append((smp["numel"], smp["measured_ns"]))
    numel = _param_numel(cfg)
    for op, per_p in costs.items():
        w = numel.get(op, (0, 0))[0]
        if not w:
            continue
        for p, e in per_p.items():
            if p == FP32 or (FP32, p) not in keys:
                continue
            a, b = fit_cast(keys[(FP32, p)])
            wc = int(math.floor(a * w + b + 0.5))  # llround of a nonnegative value (profile.cpp:95)
            fwd = e["pure_cost_ns"] * e["fwd_fraction"]
            cut = min(wc, int(fwd))
            tot = max(1, e["pure_cost_ns"] - cut)
            e["pure_cost_ns"] = tot
            e["fwd_fraction"] = max(0.0, min(1.0, (fwd - cut) / tot))
    return costs


def profile_bert_fused(cfg: BertConfig, batch: int, stat_steps: int = 3, infer_cap_bytes: int | None = None,
                       reps: int = 5, with_comm: bool = True) -> dict:
    """The bundle of the layer-fused implementation (the one the train step runs),
    with the measured gradient-exchange slots (``comm``) of every device."""
    model = BertEncoderStack(cfg).cuda()
    model.apply_plan({})
    stats = collect_tensor_stats(model, batch, stat_steps)
    del model
    casts = measure_fused_cast_samples(cfg)
    costs = net_weight_casts(cfg, measure_fused_costs(cfg, batch, reps), casts)
    graph = bert_graph(cfg, batch)
    cap = infer_cap_bytes or default_cap(graph, costs)
    devices = [{"id": "trainer", "is_inference": False, "mem_capacity_bytes": 183_000_000_000},
               {"id": "infer", "is_inference": True, "mem_capacity_bytes": max(cap, 1)}]
    return build_bundle(graph, costs, casts, stats, devices)


# ----------------------------------------------------------------------------- comm
def _timed_step(cfg: BertConfig, batch: int, plan: dict, comm=None, world: int = 1):
    """An eager single-stream TrainStep (wgrad on the main stream) whose gradient
    buckets go through ``comm`` (an ops.Communicator; a 1-rank one on a single
    GPU) with CommSlot timing on."""
    from .ops import Communicator
    from .train_step import TrainStep
    if comm is None:
        comm = Communicator(1, 0)
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(plan)
    st = TrainStep(m, batch=batch, world=world, graph=False, overlap_wgrad=False, comm=comm)
    st.tokens.random_(0, cfg.vocab)
    st.grads.timing = True
    for _ in range(3):
        st()
    torch.cuda.synchronize()
    return st, comm


def measure_comm_slots(cfg: BertConfig, batch: int, plan: dict | None = None, comm=None,
                       world: int = 1, reps: int = 5) -> list[dict]:
    """CommSlots (profile.hpp:118-129) of the train step's bucketed gradient
    exchange, measured through the C ABI's NCCL all-reduce: per bucket the
    earliest ready offset from the step start, the all-reduce's device time and
    the bucket's bytes; median over ``reps`` eager steps.  The replayer attaches
    slots to backward events on the FP32 timeline (cost_mapper.cpp:55-90), so the
    default plan is all-FP32 (the assignment the reference profiles at)."""
    st, comm = _timed_step(cfg, batch, plan or {}, comm, world)
    runs = []
    for _ in range(reps):
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000_000)  # enqueue the whole step before it runs
        st()
        runs.append(st.grads.comm_slots())
    med = statistics.median
    out = []
    for k in range(len(runs[0])):
        out.append({"earliest_ready_offset_ns": int(med(r[k]["earliest_ready_offset_ns"] for r in runs)),
                    "duration_ns": max(1, int(med(r[k]["duration_ns"] for r in runs))),
                    "bucket_bytes": runs[0][k]["bucket_bytes"]})
    measure_comm_slots.last_world = comm.world
    return out


def measured_op_trace(cfg: BertConfig, batch: int, plan: dict, device_id: str = "b200", comm=None,
                      world: int = 1) -> dict:
    """One measured eager step as a Chrome trace in the reference replayer's
    format (replayer.cpp:126-148): event name = the replayer's event id
    ("fwd:<op>", "bwd:<op>", "optimizer"; the input conversion of an op is part of
    its "fwd:" event, as the cost mapper charges fwd_cast to it,
    cost_mapper.cpp:34-43), pid = device, tid 0 = compute, tid 1 =
    "allreduce:<n>" slots.  Regions come from the fused step's operator marks
    (fused.REGION); "zero_grad" (the flat-gradient memset) has no replayer
    counterpart."""
    from . import fused
    st, comm = _timed_step(cfg, batch, plan, comm, world)
    marks = []

    def hook(kind, op):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((kind, op, e))

    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)
    fused.REGION = hook
    try:
        st()
    finally:
        fused.REGION = None
    torch.cuda.synchronize()
    t0 = st.grads.t0
    names = {"fwd": "fwd:", "cast": "fwd:", "bwd": "bwd:"}
    events = []
    for (k, o, e0), (_, _, e1) in zip(marks, marks[1:]):
        if k == "opt":
            name = "optimizer" if o == "optimizer" else "zero_grad"
        else:
            name = names[k] + o
        s_us, e_us = t0.elapsed_time(e0) * 1e3, t0.elapsed_time(e1) * 1e3
        if events and events[-1]["name"] == name and events[-1]["tid"] == 0:
            events[-1]["dur"] = e_us - events[-1]["ts"]  # cast + fwd of one op: one event
            continue
        events.append({"name": name, "ph": "X", "ts": s_us, "dur": e_us - s_us, "pid": device_id, "tid": 0})
    for n, (i, r_main, r_side, e_s, e_e, nbytes) in enumerate(sorted(st.grads._slot_events, key=lambda t: t[0])):
        s_us, e_us = t0.elapsed_time(e_s) * 1e3, t0.elapsed_time(e_e) * 1e3
        events.append({"name": f"allreduce:{n + 1}", "ph": "X", "ts": s_us, "dur": e_us - s_us,
                       "pid": device_id, "tid": 1, "args": {"bucket_bytes": nbytes}})
    return {"traceEvents": events, "displayTimeUnit": "ms"}


# ----------------------------------------------------------------------------- casts
def measure_cast_samples(sizes=(1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24), reps: int = 10):
    """Measured latencies for every key required_cast_keys asks for (profile.cpp:212-228)."""
    samples = []
    for n in sizes:
        x32 = torch.randn(n, device="cuda")
        x16 = x32.half()
        q = torch.randint(-127, 128, (n,), dtype=torch.int8, device="cuda")
        sc = torch.tensor([0.01], device="cuda")
        cases = [
            (FP32, FP16, "float_to_float", lambda: ops.cast(x32, torch.float16)),
            (FP16, FP32, "float_to_float", lambda: ops.cast(x16, torch.float32)),
            (FP32, INT8, "quantize_fixed", lambda: ops.quantize_per_tensor(x32.view(1, -1))),
            (FP16, INT8, "quantize_fixed", lambda: ops.quantize_per_tensor(x16.view(1, -1))),
            (INT8, FP32, "dequantize_fixed", lambda: ops.dequantize_per_tensor(q, sc)),
        ]
        for src, dst, scheme, fn in cases:
            samples.append({"src": src, "dst": dst, "scheme": scheme, "numel": n,
                            "measured_ns": _time_ns(fn, reps)})
    return samples


# ----------------------------------------------------------------------------- stats
class StatsRecorder:
    """Collects device statistics per op for one step; ``snapshot()`` turns them
    into the OpStats JSON fields (profile.hpp:95-108)."""

    def __init__(self):
        self.cur: dict[str, dict[str, torch.Tensor]] = {}

    def record(self, name: str, kind: str, st: torch.Tensor) -> None:
        self.cur.setdefault(name, {})[kind] = st

    def snapshot(self) -> dict:
        snap = {}
        for name, d in self.cur.items():
            if not {"act", "w", "grad"} <= set(d):
                continue
            a, w, g = (d[k].tolist() for k in ("act", "w", "grad"))
            # [||x||^2, absmax, q = absmax/127, e = floor(log2 absmax), numel]
            snap[name] = {"norm_w_sq": w[0], "norm_act_sq": a[0], "norm_grad_act_sq": g[0],
                          "d_act": a[4], "d_w": w[4], "d_grad": g[4],
                          "q_act": a[2], "q_w": w[2], "e_act": a[3], "e_w": w[3], "e_grad": g[3]}
        self.cur = {}
        return snap


def collect_tensor_stats(model: BertEncoderStack, batch: int, steps: int, seed: int = 0):
    """Run `steps` eager training steps (SGD, the plan currently applied) and record
    one statistics snapshot per step."""
    cfg = model.cfg
    g = torch.Generator().manual_seed(seed)
    opt = torch.optim.SGD(model.parameters(), lr=1e-4)
    rec = StatsRecorder()
    snaps = []
    qlinear.STATS_RECORDER = rec
    try:
        for _ in range(steps):
            tok = torch.randint(0, cfg.vocab, (batch, cfg.seq), generator=g).cuda()
            lab = torch.randint(0, cfg.num_labels, (batch,), generator=g).cuda()
            opt.zero_grad(set_to_none=True)
            model(tok, lab).backward()
            opt.step()
            snaps.append(rec.snapshot())
    finally:
        qlinear.STATS_RECORDER = None
    return snaps


# ----------------------------------------------------------------------------- bundle
def build_bundle(graph: dict, op_costs: dict, cast_samples: list, tensor_stats: list,
                 devices: list, comm: dict | None = None) -> dict:
    b = {"schema_version": 1, "graph": graph, "op_costs": op_costs,
         "cast_samples": cast_samples, "tensor_stats": tensor_stats, "devices": devices}
    if comm:
        b["comm"] = comm
    return b


def default_cap(graph: dict, costs: dict, frac: float = 0.75) -> int:
    """A binding but feasible memory cap for the inference device: halfway between
    the all-lowest-precision and the all-FP32 footprint (the paper's cluster B caps
    inference GPUs at 30% of their memory; here the cap is set relative
    to this model's own footprint so the allocator has a real trade-off)."""
    full = sum(costs[n["id"]][FP32]["memory_bytes"] if FP32 in costs[n["id"]] else
               max(v["memory_bytes"] for v in costs[n["id"]].values()) for n in graph["nodes"])
    # lowest footprint: adjustable ops at their cheapest precision; dependent ops
    # may be forced up by the cascade (INT8 producers emit FP32), so take their max
    low = sum((min if n["kind"] == "adjustable" else max)(v["memory_bytes"]
                                                          for v in costs[n["id"]].values())
              for n in graph["nodes"])
    return int(low + frac * (full - low))


def profile_bert(cfg: BertConfig, batch: int, stat_steps: int = 3, infer_cap_bytes: int | None = None,
                 reps: int = 10) -> dict:
    """Measure everything on the current device and return the bundle dict."""
    model = BertEncoderStack(cfg).cuda()
    model.apply_plan({})  # statistics are profiled at FP32 (the reference's assignment)
    stats = collect_tensor_stats(model, batch, stat_steps)
    del model
    costs = measure_op_costs(cfg, batch, reps)
    casts = measure_cast_samples(reps=reps)
    graph = bert_graph(cfg, batch)
    cap = infer_cap_bytes or default_cap(graph, costs)
    devices = [{"id": "trainer", "is_inference": False, "mem_capacity_bytes": 183_000_000_000},
               {"id": "infer", "is_inference": True, "mem_capacity_bytes": max(cap, 1)}]
    return build_bundle(graph, costs, casts, stats, devices)


def main(argv=None):
    import argparse
    ap = argparse.ArgumentParser(description="profile the B200 hot path into a QSync bundle")
    ap.add_argument("--out", required=True)
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--stat-steps", type=int, default=3)
    args = ap.parse_args(argv)
    cfg = BertConfig(layers=args.layers)
    bundle = profile_bert(cfg, args.batch, args.stat_steps)
    with open(args.out, "w") as f:
        json.dump(bundle, f, indent=1)
    print(f"wrote {args.out}")


if __name__ == "__main__":
    main()
