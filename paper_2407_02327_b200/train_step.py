"""The QSync data-parallel training step on B200 (BERT-base encoder stack).

One process per GPU.  Each rank runs its OWN per-layer precision plan (the
allocator's ``PrecisionPlan.per_device`` entry, graph.hpp:132-134): every
adjustable Linear executes the INT8 / FP16 / FP32 kernel the plan names; ops a
plan omits run FP32 (replayer.cpp:86-94, pinned by test_replayer.cpp:209-214).
Gradients are FP32 on every rank whatever its plan (INT8 wgrad is emitted FP32,
cost_mapper.cpp:48-50), so the DP all-reduce layout is rank-independent.

Gradient buckets are reduced in reverse-topological (backward) order
(cost_mapper.cpp:115-126); bucket n is issued once every rank produced it and
after bucket n-1 (one NCCL stream, in-order) -- the Eq. 6 slot semantics of
replayer.cpp:48-62; the optimizer runs after the last bucket (:64-73).

Glue ops around the planned Linears (embeddings, LayerNorm, GELU, attention
core softmax(QK^T)V -- which QSync leaves in floating point, PAPER.md:399 --
and the optimizer) are PyTorch plumbing; the hot path is the Linear kernels.
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import qlinear as _ql
from .glue import AddLayerNorm, attention, gelu
from .qlinear import EXTENDED, FP16, FP32, INT8, QLinear, cast


@dataclass
class BertConfig:
    vocab: int = 30522
    hidden: int = 768
    layers: int = 12
    heads: int = 12
    ffn: int = 3072
    max_pos: int = 512
    type_vocab: int = 2
    num_labels: int = 2
    seq: int = 128


def adjustable_ops(cfg: BertConfig) -> list[str]:
    """Names of the planned (adjustable) operators, in forward topological order."""
    names = []
    for i in range(cfg.layers):
        names += [f"layer{i}.qkv", f"layer{i}.o", f"layer{i}.ff1", f"layer{i}.ff2"]
    names.append("pooler")
    return names


def mixed_plan(cfg: BertConfig) -> dict[str, str]:
    """Default heterogeneous plan of the bench: even layers INT8, odd layers FP16
    (the paper's 'Half-BertLayer1,3,5' / 'INT-Linears' pattern),
    the pooler FP32."""
    plan = {}
    for i in range(cfg.layers):
        p = INT8 if i % 2 == 0 else FP16
        for op in ("qkv", "o", "ff1", "ff2"):
            plan[f"layer{i}.{op}"] = p
    plan["pooler"] = FP32
    return plan


def uniform_plan(cfg: BertConfig, precision: str) -> dict[str, str]:
    return {name: precision for name in adjustable_ops(cfg)}


def load_plan(path: str, device_id: str) -> dict[str, str]:
    """Read a plan file as the reference's replay accepts it (cli.cpp:38-51): a
    bare {"per_device": {dev: {op: PREC}}} mapping or a full plan report whose
    "devices" object holds the mapping."""
    with open(path) as f:
        j = json.load(f)
    table = j.get("per_device") or j.get("devices") or {}
    if device_id not in table:
        raise KeyError(f"reference: plan has no device \"{device_id}\"")
    plan = dict(table[device_id])
    for op, p in plan.items():
        if p not in EXTENDED:  # the reference's INT8/FP16/FP32 plus this ladder's FP8 / BF16
            raise ValueError(f"validation: unknown precision \"{p}\"")
    return plan


class EncoderLayer(torch.nn.Module):
    def __init__(self, cfg: BertConfig, i: int):
        super().__init__()
        h = cfg.hidden
        self.cfg = cfg
        self.qkv = QLinear(h, 3 * h, f"layer{i}.qkv")
        self.o = QLinear(h, h, f"layer{i}.o")
        self.ff1 = QLinear(h, cfg.ffn, f"layer{i}.ff1")
        self.ff2 = QLinear(cfg.ffn, h, f"layer{i}.ff2")
        self.ln1 = AddLayerNorm(h, eps=1e-12)
        self.ln2 = AddLayerNorm(h, eps=1e-12)

    def forward(self, x):  # x [B, S, H] fp32 residual stream
        B, S, H = x.shape
        nh = self.cfg.heads
        qkv = self.qkv(x)  # [B, S, 3H] fp32 (INT8) / fp16 (FP16)
        qkv = cast(qkv, torch.float16)
        # Attention core stays floating point; packed QKV in,
        # packed dQKV out -- no permute/stack copies around it.
        a = attention(qkv.view(B, S, 3, nh, H // nh))  # [B, S, nh, d]
        a = a.reshape(B, S, H)
        x = self.ln1(x, _ln_operand(self.o(a)))        # fused residual add (FP32 or FP16 operand)
        f = gelu(self.ff1(x))
        x = self.ln2(x, _ln_operand(self.ff2(f)))
        return x


def _ln_operand(y):
    """The residual LayerNorm reads an FP32 or FP16 operand; a BF16 op's output
    is widened to FP32 (exact) on the way in."""
    return cast(y, torch.float32) if y.dtype == torch.bfloat16 else y


def _fusable(layer: EncoderLayer) -> bool:
    """The layer-fused path (fused.py) covers the reference ladder INT8 / FP16 /
    FP32; a layer with a BF16 or FP8 op runs the per-operator QLinear path."""
    return all(m.precision in (INT8, FP16, FP32) for m in (layer.qkv, layer.o, layer.ff1, layer.ff2))


# Fused path: pooler + classifier + CE on csrc/head.cu (A/B: tools/ab_step.py head=1,0).
HEAD_KERNELS = True
# Gradient-buffer reset on the wgrad side stream, overlapping the forward pass
# (A/B: tools/ab_step.py zero=1,0).
ZERO_OVERLAP = True


class BertEncoderStack(torch.nn.Module):
    """BERT-base: embeddings + 12 encoder layers + pooler + classifier."""

    def __init__(self, cfg: BertConfig):
        super().__init__()
        self.cfg = cfg
        self.word = torch.nn.Embedding(cfg.vocab, cfg.hidden)
        self.pos = torch.nn.Embedding(cfg.max_pos, cfg.hidden)
        self.typ = torch.nn.Embedding(cfg.type_vocab, cfg.hidden)
        self.ln = AddLayerNorm(cfg.hidden, eps=1e-12)
        self.layers = torch.nn.ModuleList([EncoderLayer(cfg, i) for i in range(cfg.layers)])
        self.pooler = QLinear(cfg.hidden, cfg.hidden, "pooler")
        # Layer-fused execution (fused.py); the per-operator path stays for
        # profiling (per-op statistics) and as the parity reference.
        self.fused = False
        self.cls = torch.nn.Linear(cfg.hidden, cfg.num_labels)
        for emb in (self.word, self.pos, self.typ):
            torch.nn.init.normal_(emb.weight, std=0.02)

    def qlinears(self) -> dict[str, QLinear]:
        return {m.name: m for m in self.modules() if isinstance(m, QLinear)}

    def apply_plan(self, plan: dict[str, str]) -> None:
        """Operators the plan omits run FP32 (replayer.cpp:86-94)."""
        for name, m in self.qlinears().items():
            m.precision = plan.get(name, FP32)

    def forward(self, tokens, labels):
        B, S = tokens.shape
        if self.fused:
            from .fused import fused_layer
            from .glue import embed_layernorm
            fusable = [_fusable(layer) for layer in self.layers]
            p0 = self.layers[0].qkv.precision if len(self.layers) and fusable[0] else None
            x, aux = embed_layernorm(tokens, self.word, self.pos, self.typ, self.ln,
                                     want_f16=p0 == FP16, want_quant=p0 == INT8)
            n = len(self.layers)
            for i, layer in enumerate(self.layers):
                if not fusable[i]:  # a BF16 / FP8 op: the per-operator layer
                    x, aux = layer(x), None
                    continue
                nxt = self.layers[i + 1].qkv.precision if i + 1 < n and fusable[i + 1] else None
                x, aux = fused_layer(layer, x, aux, nxt)
        else:
            pos = torch.arange(S, device=tokens.device)
            x = self.word(tokens) + self.pos(pos)[None] + self.typ.weight[0][None, None]
            x = self.ln(x)
            for layer in self.layers:
                x = layer(x)
        if self.fused:
            from .fused import _mark
            if HEAD_KERNELS and self.pooler.precision == FP32 and x.dtype == torch.float32 and x.is_cuda:
                # pooler + classifier + CE on the library's head kernels (csrc/head.cu);
                # profiling charges the head to "loss" (the pooler op is costed from
                # its own kernels, profiler.measure_linear)
                from .glue import cls_head
                _mark("fwd", "loss")
                return cls_head(x, self.pooler, self.cls, labels)
            _mark("fwd", "pooler")
        pooled = torch.tanh(cast(self.pooler(x[:, 0].contiguous()), torch.float32))
        if self.fused:
            _mark("fwd", "loss")
        logits = self.cls(pooled)
        loss = F.cross_entropy(logits, labels)
        if self.fused and loss.requires_grad:
            from . import fused as _fz
            if _fz.REGION is not None:  # operator regions of the backward head (profiling only)
                loss.register_hook(lambda g: (_fz._mark("bwd", "loss"), g)[1])
                pooled.register_hook(lambda g: (_fz._mark("bwd", "pooler"), g)[1])
        return loss


def linear_flops_per_step(cfg: BertConfig, tokens: int) -> float:
    """fwd + dgrad + wgrad of the 48 encoder Linears."""
    h, f = cfg.hidden, cfg.ffn
    per_layer = 2 * tokens * (h * 3 * h + h * h + h * f + f * h)
    return 3.0 * per_layer * cfg.layers


# --------------------------------------------------------------------------- DP
class FlatGrads:
    """All FP32 gradients in ONE flat buffer laid out in backward order (last
    layer first), so that (a) each parameter's ``grad`` and ``main_grad`` are
    views of it -- QLinear wgrad/bias-grad kernels accumulate straight into their
    slice and the optimizer reads it in place; (b) zeroing is one memset; (c) DP
    buckets are contiguous slices, all-reduced without packing copies."""

    def __init__(self, params: list[torch.nn.Parameter], bucket_bytes: int = 32 << 20):
        self.params = [p for p in params if p.requires_grad]
        order = list(reversed(self.params))
        # Every slot starts on a 64-byte boundary: the GEMM epilogue's TMA
        # reduce-add (and vector paths) need 16-byte aligned rows.
        align = 16
        slots, total = [], 0
        for p in order:
            slots.append(total)
            total += (p.numel() + align - 1) // align * align
        dev = order[0].device
        self.flat = torch.zeros(total, device=dev, dtype=torch.float32)
        self.buckets: list[tuple[int, int]] = []  # (start, end) element ranges
        off = 0
        b_start = 0
        for p, start in zip(order, slots):
            n = p.numel()
            view = self.flat[start:start + n].view_as(p)
            p.main_grad = view
            p.grad = view
            off = start + (n + align - 1) // align * align
            if (off - b_start) * 4 >= bucket_bytes:
                self.buckets.append((b_start, off))
                b_start = off
        if off > b_start:
            self.buckets.append((b_start, off))

        # Bucket membership for the overlapped all-reduce: params never straddle.
        self.bucket_of: dict[int, int] = {}
        self._members = [0] * len(self.buckets)
        self.bucket_params: list[list] = [[] for _ in self.buckets]
        for p, start in zip(order, slots):
            b = next(i for i, (a, e) in enumerate(self.buckets) if a <= start < e)
            self.bucket_of[id(p)] = b
            self._members[b] += 1
            self.bucket_params[b].append(p)
        self._on_final = None
        self._active = False
        self._pending: list[int] = []
        self._next = 0
        self._world = 1
        self._side = None
        self.comm_stream = None
        self.issue_log: list[tuple[int, int]] = []  # (bucket, pending params at issue) -- tests
        # The C1 exchange: an ops.Communicator (NCCL through the C ABI) when the
        # flat buffer lives on a GPU; None -> torch.distributed (the gloo tests).
        self.comm = None
        # CommSlot measurement (profile.hpp:118-129): with ``timing`` on (eager
        # steps only -- no events inside a CUDA-graph capture) every bucket gets
        # ready / start / end events; ``t0`` is the step-start event the ready
        # offsets are measured from (the replayer's clock starts at the first
        # forward event, cost_mapper.cpp:60-70).
        self.timing = False
        self.t0 = None
        self._slot_events: list[tuple] = []

    def zero(self) -> None:
        if self.flat.is_cuda:
            from . import ops
            ops.zero_(self.flat)  # the library's PDL kernel, not a framework memset
        else:  # host-logic tests (gloo, world 2, CPU)
            self.flat.zero_()

    # ---- overlapped, in-order bucket all-reduce (Eq. 6 slots, replayer.cpp:48-62)
    def begin(self, world: int, side_stream=None, on_final=None) -> None:
        """Start a backward pass: bucket n is all-reduced as soon as all of its
        parameters are final AND bucket n-1 has been issued -- one comm stream,
        in order, identical on every rank whatever its precision plan.
        ``on_final(n)`` (optional) runs on the comm stream right after bucket n is
        reduced (or, on one rank, as soon as it is final): the optimizer of that
        bucket, overlapping the rest of the backward."""
        self._world = world
        self._on_final = on_final
        self._active = world > 1 or on_final is not None or self.comm is not None
        self._pending = list(self._members)
        self._next = 0
        self._side = side_stream
        self.issue_log = []
        self._slot_events = []
        if self.flat.is_cuda and self._active and self.comm_stream is None:
            self.comm_stream = torch.cuda.Stream(priority=-1)

    def params_ready(self, params) -> None:
        """The gradients of ``params`` are final (their producing kernels are
        enqueued on the current stream and, for wgrad, the side stream)."""
        if not self._active:
            return
        for p in params:
            b = self.bucket_of.get(id(p))
            if b is not None and self._pending[b] > 0:
                self._pending[b] -= 1
        self._issue(force=False)

    def finish(self) -> None:
        """End of backward: issue every remaining bucket, then make the current
        stream (the optimizer) wait for the last one (replayer.cpp:64-73)."""
        if not self._active:
            return
        self._issue(force=True)
        if self.comm_stream is not None:
            torch.cuda.current_stream().wait_stream(self.comm_stream)

    def _issue(self, force: bool) -> None:
        import torch.distributed as dist
        ready = []
        while self._next < len(self.buckets) and (force or self._pending[self._next] == 0):
            ready.append(self._next)
            self.issue_log.append((self._next, self._pending[self._next]))
            self._next += 1
        if not ready:
            return
        world = self._world
        timing = self.timing and self.flat.is_cuda and not torch.cuda.is_current_stream_capturing()
        if timing:
            # Ready = the producing streams reached this point (main and wgrad side stream).
            r_main = torch.cuda.Event(enable_timing=True)
            r_main.record()
            r_side = None
            if self._side is not None:
                r_side = torch.cuda.Event(enable_timing=True)
                r_side.record(self._side)
        if self.comm_stream is not None:
            self.comm_stream.wait_stream(torch.cuda.current_stream())
            if self._side is not None:
                self.comm_stream.wait_stream(self._side)
            ctx = torch.cuda.stream(self.comm_stream)
        else:
            import contextlib
            ctx = contextlib.nullcontext()
        with ctx:
            for i in ready:
                a, b = self.buckets[i]
                chunk = self.flat[a:b]
                if timing:
                    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e_s.record()
                if self.comm is not None:
                    self.comm.allreduce_bucket(chunk, average=True)  # C ABI -> ncclAllReduce(ncclAvg)
                elif world > 1:
                    dist.all_reduce(chunk)
                    chunk.div_(world)
                if timing:
                    e_e.record()
                    self._slot_events.append((i, r_main, r_side, e_s, e_e, (b - a) * 4))
                if self._on_final is not None:
                    self._on_final(i)

    def comm_slots(self) -> list[dict]:
        """The last timed backward's buckets as CommSlot records
        (profile.hpp:118-129; schema profile.cpp:385-403), in slot order:
        earliest_ready_offset_ns = ready - step start, duration_ns = the
        all-reduce's device time, bucket_bytes = the FP32 bucket size."""
        if not self._slot_events:
            return []
        torch.cuda.synchronize()
        out = []
        for i, r_main, r_side, e_s, e_e, nbytes in sorted(self._slot_events, key=lambda t: t[0]):
            ready_ms = self.t0.elapsed_time(r_main) if self.t0 is not None else 0.0
            if r_side is not None and self.t0 is not None:
                ready_ms = max(ready_ms, self.t0.elapsed_time(r_side))
            out.append({"earliest_ready_offset_ns": max(0, int(round(ready_ms * 1e6))),
                        "duration_ns": max(1, int(round(e_s.elapsed_time(e_e) * 1e6))),
                        "bucket_bytes": int(nbytes)})
        return out

    def allreduce(self, world: int) -> None:
        """Non-overlapped form: every bucket in order after the backward."""
        if world <= 1:
            return
        self.begin(world)
        self.finish()


class TrainStep:
    """One synchronous DP step: fwd + bwd (planned kernels) + bucketed all-reduce
    + AdamW on FP32 master weights.  Optionally captured into a CUDA graph."""

    def __init__(self, model: BertEncoderStack, batch: int, world: int = 1, lr: float = 1e-4,
                 graph: bool = True, overlap_wgrad: bool = True, fused: bool = True,
                 overlap_opt: bool | None = None, comm="auto"):
        self.model = model
        self.world = world
        cfg = model.cfg
        dev = next(model.parameters()).device
        self.tokens = torch.zeros((batch, cfg.seq), dtype=torch.long, device=dev)
        self.labels = torch.zeros((batch,), dtype=torch.long, device=dev)
        # d(loss)/d(loss) = 1, allocated once: backward() would fill a new one per step
        self._one = torch.ones((), dtype=torch.float32, device=dev)
        self.params = [p for p in model.parameters() if p.requires_grad]
        self.grads = FlatGrads(self.params)
        # C1: the gradient buckets go through this library's NCCL entry points
        # (qsync_allreduce_bucket); "auto" = one communicator per rank when DP runs
        # on GPUs under an NCCL process group.  Pass an ops.Communicator (e.g. a 1-rank one) to time the
        # exchange on a single GPU, or None for torch.distributed (CPU / gloo).
        if comm == "auto":
            comm = None
            import torch.distributed as dist
            if world > 1 and dev.type == "cuda" and dist.get_backend() == "nccl":
                from .ops import Communicator
                comm = Communicator(world, dist.get_rank())
        self.grads.comm = comm
        self.fused = fused
        model.fused = fused
        if fused:
            # One kernel: AdamW + the planned Linears' weight copies for the next step.
            from .fused import FusedAdamW
            self.opt = FusedAdamW(self.params, lr=lr)
            self.opt.attach(model.qlinears().values())
        else:
            self.opt = torch.optim.AdamW(self.params, lr=lr, fused=True, capturable=graph)
        self.use_graph = graph
        self.graph = None
        self.loss = None
        # Stream priorities: the critical-path chain (main stream, captured at
        # high priority) wins free SMs over the wgrad GEMMs, which only feed the
        # all-reduce / optimizer and fill the gaps.
        self.wgrad_stream = torch.cuda.Stream(priority=0) if overlap_wgrad else None
        if overlap_wgrad and fused:
            # Side-stream wgrad GEMM grid cap (persistent kernels).  A 2/3-of-SMs
            # cap once paid (5.55 -> 5.25 ms); with 192-wide tiles and the FP16
            # wgrad operands written by the quantizer the uncapped grid is best
            # (tools/ab_step.py wgrad_cap=0,98: 5.09 ms uncapped vs 5.20).
            from . import fused as _fz
            _fz.WGRAD_CTAS = 0
        # Bucket-wise optimizer (DP): each bucket's AdamW runs on the comm stream
        # right after its all-reduce, overlapping the remaining buckets' reductions
        # and the rest of the backward.  On one GPU it only contends with the
        # backward for HBM (tools/ab_step.py overlap_opt=0,1: 5.01 vs 4.97 ms), so it is off there.
        self.overlap_opt = fused and (world > 1 if overlap_opt is None else overlap_opt)
        self._hooked = (world > 1 or self.overlap_opt or comm is not None) and fused
        if self._hooked:
            for m in (model.pooler, model.cls):
                for prm in m.parameters():
                    prm.register_post_accumulate_grad_hook(lambda t: self.grads.params_ready([t]))

    def apply_plan(self, plan: dict[str, str]) -> None:
        """Switch this rank's plan (re-capture afterwards when graphed)."""
        self.model.apply_plan(plan)
        if self.fused:
            self.opt.attach(self.model.qlinears().values())

    def _body(self):
        if self.grads.timing and not torch.cuda.is_current_stream_capturing():
            self.grads.t0 = torch.cuda.Event(enable_timing=True)
            self.grads.t0.record()
        if self.fused:
            from .fused import _mark
            _mark("opt", "zero")
        overlap_zero = ZERO_OVERLAP and self.wgrad_stream is not None and self.grads.timing is False
        if overlap_zero:
            # reset the gradient buffer on the side stream, under the forward pass
            # (which writes no gradient); joined before the backward starts
            self.wgrad_stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.wgrad_stream):
                self.grads.zero()
        else:
            self.grads.zero()
        loss = self.model(self.tokens, self.labels)
        _ql.WGRAD_STREAM = self.wgrad_stream
        if self.wgrad_stream is not None:
            if overlap_zero:
                torch.cuda.current_stream().wait_stream(self.wgrad_stream)  # gradients zeroed
            self.wgrad_stream.wait_stream(torch.cuda.current_stream())  # after the zeroing
        # Buckets are all-reduced while the backward continues: a fused layer
        # reports its parameters final when its backward is enqueued, autograd
        # parameters (pooler, classifier) through their post-accumulate hooks.
        self.grads.begin(self.world, self.wgrad_stream,
                         on_final=self._opt_bucket if self.overlap_opt else None)
        _ql.GRAD_READY = self.grads.params_ready if self._hooked else None
        try:
            loss.backward(self._one)
        finally:
            _ql.WGRAD_STREAM = None
            _ql.GRAD_READY = None
        if self.wgrad_stream is not None:
            torch.cuda.current_stream().wait_stream(self.wgrad_stream)  # join before the last buckets
        self.grads.finish()
        if self.fused:
            from .fused import _mark
            _mark("opt", "optimizer")
        if self.overlap_opt:
            self.opt.advance()
        else:
            self.opt.step()
        if self.fused:
            _mark("end", "")
        return loss.detach()

    def _opt_bucket(self, i: int) -> None:
        r0, r1 = self.opt.rows_of(self.grads.bucket_params[i])
        self.opt.step_range(r0, r1)

    def capture(self, warmup: int = 3) -> None:
        s = torch.cuda.Stream(priority=-1)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream().wait_stream(s)
        if self.use_graph:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.loss = self._body()

    def __call__(self):
        if self.graph is not None:
            self.graph.replay()
            return self.loss
        self.loss = self._body()
        return self.loss
