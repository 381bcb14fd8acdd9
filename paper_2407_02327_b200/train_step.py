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
import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .qlinear import FP16, FP32, INT8, QLinear, cast


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
        if p not in (INT8, FP16, FP32):
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
        self.ln1 = torch.nn.LayerNorm(h, eps=1e-12)
        self.ln2 = torch.nn.LayerNorm(h, eps=1e-12)

    def forward(self, x):  # x [B, S, H] fp32 residual stream
        B, S, H = x.shape
        nh = self.cfg.heads
        qkv = self.qkv(x)  # [B, S, 3H] fp32 (INT8) / fp16 (FP16)
        qkv = cast(qkv, torch.float16)
        q, k, v = qkv.view(B, S, 3, nh, H // nh).permute(2, 0, 3, 1, 4).unbind(0)
        a = F.scaled_dot_product_attention(q, k, v)  # [B, nh, S, d] fp16
        a = a.transpose(1, 2).reshape(B, S, H)
        x = self.ln1(x + cast(self.o(a), torch.float32))
        f = F.gelu(self.ff1(x))
        x = self.ln2(x + cast(self.ff2(f), torch.float32))
        return x


class BertEncoderStack(torch.nn.Module):
    """BERT-base: embeddings + 12 encoder layers + pooler + classifier."""

    def __init__(self, cfg: BertConfig):
        super().__init__()
        self.cfg = cfg
        self.word = torch.nn.Embedding(cfg.vocab, cfg.hidden)
        self.pos = torch.nn.Embedding(cfg.max_pos, cfg.hidden)
        self.typ = torch.nn.Embedding(cfg.type_vocab, cfg.hidden)
        self.ln = torch.nn.LayerNorm(cfg.hidden, eps=1e-12)
        self.layers = torch.nn.ModuleList([EncoderLayer(cfg, i) for i in range(cfg.layers)])
        self.pooler = QLinear(cfg.hidden, cfg.hidden, "pooler")
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
        pos = torch.arange(S, device=tokens.device)
        x = self.word(tokens) + self.pos(pos)[None] + self.typ.weight[0][None, None]
        x = self.ln(x)
        for layer in self.layers:
            x = layer(x)
        pooled = torch.tanh(cast(self.pooler(x[:, 0].contiguous()), torch.float32))
        logits = self.cls(pooled)
        return F.cross_entropy(logits, labels)


def linear_flops_per_step(cfg: BertConfig, tokens: int) -> float:
    """fwd + dgrad + wgrad of the 48 encoder Linears."""
    h, f = cfg.hidden, cfg.ffn
    per_layer = 2 * tokens * (h * 3 * h + h * h + h * f + f * h)
    return 3.0 * per_layer * cfg.layers


# --------------------------------------------------------------------------- DP
class BucketReducer:
    """Bucketed FP32 gradient all-reduce in backward (reverse-topological) order.

    Buckets are fixed at construction from the parameter order, identical on all
    ranks; ``reduce()`` issues one all-reduce per bucket, in order, on the
    current stream, then divides by the world size.  Works on any device / any
    torch.distributed backend (NCCL on B200, gloo in the CPU tests).
    """

    def __init__(self, params: list[torch.nn.Parameter], bucket_bytes: int = 25 << 20):
        self.params = [p for p in params if p.requires_grad]
        self.buckets: list[list[torch.nn.Parameter]] = []
        cur: list[torch.nn.Parameter] = []
        size = 0
        for p in reversed(self.params):  # backward order: last layer's grads first
            cur.append(p)
            size += p.numel() * 4
            if size >= bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
        if cur:
            self.buckets.append(cur)
        self.flat = None

    def _flat(self, device):
        if self.flat is None:
            self.flat = [torch.zeros(sum(p.numel() for p in b), device=device) for b in self.buckets]
        return self.flat

    def reduce(self, world: int) -> None:
        import torch.distributed as dist
        if world <= 1:
            return
        flats = self._flat(self.params[0].device)
        for b, flat in zip(self.buckets, flats):
            off = 0
            for p in b:
                n = p.numel()
                flat[off:off + n].copy_(p.grad.reshape(-1))
                off += n
            dist.all_reduce(flat)
            flat.div_(world)
            off = 0
            for p in b:
                n = p.numel()
                p.grad.copy_(flat[off:off + n].view_as(p.grad))
                off += n


class TrainStep:
    """One synchronous DP step: fwd + bwd (planned kernels) + bucketed all-reduce
    + AdamW on FP32 master weights.  Optionally captured into a CUDA graph."""

    def __init__(self, model: BertEncoderStack, batch: int, world: int = 1, lr: float = 1e-4,
                 graph: bool = True):
        self.model = model
        self.world = world
        cfg = model.cfg
        dev = next(model.parameters()).device
        self.tokens = torch.zeros((batch, cfg.seq), dtype=torch.long, device=dev)
        self.labels = torch.zeros((batch,), dtype=torch.long, device=dev)
        self.params = [p for p in model.parameters() if p.requires_grad]
        for p in self.params:
            p.grad = torch.zeros_like(p)
        self.opt = torch.optim.AdamW(self.params, lr=lr, fused=True, capturable=graph)
        self.reducer = BucketReducer(self.params)
        self.use_graph = graph
        self.graph = None
        self.loss = None

    def _body(self):
        loss = self.model(self.tokens, self.labels)
        loss.backward()
        self.reducer.reduce(self.world)
        self.opt.step()
        for p in self.params:
            p.grad.zero_()
        return loss.detach()

    def capture(self, warmup: int = 3) -> None:
        s = torch.cuda.Stream()
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
