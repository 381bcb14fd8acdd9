"""ResNet-50 ProfileBundle: the conv workload measured on the B200 for the planner.

The reference's `OpCostEntry` sink (profile.hpp:72-76) is op-generic; this module
fills it for the 53 convolutions of BASELINE configs[2] (K8 implicit-GEMM conv) so
the unmodified planner (`solve`, cli.cpp:116-136) and replayer can plan and replay
the conv model on B200 numbers, as `profiler.profile_bert` does for BERT-base.

* ``graph``     -- conv (adjustable INT8/FP16/FP32), BN+ReLU (fixed FP32) per conv,
                   residual add+ReLU (fixed), pool, fc (adjustable), loss (fixed);
                   residual and shortcut edges included.
* ``op_costs``  -- per distinct conv geometry and precision: device time of the
                   op's forward and forward+backward kernels (launches queued behind a
                   device spin, CUDA events, median). The operator is fed the format
                   its producer hands it at that precision (FP16 conv: FP16 input), and
                   the conversions the cost mapper charges itself (cost_mapper.cpp:36-50:
                   the forward weight cast; for INT8 also the input quantizer and the
                   FP32 -> FP16 cast of the incoming gradient) are measured and netted out.
* ``cast_samples`` / ``devices`` -- as for BERT (profiler.measure_cast_samples).
* ``tensor_stats`` -- K5 device statistics of every conv's input, weight and
                   incoming gradient over FP32 training steps of `resnet.ResNet50`.
"""
from __future__ import annotations

import statistics

import torch
import torch.nn.functional as F

from . import ops, qlinear
from .profiler import (StatsRecorder, build_bundle, default_cap, linear_memory_bytes,
                       measure_cast_samples, measure_linear)
from .qconv import qconv2d
from .qlinear import FP16, FP32, INT8
from .resnet import STAGES, ResNet50, conv_specs


def _spin_ns(fn, reps: int = 5) -> int:
    """Median device time of fn() with its launches queued behind a device spin
    (host launch overhead excluded, as in a graphed step)."""
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(20_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e6)
    return max(1, int(statistics.median(ts)))


def _out_hw(h: int, r: int, s: int, p: int) -> int:
    return (h + 2 * p - r) // s + 1


# ----------------------------------------------------------------------------- graph
def resnet50_graph(batch: int, image: int = 224, num_classes: int = 1000) -> dict:
    nodes, edges = [], []
    all3 = [INT8, FP16, FP32]

    def node(i, kind, out, sub, prec, w=0):
        nodes.append({"id": i, "kind": kind, "output_numel": out, "subgraph_id": sub,
                      "supported_precisions": prec, "has_weight": w > 0, "weight_numel": w})

    def conv(name, src, n, h, c, cout, r, s, p, blk):
        q = _out_hw(h, r, s, p)
        node(name, "adjustable", n * q * q * cout, blk, all3, cout * r * r * c)
        node(f"{name}.bn", "fixed", n * q * q * cout, blk, [FP32])
        edges.extend([[src, name], [name, f"{name}.bn"]])
        return f"{name}.bn", q

    specs = {s[0]: s for s in conv_specs(batch, image)}
    _, n, h, _, c, cout, r, st, p, blk = specs["conv1"]
    prev, h = conv("conv1", "input", n, h, c, cout, r, st, p, blk)
    node("input", "fixed", batch * image * image * 3, "stem", [FP32])
    h = h // 2  # max pool
    for si, (_, blocks, _) in enumerate(STAGES):
        for b in range(blocks):
            blk = f"res{si + 2}.{b}"
            y = prev
            for part in ("a", "b", "c"):
                _, n, hh, _, c, cout, r, st, p, _ = specs[f"{blk}.{part}"]
                y, _ = conv(f"{blk}.{part}", y, n, hh, c, cout, r, st, p, blk)
            if b == 0:
                _, n, hh, _, c, cout, r, st, p, _ = specs[f"{blk}.ds"]
                sc, _ = conv(f"{blk}.ds", prev, n, hh, c, cout, r, st, p, blk)
            else:
                sc = prev
            _, n, hh, _, c, cout, r, st, p, _ = specs[f"{blk}.c"]
            node(f"{blk}.add", "fixed", n * hh * hh * cout, blk, [FP32])
            edges.extend([[y, f"{blk}.add"], [sc, f"{blk}.add"]])
            prev = f"{blk}.add"
    node("fc", "adjustable", batch * num_classes, "head", all3, 2048 * num_classes)
    node("loss", "fixed", batch, "head", [FP32])
    edges.extend([[prev, "fc"], ["fc", "loss"]])
    return {"nodes": nodes, "edges": edges, "assignment": {x["id"]: FP32 for x in nodes}}


# ----------------------------------------------------------------------------- op costs
def conv_memory_bytes(precision: str, n: int, h: int, c: int, cout: int, r: int) -> int:
    """Bytes the conv keeps resident at a precision: FP32 master weight + gradient +
    AdamW moments, and the operand saved for backward (the INT8 op keeps its int8
    NHWC input, FP16 its FP16 input and weight copy, FP32 its FP32 input)."""
    w = cout * r * r * c
    act = n * h * h * c
    base = 16 * w
    if precision == INT8:
        return base + act
    if precision == FP16:
        return base + 2 * act + 2 * w
    return base + 4 * act


def measure_conv(n, h, c, cout, r, stride, pad, precision: str, reps: int = 5) -> dict:
    x32 = torch.randn(n, h, h, c, device="cuda")
    xin = x32.half() if precision == FP16 else x32
    w = (torch.randn(cout, r, r, c, device="cuda") / (r * r * c) ** 0.5).requires_grad_(True)
    xg = xin.detach().clone().requires_grad_(c != 3)  # the stem's input (images) has no dgrad
    wrt = [t for t in (xg, w) if t.requires_grad]
    st, pd = (stride, stride), (pad, pad)
    y = qconv2d(xg, w, None, st, pd, precision)
    gy = torch.randn_like(y)

    def fwd():
        with torch.no_grad():
            qconv2d(xin, w, None, st, pd, precision)

    def fwd_bwd():
        torch.autograd.grad(qconv2d(xg, w, None, st, pd, precision), wrt, gy)

    f, t = _spin_ns(fwd, reps), _spin_ns(fwd_bwd, reps)
    # Conversions the cost mapper charges itself (cost_mapper.cpp:36-50) are netted
    # out of the op: the forward weight cast (both precisions), and for INT8 the
    # input quantizer and the FP32 -> FP16 cast of the incoming gradient.
    w2 = w.detach().reshape(cout, -1).contiguous()
    if precision == INT8:
        k = w2.shape[1]
        w2p = torch.zeros(cout, (k + 15) // 16 * 16, device="cuda") if k % 16 else w2
        if k % 16:
            w2p[:, :k] = w2
        fc = _spin_ns(lambda: ops.quantize_per_tensor(x32.view(1, -1)), reps) + \
            _spin_ns(lambda: ops.quantize_per_channel(w2p), reps)
        g2 = gy.reshape(-1, cout).contiguous()
        bc = _spin_ns(lambda: ops.cast_transpose(g2, True, False, False), reps)
    elif precision == FP16:
        fc, bc = _spin_ns(lambda: ops.cast(w2, torch.float16), reps), 0
    else:
        fc = bc = 0
    f, t = max(1, f - fc), max(2, t - fc - bc)
    t = max(t, f + 1)
    return {"pure_cost_ns": t, "fwd_fraction": min(1.0, f / t),
            "memory_bytes": conv_memory_bytes(precision, n, h, c, cout, r)}


def _bn_relu_ns(n, q, c, reps) -> int:
    bn = torch.nn.BatchNorm2d(c).cuda()
    x = torch.randn(n, c, q, q, device="cuda").to(memory_format=torch.channels_last).requires_grad_(True)
    g = torch.randn_like(x)
    return _spin_ns(lambda: torch.autograd.grad(F.relu(bn(x)), x, g), reps)


def _add_relu_ns(numel, reps) -> int:
    a = torch.randn(numel, device="cuda", requires_grad=True)
    b = torch.randn(numel, device="cuda", requires_grad=True)
    g = torch.randn(numel, device="cuda")
    return _spin_ns(lambda: torch.autograd.grad(F.relu(a + b), (a, b), g), reps)


def measure_resnet50_costs(batch: int, image: int = 224, num_classes: int = 1000,
                           reps: int = 5) -> dict:
    graph = resnet50_graph(batch, image, num_classes)
    by_id = {x["id"]: x for x in graph["nodes"]}
    geom = {}
    for name, n, h, _, c, cout, r, s, p, _ in conv_specs(batch, image):
        geom[name] = (n, h, c, cout, r, s, p)
    cache, costs = {}, {}
    for name, g in geom.items():
        if g not in cache:
            cache[g] = {pr: measure_conv(*g, pr, reps=reps) for pr in (INT8, FP16, FP32)}
            torch.cuda.empty_cache()
        costs[name] = cache[g]
    fixed = {}
    for nid, nd in by_id.items():
        if nid.endswith(".bn"):
            n, h, c, cout, r, s, p = geom[nid[:-3]]
            key = ("bn", n, _out_hw(h, r, s, p), cout)
            if key not in fixed:
                fixed[key] = _bn_relu_ns(n, key[2], cout, reps)
            t = fixed[key]
        elif nid.endswith(".add"):
            key = ("add", nd["output_numel"])
            if key not in fixed:
                fixed[key] = _add_relu_ns(nd["output_numel"], reps)
            t = fixed[key]
        elif nid in ("input", "loss"):
            t = 1000
        else:
            continue
        costs[nid] = {FP32: {"pure_cost_ns": t, "fwd_fraction": 1.0 / 3.0,
                             "memory_bytes": nd["output_numel"] * 4}}
    costs["fc"] = {pr: measure_linear(batch, num_classes, 2048, pr, reps) for pr in (INT8, FP16, FP32)}
    for pr in costs["fc"]:
        costs["fc"][pr]["memory_bytes"] = linear_memory_bytes(pr, batch, num_classes, 2048)
    return costs


# ----------------------------------------------------------------------------- stats
def collect_conv_stats(model: ResNet50, batch: int, steps: int, seed: int = 0) -> list:
    """`steps` FP32 SGD steps of the model on synthetic images; one OpStats snapshot
    per step for every conv and the classifier."""
    g = torch.Generator().manual_seed(seed)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3)
    rec = StatsRecorder()
    snaps = []
    qlinear.STATS_RECORDER = rec
    try:
        for _ in range(steps):
            img = torch.randn(batch, model.image, model.image, 3, generator=g).cuda()
            lab = torch.randint(0, model.fc.out_features, (batch,), generator=g).cuda()
            opt.zero_grad(set_to_none=True)
            model(img, lab).backward()
            opt.step()
            snaps.append(rec.snapshot())
    finally:
        qlinear.STATS_RECORDER = None
    return snaps


def profile_resnet50(batch: int, image: int = 224, num_classes: int = 1000, stat_steps: int = 3,
                     stat_batch: int | None = None, reps: int = 5,
                     infer_cap_bytes: int | None = None) -> dict:
    """Measure the conv model on the current device and return the bundle dict."""
    model = ResNet50(num_classes, image).cuda()
    model.apply_plan({})  # statistics at FP32 (the reference's assignment)
    stats = collect_conv_stats(model, stat_batch or min(batch, 16), stat_steps)
    del model
    torch.cuda.empty_cache()
    costs = measure_resnet50_costs(batch, image, num_classes, reps)
    casts = measure_cast_samples(reps=reps)
    graph = resnet50_graph(batch, image, num_classes)
    cap = infer_cap_bytes or default_cap(graph, costs)
    devices = [{"id": "trainer", "is_inference": False, "mem_capacity_bytes": 183_000_000_000},
               {"id": "infer", "is_inference": True, "mem_capacity_bytes": max(cap, 1)}]
    return build_bundle(graph, costs, casts, stats, devices)


def main(argv=None):
    import argparse
    import gzip
    import json
    ap = argparse.ArgumentParser(description="profile ResNet-50 convs into a QSync bundle")
    ap.add_argument("--out", required=True)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--stat-steps", type=int, default=3)
    args = ap.parse_args(argv)
    b = profile_resnet50(args.batch, stat_steps=args.stat_steps)
    op = gzip.open if args.out.endswith(".gz") else open
    with op(args.out, "wt") as f:
        json.dump(b, f)
    print(f"wrote {args.out}")


if __name__ == "__main__":
    main()
