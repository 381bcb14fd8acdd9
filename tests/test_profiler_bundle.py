"""The profiler's bundle is accepted by the UNMODIFIED reference planner: the
schema (profile.cpp:283-413) validates, score_all ranks the ops, solve emits a
per-device plan, and the plan loads into the training path."""
import json

import pytest

from paper_2407_02327_b200.profiler import (bert_graph, build_bundle, default_cap,
                                            linear_memory_bytes)
from paper_2407_02327_b200.qlinear import FP16, FP32, INT8
from paper_2407_02327_b200.train_step import BertConfig, load_plan


def _fake_costs(graph, cfg, batch):
    T, H = batch * cfg.seq, cfg.hidden
    costs = {}
    speed = {INT8: 0.4, FP16: 0.6, FP32: 1.0}
    for n in graph["nodes"]:
        c = {}
        for p in n["supported_precisions"]:
            w = n["weight_numel"]
            mem = (linear_memory_bytes(p, T, n["output_numel"] // T or 1, max(1, w // max(1, n["output_numel"] // T)))
                   if w else n["output_numel"] * 4)
            c[p] = {"pure_cost_ns": max(1, int((w + n["output_numel"]) * speed[p] * 0.01)),
                    "fwd_fraction": 1.0 / 3.0, "memory_bytes": int(mem)}
        costs[n["id"]] = c
    return costs


def _fake_casts():
    out = []
    for src, dst, sch in [(FP32, FP16, "float_to_float"), (FP16, FP32, "float_to_float"),
                          (FP32, INT8, "quantize_fixed"), (FP16, INT8, "quantize_fixed"),
                          (INT8, FP32, "dequantize_fixed")]:
        for n in (1 << 16, 1 << 20, 1 << 24):
            out.append({"src": src, "dst": dst, "scheme": sch, "numel": n, "measured_ns": 2000 + n // 1000})
    return out


def _fake_stats(cfg, steps=3):
    snaps = []
    for s in range(steps):
        snap = {}
        for i in range(cfg.layers):
            for k in ("qkv", "o", "ff1", "ff2"):
                snap[f"layer{i}.{k}"] = {"norm_w_sq": 100.0 + i, "norm_act_sq": 5e5, "norm_grad_act_sq": 1e-4,
                                         "d_act": 3e6, "d_w": 1e6, "d_grad": 3e6, "q_act": 0.05 + 0.01 * s,
                                         "q_w": 0.001, "e_act": 2, "e_w": -3, "e_grad": -12}
        snap["pooler"] = {"norm_w_sq": 50.0, "norm_act_sq": 1e3, "norm_grad_act_sq": 1e-3, "d_act": 6e3,
                          "d_w": 6e5, "d_grad": 6e3, "q_act": 0.02, "q_w": 0.002, "e_act": 1, "e_w": -4,
                          "e_grad": -10}
        snaps.append(snap)
    return snaps


def test_bundle_accepted_by_reference_planner(tmp_path, reflib):
    cfg = BertConfig(layers=3)
    batch = 8
    g = bert_graph(cfg, batch)
    costs = _fake_costs(g, cfg, batch)
    devices = [{"id": "trainer", "is_inference": False, "mem_capacity_bytes": 10**12},
               {"id": "infer", "is_inference": True, "mem_capacity_bytes": default_cap(g, costs)}]
    b = build_bundle(g, costs, _fake_casts(), _fake_stats(cfg), devices)
    path = tmp_path / "bundle.json"
    path.write_text(json.dumps(b))
    rows = reflib.score_bundle(str(path), 0, 32)
    omegas = {(op, p): w for op, p, w in rows}
    assert omegas[("layer0.qkv", "INT8")] > omegas[("layer0.qkv", "FP16")] > 0
    assert omegas[("layer0.qkv", "FP32")] == 0.0
    rep = reflib.plan_bundle(str(path), 0, 32, 50, "infer", default_cap(g, costs))
    assert rep["memory_ok"]
    assert set(rep["devices"]) == {"trainer", "infer"}
    assert all(p == FP32 for p in rep["devices"]["trainer"].values())  # trainers stay FP32
    ppath = tmp_path / "plan.json"
    ppath.write_text(json.dumps(rep))
    plan = load_plan(str(ppath), "infer")
    assert plan["layer0.qkv"] in (INT8, FP16, FP32)
    # the reference replayer accepts the plan it produced
    assert reflib.replay_bundle(str(path), {"per_device": rep["devices"]}) > 0


@pytest.mark.gpu
def test_profiled_bundle_closes_the_loop(tmp_path, reflib):
    """Measure on the B200 -> reference plan -> apply the plan -> train."""
    import torch

    from paper_2407_02327_b200.profiler import profile_bert
    from paper_2407_02327_b200.train_step import BertEncoderStack, TrainStep
    cfg = BertConfig(vocab=2000, layers=2, max_pos=128)
    batch = 4
    from paper_2407_02327_b200.profiler import default_cap
    b = profile_bert(cfg, batch, stat_steps=2, reps=3)
    path = tmp_path / "bundle.json"
    path.write_text(json.dumps(b))
    rep = None
    for frac in (0.75, 0.9, 1.0):  # tightest cap the reference allocator can satisfy
        cap = default_cap(b["graph"], b["op_costs"], frac)
        try:
            rep = reflib.plan_bundle(str(path), 1, batch, 50, "infer", cap)
            break
        except RuntimeError as e:
            assert "infeasible" in str(e)
    assert rep is not None and rep["memory_ok"]
    ppath = tmp_path / "plan.json"
    ppath.write_text(json.dumps(rep))
    plan = load_plan(str(ppath), "infer")
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(plan)
    st = TrainStep(m, batch=batch, graph=False)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=1)
    loss = float(st().item())
    assert loss == loss and loss > 0  # finite
    # replayer prediction for the measured costs (row (f)2 fidelity, reported not pinned)
    assert reflib.replay_bundle(str(path), {"per_device": rep["devices"]}) > 0
