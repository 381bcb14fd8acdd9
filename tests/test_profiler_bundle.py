"""The profiler's bundle is accepted by the UNMODIFIED reference planner: the
schema (profile.cpp:283-413) validates, score_all ranks the ops, solve emits a
per-device plan, and the plan loads into the training path."""
import json

import pytest

from paper_2407_02327_b200.profiler import (bert_graph, build_bundle, default_cap, fit_cast,
                                            linear_memory_bytes, net_weight_casts)
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


def test_comm_slots_accepted_and_replayed(tmp_path, reflib):
    """The CommSlot sink (profile.hpp:118-129): a bundle carrying per-device
    bucket slots validates (profile.cpp:385-410) and the replayer's Eq. 6 slots
    (replayer.cpp:48-73) lengthen the step when the exchange is exposed."""
    cfg = BertConfig(layers=3)
    batch = 8
    g = bert_graph(cfg, batch)
    costs = _fake_costs(g, cfg, batch)
    devices = [{"id": "trainer", "is_inference": False, "mem_capacity_bytes": 10**12},
               {"id": "infer", "is_inference": True, "mem_capacity_bytes": 10**12}]
    plan = {"per_device": {"trainer": {}, "infer": {}}}
    base = build_bundle(g, costs, _fake_casts(), _fake_stats(cfg), devices)
    p0 = tmp_path / "b0.json"
    p0.write_text(json.dumps(base))
    t0 = reflib.replay_bundle(str(p0), plan)
    slots = [{"earliest_ready_offset_ns": 1000 * (i + 1), "duration_ns": 10_000_000, "bucket_bytes": 32 << 20}
             for i in range(3)]
    withc = build_bundle(g, costs, _fake_casts(), _fake_stats(cfg), devices,
                         comm={"trainer": slots, "infer": slots})
    p1 = tmp_path / "b1.json"
    p1.write_text(json.dumps(withc))
    t1 = reflib.replay_bundle(str(p1), plan)
    # three 10 ms slots run back to back (in order) and the optimizer waits for the last
    assert t1 > t0 and t1 >= 3 * 10_000_000
    bad = build_bundle(g, costs, _fake_casts(), _fake_stats(cfg), devices,
                       comm={"trainer": slots, "infer": slots[:2]})
    p2 = tmp_path / "b2.json"
    p2.write_text(json.dumps(bad))
    with pytest.raises(Exception) as e:
        reflib.replay_bundle(str(p2), plan)
    assert "topology" in str(e.value)


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


def test_fit_cast_mirrors_reference_cast_model():
    """OLS a*numel + b with the reference's clamps (profile.cpp:33-83)."""
    a, b = fit_cast([(100, 300), (200, 500), (400, 900)])
    assert abs(a - 2.0) < 1e-12 and abs(b - 100.0) < 1e-9
    a, b = fit_cast([(100, 900), (200, 500)])            # negative slope -> flat mean
    assert a == 0.0 and b == 700.0
    a, b = fit_cast([(100, 1), (200, 400), (300, 800)])  # negative intercept -> through the origin
    assert b == 0.0 and abs(a - (100 * 1 + 200 * 400 + 300 * 800) / (100**2 + 200**2 + 300**2)) < 1e-12


def test_net_weight_casts_cancel_the_mappers_weight_cast(tmp_path, reflib):
    """Storing each weighted op net of its FP32 -> k weight cast (the fused step
    converts weights inside the optimizer) lowers the reference replayer's
    prediction by exactly the casts its cost mapper adds (cost_mapper.cpp:42-43)."""
    import copy
    import math

    from paper_2407_02327_b200.profiler import _param_numel
    from paper_2407_02327_b200.train_step import uniform_plan
    cfg = BertConfig(layers=3)
    batch = 8
    g = bert_graph(cfg, batch)
    costs = _fake_costs(g, cfg, batch)
    for per_p in costs.values():  # forward shares large enough to absorb the casts
        for e in per_p.values():
            e["pure_cost_ns"] += 10**7
            e["fwd_fraction"] = 0.5
    casts = _fake_casts()
    dev = [{"id": "d", "is_inference": True, "mem_capacity_bytes": 10**13}]
    raw = tmp_path / "raw.json"
    raw.write_text(json.dumps(build_bundle(g, costs, casts, _fake_stats(cfg), dev)))
    net = tmp_path / "net.json"
    net.write_text(json.dumps(build_bundle(g, net_weight_casts(cfg, copy.deepcopy(costs), casts),
                                           casts, _fake_stats(cfg), dev)))
    for p in (INT8, FP16):
        plan = {"per_device": {"d": uniform_plan(cfg, p)}}
        a, b = fit_cast([(s["numel"], s["measured_ns"]) for s in casts if s["src"] == FP32 and s["dst"] == p])
        want = sum(int(math.floor(a * w + b + 0.5)) for op, (w, _) in _param_numel(cfg).items()
                   if w and op in plan["per_device"]["d"])
        assert reflib.replay_bundle(str(raw), plan) - reflib.replay_bundle(str(net), plan) == pytest.approx(want, abs=2 * len(costs))


@pytest.mark.gpu
def test_fused_bundle_closes_the_loop(tmp_path, reflib):
    """The fused-implementation bundle (operator regions of the fused step,
    conversions as marginal costs) is accepted by the reference planner and its
    replayer predicts the measured graphed step of a uniform plan closely."""
    from paper_2407_02327_b200.profiler import graph_step_ms, measure_fused_costs, profile_bert_fused
    from paper_2407_02327_b200.train_step import uniform_plan
    cfg = BertConfig(vocab=2000, layers=2, max_pos=128)
    batch = 8
    b = profile_bert_fused(cfg, batch, stat_steps=2, reps=3)
    path = tmp_path / "bundle.json"
    path.write_text(json.dumps(b))
    assert set(measure_fused_costs.last_diag) == {INT8, FP16, FP32}
    rep = reflib.plan_bundle(str(path), 1, batch, 50, "infer", 10**12)
    assert rep["memory_ok"] and set(rep["devices"]) == {"trainer", "infer"}
    # replay one device (the bundle's trainer would stay FP32 and set the makespan)
    b["devices"] = [d for d in b["devices"] if d["id"] == "infer"]
    path.write_text(json.dumps(b))
    plan = {"per_device": {"infer": uniform_plan(cfg, FP16)}}
    pred_ms = reflib.replay_bundle(str(path), plan) / 1e6
    meas_ms = graph_step_ms(cfg, batch, plan["per_device"]["infer"])
    assert abs(pred_ms - meas_ms) / meas_ms < 0.25


def test_resnet50_bundle_accepted_by_reference_planner(tmp_path, reflib):
    """The conv model's graph (53 adjustable convs, fixed BN/add, fc) with conv op
    costs goes through the unmodified reference score / solve / replay."""
    from paper_2407_02327_b200.profiler_resnet import conv_memory_bytes, resnet50_graph
    from paper_2407_02327_b200.resnet import conv_specs
    batch = 8
    g = resnet50_graph(batch)
    adj = [n["id"] for n in g["nodes"] if n["kind"] == "adjustable"]
    assert len(adj) == 54 and "fc" in adj  # 53 convs + classifier
    specs = {s[0]: s for s in conv_specs(batch)}
    speed = {INT8: 0.5, FP16: 0.7, FP32: 1.0}
    costs = {}
    for n in g["nodes"]:
        costs[n["id"]] = {}
        for p in n["supported_precisions"]:
            if n["id"] in specs:
                _, nb, h, _, c, cout, r, _, _, _ = specs[n["id"]]
                mem = conv_memory_bytes(p, nb, h, c, cout, r)
            else:
                mem = n["output_numel"] * 4 + n["weight_numel"] * 16
            costs[n["id"]][p] = {"pure_cost_ns": max(1, int(n["output_numel"] * speed[p] * 0.01)),
                                 "fwd_fraction": 1.0 / 3.0, "memory_bytes": int(mem)}
    stats = []
    for s in range(2):
        stats.append({op: {"norm_w_sq": 10.0, "norm_act_sq": 4e4, "norm_grad_act_sq": 1e-5,
                           "d_act": 1e5, "d_w": 4e4, "d_grad": 1e5, "q_act": 0.03 + 0.01 * s,
                           "q_w": 0.002, "e_act": 1, "e_w": -4, "e_grad": -14} for op in adj})
    cap = default_cap(g, costs)
    devices = [{"id": "trainer", "is_inference": False, "mem_capacity_bytes": 10**12},
               {"id": "infer", "is_inference": True, "mem_capacity_bytes": cap}]
    path = tmp_path / "rn50.json"
    path.write_text(json.dumps(build_bundle(g, costs, _fake_casts(), stats, devices)))
    omegas = {(op, p): w for op, p, w in reflib.score_bundle(str(path), 0, batch)}
    assert omegas[("res3.0.b", "INT8")] > omegas[("res3.0.b", "FP16")] > 0
    rep = reflib.plan_bundle(str(path), 0, batch, 50, "infer", cap)
    assert rep["memory_ok"]
    assert all(p == FP32 for p in rep["devices"]["trainer"].values())
    assert any(rep["devices"]["infer"][op] != FP32 for op in adj)
    assert reflib.replay_bundle(str(path), {"per_device": rep["devices"]}) > 0
