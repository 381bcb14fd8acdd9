"""Config 3 as a model: ResNet-50 (NHWC) trained under a per-conv precision plan,
and its measured ProfileBundle closing the loop through the unmodified reference
planner (profile.hpp:72-76 OpCostEntry for K8; cli.cpp:116-136 solve)."""
import json

import pytest
import torch

from paper_2407_02327_b200.qlinear import FP16, FP32, INT8
from paper_2407_02327_b200.resnet import ResNet50, conv_specs
from paper_2407_02327_b200.train_step import load_plan

pytestmark = pytest.mark.gpu


def _loss_and_grads(model, img, lab):
    model.zero_grad(set_to_none=True)
    loss = model(img, lab)
    loss.backward()
    g = {n: m.weight.grad.detach().clone() for n, m in model.qops().items()}
    return float(loss.item()), g


@pytest.mark.parametrize("plan_kind", ["int8", "fp16", "mixed"])
def test_resnet50_plan_tracks_fp32(plan_kind):
    """Every conv switched to INT8 / FP16 (or alternating) keeps the loss and the
    weight gradients of the FP32 model within quantization tolerance."""
    torch.manual_seed(0)
    m = ResNet50(num_classes=16, image=64).cuda()
    img = torch.randn(4, 64, 64, 3, device="cuda")
    lab = torch.randint(0, 16, (4,), device="cuda")
    m.train(False)  # BN in inference mode: the comparison isolates the conv kernels
    m.apply_plan({})
    l32, g32 = _loss_and_grads(m, img, lab)
    names = [s[0] for s in conv_specs(1)]
    if plan_kind == "int8":
        plan = {n: INT8 for n in names}
    elif plan_kind == "fp16":
        plan = {n: FP16 for n in names}
    else:
        plan = {n: (INT8 if i % 2 else FP16) for i, n in enumerate(names)}
    m.apply_plan(plan)
    lq, gq = _loss_and_grads(m, img, lab)
    tol = 5e-2 if plan_kind != "fp16" else 1e-2
    assert abs(lq - l32) <= tol * abs(l32)
    # Quantization noise compounds through the backward of the 53-conv stack: the
    # gradient direction is the bar (cosine), tighter near the head.
    for n, lo in (("conv1", 0.9), ("res3.0.b", 0.9), ("res5.2.c", 0.97), ("fc", 0.99)):
        cos = torch.nn.functional.cosine_similarity(gq[n].flatten(), g32[n].flatten(), dim=0).item()
        assert cos > (lo if plan_kind != "fp16" else 0.999), (n, cos)


def test_resnet50_bundle_closes_the_loop(tmp_path, reflib):
    """Measure the conv model on the B200 -> reference plan -> apply -> train."""
    from paper_2407_02327_b200.profiler import default_cap
    from paper_2407_02327_b200.profiler_resnet import profile_resnet50
    batch = 4
    b = profile_resnet50(batch, image=64, num_classes=16, stat_steps=2, reps=2)
    convs = [s[0] for s in conv_specs(batch, 64)]
    for op in convs + ["fc"]:
        c = b["op_costs"][op]
        assert set(c) == {INT8, FP16, FP32} and all(v["pure_cost_ns"] > 0 for v in c.values())
    assert len(b["tensor_stats"]) == 2 and set(convs) <= set(b["tensor_stats"][0])
    path = tmp_path / "rn50.json"
    path.write_text(json.dumps(b))
    omegas = {(op, p): w for op, p, w in reflib.score_bundle(str(path), 1, batch)}
    assert omegas[("res4.1.b", INT8)] > 0 and omegas[("res4.1.b", FP32)] == 0.0
    rep = None
    for frac in (0.75, 0.9, 1.0):
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
    m = ResNet50(num_classes=16, image=64).cuda()
    m.apply_plan(plan)
    img = torch.randn(batch, 64, 64, 3, device="cuda")
    lab = torch.randint(0, 16, (batch,), device="cuda")
    loss = m(img, lab)
    loss.backward()
    assert torch.isfinite(loss) and all(torch.isfinite(p.grad).all() for p in m.parameters()
                                        if p.grad is not None)
    assert reflib.replay_bundle(str(path), {"per_device": rep["devices"]}) > 0
