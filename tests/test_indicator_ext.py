"""The extended indicator (paper_2407_02327_b200/indicator_ext.py) against the
UNMODIFIED reference library (oracle/_ref/libqsync_ref.so):

* INT8 / FP16 / FP32 sigma and Omega equal the reference's (k = 9);
* BF16 is the reference's float branch with k = 7;
* FP8 forward is the reference's float branch with k = 3, FP8 backward is the
  reference's INT8 branch with q_act := 2^(e_act - 3) (the FP8 grid spacing);
* score_bundle over a bundle equals the reference's score_all for the
  reference's rungs and orders the float rungs FP8 >= BF16 >= FP16 > FP32 = 0.
CPU only."""
import json

import numpy as np
import pytest

from paper_2407_02327_b200 import indicator_ext as ix
from paper_2407_02327_b200.qlinear import BF16, FP8, FP16, FP32, INT8

REF_P = {INT8: 0, FP16: 1, FP32: 2}
LOSS = {"mse_mean": 0, "ce_mean": 1, "generic_negone": 2}


def _stats(rng):
    return {"norm_w_sq": float(rng.uniform(1, 500)), "norm_act_sq": float(rng.uniform(1e2, 1e6)),
            "norm_grad_act_sq": float(rng.uniform(1e-6, 1e-2)), "d_act": float(rng.integers(1e3, 1e7)),
            "d_w": float(rng.integers(1e3, 1e7)), "d_grad": float(rng.integers(1e3, 1e7)),
            "q_act": float(rng.uniform(1e-3, 0.1)), "q_w": float(rng.uniform(1e-4, 1e-2)),
            "e_act": float(rng.integers(-4, 5)), "e_w": float(rng.integers(-8, 0)),
            "e_grad": float(rng.integers(-20, -5))}


def _packed(s):
    v = np.array([s.get(f, 0.0) for f in ix.STAT_FIELDS], np.float64)
    mask = sum(1 << i for i, f in enumerate(ix.STAT_FIELDS) if f in s)
    return v, mask


@pytest.mark.parametrize("seed", range(8))
def test_reference_rungs_match(reflib, seed):
    rng = np.random.default_rng(seed)
    s = _stats(rng)
    v, mask = _packed(s)
    for p in (INT8, FP16, FP32):
        for pf in (False, True):
            for which, fn in ((0, ix.sigma_fwd), (1, ix.sigma_bwd)):
                want = reflib.sigma(which, v, mask, REF_P[p], int(pf))
                got = fn(s, p, "op", pf)
                assert got == pytest.approx(want, rel=1e-12, abs=0.0), (p, pf, which)
        for loss in LOSS:
            want = reflib.omega(v, mask, True, 3, 10, LOSS[loss], 32, REF_P[p])
            got = ix.omega("op", 3, True, p, 10, ix.loss_gamma(loss, 32), {"op": s})
            assert got == pytest.approx(want, rel=1e-12, abs=0.0)


@pytest.mark.parametrize("seed", range(8))
def test_bf16_is_reference_float_branch_k7(reflib, seed):
    s = _stats(np.random.default_rng(100 + seed))
    v, mask = _packed(s)
    for pf in (False, True):
        assert ix.sigma_fwd(s, BF16, "op", pf) == pytest.approx(reflib.sigma(0, v, mask, 1, int(pf), k=7), rel=1e-12)
        assert ix.sigma_bwd(s, BF16, "op", pf) == pytest.approx(reflib.sigma(1, v, mask, 1, int(pf), k=7), rel=1e-12)
    assert ix.omega("op", 4, True, BF16, 9, 0.5, {"op": s}) == pytest.approx(
        reflib.omega(v, mask, True, 4, 9, 0, 4, 1, k=7), rel=1e-12)


@pytest.mark.parametrize("seed", range(8))
def test_fp8_pinned_to_reference_formulas(reflib, seed):
    s = _stats(np.random.default_rng(200 + seed))
    v, mask = _packed(s)
    for pf in (False, True):
        assert ix.sigma_fwd(s, FP8, "op", pf) == pytest.approx(reflib.sigma(0, v, mask, 1, int(pf), k=3), rel=1e-12)
    s8 = dict(s, q_act=2.0 ** (s["e_act"] - 3))  # the FP8 grid spacing in the INT8 backward branch
    v8, m8 = _packed(s8)
    assert ix.sigma_bwd(s, FP8, "op", False) == pytest.approx(reflib.sigma(1, v8, m8, 0, 0), rel=1e-12)


def test_errors_mirror_reference():
    with pytest.raises(ix.IndicatorError) as e:
        ix.sigma_fwd({"norm_w_sq": 1.0}, BF16, "layer0.qkv", False)
    assert e.value.kind == "stats-incomplete" and "layer0.qkv" in str(e.value)
    with pytest.raises(ix.IndicatorError) as e:
        ix.omega("x", 0, True, FP8, 4, 1.0, {"x": {}})
    assert e.value.kind == "domain"


def test_score_bundle_matches_score_all_and_orders_ladder(tmp_path, reflib):
    from test_profiler_bundle import _fake_casts, _fake_costs, _fake_stats

    from paper_2407_02327_b200.profiler import bert_graph, build_bundle
    from paper_2407_02327_b200.train_step import BertConfig
    cfg = BertConfig(layers=2)
    g = bert_graph(cfg, 8)
    b = build_bundle(g, _fake_costs(g, cfg, 8), _fake_casts(), _fake_stats(cfg),
                     [{"id": "infer", "is_inference": True, "mem_capacity_bytes": 10 ** 12}])
    path = tmp_path / "b.json"
    path.write_text(json.dumps(b))
    ref = {(op, p): w for op, p, w in reflib.score_bundle(str(path), LOSS["ce_mean"], 32)}
    ours = ix.score_bundle(b, "ce_mean", 32)
    for op, row in ours.items():
        for p in (INT8, FP16, FP32):
            assert row[p] == pytest.approx(ref[(op, p)], rel=1e-12, abs=1e-300)
        # the float rungs order by mantissa width; INT8 vs FP8 depends on the data
        # (the bound charges FP8 its top-binade spacing 2^(e-3) against INT8's absmax/127)
        assert row[FP8] >= row[BF16] >= row[FP16] > row[FP32] == 0.0 and row[INT8] > 0.0
