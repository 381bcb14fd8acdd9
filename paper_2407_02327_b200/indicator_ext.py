"""The bi-directional indicator extended to this ladder's extra rungs (BF16, FP8).

The reference scores INT8 / FP16 / FP32 only (``score_all``,
indicator.cpp:144-162) but keeps the mantissa width ``k`` a parameter
(indicator.hpp:45-56: "k is a parameter so BF16 (k=7) can be added
without code change").  This module applies the reference's formulas
(indicator.cpp:35-132, Prop. 2 / Eq. 3-5 of PAPER.md) unchanged to

  * BF16: the float branch with k = 7 (BF16 forward AND backward, emitted BF16);
  * FP8 (E4M3, scaled): forward on a float grid with k = 3 (E4M3's explicit
    mantissa bits, the BF16 convention above) for both the activation and the
    weight; backward like the INT8 op's (cost_mapper.cpp:13-15: the backward
    runs in FP16) -- the saved activation keeps its FP8 grid (k = 3), the
    incoming gradient sits on the FP16 grid (k = 9): the INT8 branch of
    sigma_bwd (indicator.cpp:99-107) with the fixed-point term q_act^2 replaced
    by the FP8 spacing 2^(2 e_act) 2^(-6).

For INT8 / FP16 / FP32 the functions reproduce the reference exactly (k = 9).
Inputs are the ``OpStats`` fields (profile.hpp:95-108) as a dict, reduced over
the first W snapshots as ``reduce_stats`` does (profile.cpp:134-162).
tests/test_indicator_ext.py pins every value against the reference library.
"""
from __future__ import annotations

from .qlinear import BF16, FP8, FP16, FP32, INT8

FLOAT_K = {FP16: 9, BF16: 7, FP8: 3}  # kFp16MantissaBits = 9 (indicator.hpp:31)
STAT_FIELDS = ("norm_w_sq", "norm_act_sq", "norm_grad_act_sq", "norm_grad_act_hat_sq", "d_act", "d_w",
               "d_grad", "q_act", "q_w", "e_act", "e_w", "e_grad")


class IndicatorError(ValueError):
    """Mirror of qsync::Error for this module: ``kind`` is the ErrorKind tag."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def _need(s: dict, field: str, op: str) -> float:
    v = s.get(field)
    if v is None:  # indicator.cpp:49-53
        raise IndicatorError("stats-incomplete", f"operator \"{op}\" is missing statistic {field}")
    return float(v)


def fixed_point_tensor_variance(q: float, d: float) -> float:
    """q^2 D / 6 (indicator.cpp:35-39)."""
    if q <= 0:
        raise IndicatorError("domain", "fixed-point scaling factor must be > 0")
    if d < 0:
        raise IndicatorError("domain", "element count must be >= 0")
    return q * q * d / 6.0


def float_tensor_variance(e: float, k: int, d: float) -> float:
    """2^(2e) 2^(-2k) D / 6 (indicator.cpp:41-45)."""
    if k < 1:
        raise IndicatorError("domain", "mantissa bit count must be at least 1")
    if d < 0:
        raise IndicatorError("domain", "element count must be >= 0")
    return 2.0 ** (2.0 * e) * 2.0 ** (-2.0 * k) * d / 6.0


def sigma_fwd(s: dict, p: str, op: str, parameter_free: bool) -> float:
    """Forward variance increment of running ``op`` at ``p`` (indicator.cpp:65-89)."""
    if p == FP32:
        return 0.0
    if parameter_free:
        d_act = _need(s, "d_act", op)
        if p == INT8:
            return fixed_point_tensor_variance(_need(s, "q_act", op), d_act)
        return float_tensor_variance(_need(s, "e_act", op), FLOAT_K[p], d_act)
    norm_w = _need(s, "norm_w_sq", op)
    norm_act = _need(s, "norm_act_sq", op)
    d_act = _need(s, "d_act", op)
    d_w = _need(s, "d_w", op)
    if p == INT8:
        q_act, q_w = _need(s, "q_act", op), _need(s, "q_w", op)
        return (norm_w * q_act * q_act * d_act + norm_act * q_w * q_w * d_w) / 6.0
    eps_sq = 2.0 ** (-2.0 * FLOAT_K[p])
    e_act, e_w = _need(s, "e_act", op), _need(s, "e_w", op)
    return eps_sq * (norm_w * 2.0 ** (2.0 * e_act) * d_act + norm_act * 2.0 ** (2.0 * e_w) * d_w) / 6.0


def sigma_bwd(s: dict, p: str, op: str, parameter_free: bool) -> float:
    """Backward variance increment (indicator.cpp:91-114); FP8 as documented above."""
    if p == FP32 or parameter_free:
        return 0.0
    norm_act = _need(s, "norm_act_sq", op)
    d_act = _need(s, "d_act", op)
    d_grad = _need(s, "d_grad", op)
    e_grad = _need(s, "e_grad", op)
    if p in (INT8, FP8):
        # the backward runs in FP16: the incoming gradient on the FP16 grid
        eps16_sq = 2.0 ** (-2.0 * FLOAT_K[FP16])
        norm_grad = _need(s, "norm_grad_act_sq", op)
        if p == INT8:
            act_sq = _need(s, "q_act", op) ** 2
        else:  # the saved FP8 activation's grid spacing squared
            act_sq = 2.0 ** (2.0 * _need(s, "e_act", op)) * 2.0 ** (-2.0 * FLOAT_K[FP8])
        return (norm_grad * act_sq * d_act + norm_act * 2.0 ** (2.0 * e_grad) * eps16_sq * d_grad) / 6.0
    eps_sq = 2.0 ** (-2.0 * FLOAT_K[p])
    e_act = _need(s, "e_act", op)
    grad_hat = s.get("norm_grad_act_hat_sq")
    if grad_hat is None:  # indicator.cpp:57-62
        grad_hat = _need(s, "norm_grad_act_sq", op)
    return eps_sq * (grad_hat * 2.0 ** (2.0 * e_act) * d_act + norm_act * 2.0 ** (2.0 * e_grad) * d_grad) / 6.0


def loss_gamma(kind: str, n: int) -> float:
    """LossSpec::gamma (indicator.cpp:25-33)."""
    if n < 1:
        raise IndicatorError("domain", "loss batch denominator must be at least 1")
    return {"mse_mean": 2.0 / n, "ce_mean": 1.0 / n, "generic_negone": -1.0}[kind]


def omega(op: str, depth: int, has_weight: bool, p: str, d_l: int, gamma: float, stats: dict) -> float:
    """gamma^2 d_o sigma_fwd + (d_L - d_o) sigma_bwd (indicator.cpp:116-132)."""
    if p == FP32:
        return 0.0
    if depth < 1 or depth > d_l:
        raise IndicatorError("domain", f"operator \"{op}\" has depth {depth} outside [1, {d_l}]")
    if op not in stats:
        raise IndicatorError("stats-incomplete", f"operator \"{op}\" has no statistics")
    s = stats[op]
    return gamma * gamma * depth * sigma_fwd(s, p, op, not has_weight) + \
        (d_l - depth) * sigma_bwd(s, p, op, not has_weight)


def reduce_stats(snapshots: list[dict], window: int = 50) -> dict:
    """Field-wise mean over the FIRST min(window, n) snapshots (profile.cpp:134-162)."""
    take = snapshots[:max(0, window)]
    ops = set().union(*(s.keys() for s in take)) if take else set()
    out = {}
    for op in ops:
        red = {}
        for f in STAT_FIELDS:
            vals = [s[op][f] for s in take if op in s and s[op].get(f) is not None]
            if vals:
                red[f] = sum(vals) / len(vals)
        out[op] = red
    return out


def depths(graph: dict) -> tuple[dict, int]:
    """Node depth = 1 + max predecessor depth; model depth = the max (graph.cpp:172-177)."""
    preds: dict = {n["id"]: [] for n in graph["nodes"]}
    for a, b in graph["edges"]:
        preds[b].append(a)
    d: dict = {}

    def depth(i):
        if i not in d:
            d[i] = 1 + max((depth(p) for p in preds[i]), default=0)
        return d[i]
    for n in graph["nodes"]:
        depth(n["id"])
    return d, max(d.values()) if d else 0


def score_bundle(bundle: dict, loss_kind: str, loss_n: int, window: int = 50,
                 precisions=(INT8, FP8, BF16, FP16, FP32)) -> dict:
    """{op: {precision: omega}} for every adjustable op of a ProfileBundle dict
    over the extended ladder (the reference's score_all restricted to INT8 / FP16
    / FP32 gives the same numbers for those rungs)."""
    stats = reduce_stats(bundle.get("tensor_stats", []), window)
    d, d_l = depths(bundle["graph"])
    g = loss_gamma(loss_kind, loss_n)
    out = {}
    for n in bundle["graph"]["nodes"]:
        if n["kind"] != "adjustable":
            continue
        out[n["id"]] = {p: omega(n["id"], d[n["id"]], bool(n["has_weight"]), p, d_l, g, stats)
                        for p in precisions}
    return out
