"""Generate tests/golden/golden.json from the UNMODIFIED reference library.

Run in the builder container (where /root/reference exists):
    make -f oracle/Makefile && python tests/golden/make_golden.py
The reference is compiled from /root/reference/proj/src into
oracle/_ref/libqsync_ref.so (oracle/Makefile); every value below is produced by
the reference's own stochastic_round / stochastic_round_float / sigma / omega /
reduce_stats / score_all code.  The GPU box never reads /root/reference: tests
use this committed JSON.
"""
from __future__ import annotations

import base64
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.cpu_ref import RefLib  # noqa: E402

DEMO = "/root/reference/proj/tests/fixtures/demo_bundle.json"


def b64(a: np.ndarray) -> str:
    return base64.b64encode(np.ascontiguousarray(a).tobytes()).decode()


def main() -> None:
    r = RefLib()
    g: dict = {"generator": "tests/golden/make_golden.py over oracle/_ref/libqsync_ref.so"}

    # RNG: std::mt19937_64 draws (rng.hpp:12-14 consumes these).
    g["mt64"] = {str(s): [str(v) for v in r.mt64_draws(s, 8)] for s in (1, 7, 42, 5489)}
    g["mt64_tail"] = {"seed": 99, "offset": 1_000_000 - 4,
                      "draws": [str(v) for v in r.mt64_draws(99, 1_000_004)[-8:]]}

    # G1: x_i = 2*u(mt64(1)) - 1, n = 2^20, q = absmax/127, seed 7.
    x = 2.0 * r.uniform01(1, 1 << 20) - 1.0
    q = float(np.abs(x).max() / 127.0)
    rounded, _ = r.stochastic_round(x, q, 0.0, 7)
    g["G1"] = {"n": 1 << 20, "data_seed": 1, "sr_seed": 7, "q": q.hex(),
               "sum": int(rounded.sum()), "sumsq": int((rounded * rounded).sum()),
               "min": int(rounded.min()), "max": int(rounded.max()),
               "first16": rounded[:16].tolist(),
               "sha256_int8": hashlib.sha256(rounded.astype(np.int8).tobytes()).hexdigest(),
               "count_128": int((np.abs(rounded) > 127).sum())}
    # G2, G3.
    x2 = r.uniform01(5, 8)
    g["G2"] = {"x": [v.hex() for v in x2], "q": 0.01, "seed": 42,
               "rounded": r.stochastic_round(x2, 0.01, 0.0, 42)[0].tolist()}
    g["G3"] = {"x": [v.hex() for v in x[:8]], "e": 0, "k": 9, "seed": 11,
               "out": [v.hex() for v in r.stochastic_round_float(x[:8], 0, 9, 11)]}

    # Full small SR vectors (base64) incl. nonzero zero-point and negative values.
    cases = []
    for (n, dseed, q, zp, seed) in [(5000, 3, 0.037, 0.0, 11), (4099, 4, 0.25, 0.5, 123),
                                    (1, 5, 1e-3, -0.2, 9), (312 * 3 + 1, 6, 0.5, 0.0, 2024)]:
        xs = (r.uniform01(dseed, n) - 0.5) * 7.0
        rr, dd = r.stochastic_round(xs, q, zp, seed)
        cases.append({"n": n, "data_seed": dseed, "q": q, "zp": zp, "seed": seed,
                      "x": b64(xs), "rounded": b64(rr), "deq": b64(dd)})
    g["sr_cases"] = cases
    fcases = []
    for (n, dseed, e, k, seed) in [(3000, 8, 0, 9, 13), (777, 9, 3, 7, 5), (64, 10, -4, 9, 1)]:
        xs = r.uniform01(dseed, n) * 2.0 ** e
        fcases.append({"n": n, "data_seed": dseed, "e": e, "k": k, "seed": seed, "x": b64(xs),
                       "out": b64(r.stochastic_round_float(xs, e, k, seed))})
    g["srf_cases"] = fcases

    # sigma / omega on random stats (indicator.cpp:65-132), all-present mask.
    rng = np.random.default_rng(7)
    kat = []
    for i in range(40):
        v = np.array([rng.uniform(0.1, 50), rng.uniform(0.1, 50), rng.uniform(0.01, 5),
                      rng.uniform(0.0, 5), rng.integers(1, 10**6), rng.integers(1, 10**6),
                      rng.integers(1, 10**6), rng.uniform(1e-4, 0.1), rng.uniform(1e-4, 0.1),
                      rng.integers(-8, 4), rng.integers(-8, 4), rng.integers(-12, 2)], np.float64)
        mask = 0xFFF if i % 3 else 0xFFF & ~(1 << 3)  # sometimes no grad-hat norm
        row = {"v": [float(t) for t in v], "mask": mask}
        for p in (0, 1, 2):
            for pf in (0, 1):
                row[f"fwd_{p}_{pf}"] = r.sigma(0, v, mask, p, pf).hex()
                row[f"bwd_{p}_{pf}"] = r.sigma(1, v, mask, p, pf).hex()
        depth = int(rng.integers(1, 12))
        d_l = depth + int(rng.integers(0, 6))
        lk = int(rng.integers(0, 3))
        ln = int(rng.integers(1, 64))
        row.update({"depth": depth, "d_l": d_l, "loss_kind": lk, "loss_n": ln,
                    "has_weight": int(i % 4 != 0)})
        for p in (0, 1, 2):
            row[f"omega_{p}"] = r.omega(v, mask, row["has_weight"], depth, d_l, lk, ln, p).hex()
        kat.append(row)
    g["indicator_kat"] = kat

    # reduce_stats window semantics (profile.cpp:134-162: first min(W, n) snapshots).
    snaps = rng.uniform(0, 10, size=(7, 12))
    masks = np.array([0xFFF, 0x0FF, 0xFFF, 0xF0F, 0xFFF, 0x00F, 0xFFF], np.uint32)
    red = []
    for w in (1, 3, 7, 50):
        out, om = r.reduce_stats(snaps, masks, w)
        red.append({"window": w, "out": [float(t).hex() for t in out], "mask": om})
    g["reduce_stats"] = {"snaps": snaps.tolist(), "masks": masks.tolist(), "cases": red}

    # score_all on the reference's demo bundle (mse_mean, N = 8).
    if os.path.exists(DEMO):
        g["demo_omega_mse8"] = [[op, p, w.hex()] for op, p, w in r.score_bundle(DEMO, 0, 8)]

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
