"""CPU tests: pin the oracle (oracle/cpu_ref.c) to the reference's golden vectors
and to the compiled reference itself; check the C ABI library loads and exports
every declared symbol.  No GPU needed."""
import base64
import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _arr(s, dt):
    return np.frombuffer(base64.b64decode(s), dtype=dt)


def test_mt64_stream_matches_std(golden, cpuref):
    for seed, draws in golden["mt64"].items():
        assert cpuref.mt64_draws(int(seed), 8).tolist() == [int(d) for d in draws]
    t = golden["mt64_tail"]
    got = cpuref.mt64_draws(t["seed"], t["offset"] + 8)[-8:]
    assert got.tolist() == [int(d) for d in t["draws"]]


def test_baseline_rng_check(golden):
    # BASELINE.md sec. G lists {11788048577503494824, 13930160852258120406} for
    # mt19937_64(42); std::mt19937_64 emits them in the order below.
    assert [int(v) for v in golden["mt64"]["42"][:2]] == [13930160852258120406,
                                                          11788048577503494824]


def test_G1_golden(golden, cpuref):
    g = golden["G1"]
    u = cpuref.mt64_draws(1, g["n"])
    x = 2.0 * ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0
    q = float(np.abs(x).max() / 127.0)
    assert q == float.fromhex(g["q"])
    r, _ = cpuref.stochastic_round(x, q, 0.0, g["sr_seed"])
    assert int(r.sum()) == g["sum"] == -8938
    assert int((r * r).sum()) == g["sumsq"] == 5638075870
    assert int(r.min()) == g["min"] == -127 and int(r.max()) == g["max"] == 127
    assert r[:16].tolist() == g["first16"]
    assert hashlib.sha256(r.astype(np.int8).tobytes()).hexdigest() == g["sha256_int8"]


def test_G2_G3_golden(golden, cpuref):
    g2 = golden["G2"]
    x2 = np.array([float.fromhex(v) for v in g2["x"]])
    assert cpuref.stochastic_round(x2, g2["q"], 0.0, g2["seed"])[0].tolist() == g2["rounded"]
    assert g2["rounded"] == [67, 4, 22, 68, 9, 10, 13, 69]
    g3 = golden["G3"]
    x3 = np.array([float.fromhex(v) for v in g3["x"]])
    out = cpuref.stochastic_round_float(x3, g3["e"], g3["k"], g3["seed"])
    assert [v.hex() for v in out] == g3["out"]


def test_sr_cases_bit_exact(golden, cpuref):
    for c in golden["sr_cases"]:
        x = _arr(c["x"], np.float64)
        r, d = cpuref.stochastic_round(x, c["q"], c["zp"], c["seed"])
        assert np.array_equal(r, _arr(c["rounded"], np.int64))
        assert np.array_equal(d.view(np.uint64), _arr(c["deq"], np.uint64))
    for c in golden["srf_cases"]:
        x = _arr(c["x"], np.float64)
        d = cpuref.stochastic_round_float(x, c["e"], c["k"], c["seed"])
        assert np.array_equal(d.view(np.uint64), _arr(c["out"], np.uint64))


def test_sr_domain_errors(cpuref):
    with pytest.raises(ValueError, match="scaling factor"):
        cpuref.stochastic_round(np.zeros(3), 0.0, 0.0, 1)
    with pytest.raises(ValueError, match="mantissa"):
        cpuref.stochastic_round_float(np.zeros(3), 0, 0, 1)


def test_on_grid_values_untouched(cpuref):
    # test_indicator.cpp:206-216
    x = np.array([0.25 * i + 0.5 for i in range(-8, 9)])
    r, d = cpuref.stochastic_round(x, 0.25, 0.5, 123)
    assert r.tolist() == list(range(-8, 9))
    assert np.array_equal(d, x)


def test_oracle_matches_reference_library(reflib, cpuref):
    rng = np.random.default_rng(0)
    for n, q, zp, seed in [(10000, 0.013, 0.0, 5), (3331, 0.5, -1.25, 77)]:
        x = rng.normal(size=n) * 3
        r0, d0 = reflib.stochastic_round(x, q, zp, seed)
        r1, d1 = cpuref.stochastic_round(x, q, zp, seed)
        assert np.array_equal(r0, r1) and np.array_equal(d0, d1)


def test_f16_cast_matches_numpy(cpuref):
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(size=20000).astype(np.float32) * 10.0 ** rng.integers(-9, 6, 20000),
                        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 1e-8, 2.0 ** -25,
                                  2.0 ** -24, 3 * 2.0 ** -26, np.inf, -np.inf], np.float32)])
    x = x.astype(np.float32)
    ours = cpuref.cast_f32_f16(x)
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16)
    assert np.array_equal(ours.view(np.uint16), ref.view(np.uint16))


def test_quantize_semantics(cpuref):
    x = np.array([[0.0, 1.0, -2.0, 0.5], [127.0, -127.0, 63.5, 64.5]], np.float32)
    q, s = cpuref.quantize_per_tensor(x)
    assert s == np.float32(127.0) / np.float32(127.0)
    assert q.tolist() == [[0, 1, -2, 0], [127, -127, 64, 64]]  # rint: ties to even
    q0, s0 = cpuref.quantize_per_tensor(np.zeros((2, 3), np.float32))
    assert s0 == 1.0 and not q0.any()
    w = np.array([[1.0, -3.0], [0.0, 0.0], [2.0, 4.0]], np.float32)
    qw, sw = cpuref.quantize_per_channel(w)
    assert sw.tolist() == [np.float32(3.0) / np.float32(127.0), 1.0, np.float32(4.0) / np.float32(127.0)]
    assert qw[1].tolist() == [0, 0] and qw[0, 1] == -127 and qw[2, 1] == 127


def test_int_gemm_and_epilogue(cpuref):
    rng = np.random.default_rng(2)
    a = rng.integers(-127, 128, size=(37, 48), dtype=np.int8)
    b = rng.integers(-127, 128, size=(29, 48), dtype=np.int8)
    c = cpuref.gemm_s8_tn(a, b)
    assert np.array_equal(c, a.astype(np.int64) @ b.astype(np.int64).T)
    sw = rng.uniform(0.001, 0.1, 29).astype(np.float32)
    bias = rng.normal(size=29).astype(np.float32)
    y = cpuref.dequant_epilogue(c, np.float32(0.02), sw, bias)
    want = (c.astype(np.float32) * (np.float32(0.02) * sw)[None, :]).astype(np.float32) + bias
    assert np.array_equal(y, want.astype(np.float32))


def test_qlinear_oracle_consistent(cpuref):
    rng = np.random.default_rng(3)
    M, N, K = 16, 24, 32
    x = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.normal(size=N).astype(np.float32)
    dy = rng.normal(size=(M, N)).astype(np.float32)
    o = cpuref.qlinear_int8(x, w, b, dy)
    y_fp = x @ w.T + b
    assert np.abs(o["y"] - y_fp).max() < 0.05 * np.abs(y_fp).max()
    dx_fp = dy @ w
    assert np.allclose(o["dx"], dx_fp, rtol=1e-2, atol=1e-2)
    assert np.allclose(o["db"], dy.sum(0), rtol=1e-5, atol=1e-5)


def test_tensor_stats_oracle(cpuref):
    x = np.array([3.0, -4.0, 0.5], np.float32)
    s = cpuref.tensor_stats(x)
    assert s[0] == 25.25 and s[1] == 4.0 and s[2] == float(np.float32(4.0) / np.float32(127.0))
    assert s[3] == 2.0 and s[4] == 3.0


def test_indicator_kat_reference(golden, reflib):
    # The reference's sigma/omega reproduce the committed KATs (pins the fixture).
    for row in golden["indicator_kat"][:8]:
        v = np.array(row["v"])
        assert reflib.sigma(0, v, row["mask"], 0, 0).hex() == row["fwd_0_0"]
        assert reflib.omega(v, row["mask"], row["has_weight"], row["depth"], row["d_l"],
                            row["loss_kind"], row["loss_n"], 1).hex() == row["omega_1"]


def test_demo_bundle_omega(golden):
    rows = {(op, p): float.fromhex(w) for op, p, w in golden["demo_omega_mse8"]}
    assert rows[("conv1", "FP16")] == 84.700520833333329
    assert rows[("conv2", "FP16")] == 51.796875
    assert rows[("conv3", "FP16")] == 9.5182291666666661


# ---------------------------------------------------------------- C ABI library

def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "qsync_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|size_t|unsigned long long)\s+(qsync_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2407_02327_b200 import _lib
    L = _lib.lib()
    syms = _declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, s


def test_python_signatures_match_header_arity():
    """Every C entry's ctypes argtypes (the Python mirror) has the header's arity,
    so a caller can never pass a shifted argument list."""
    from paper_2407_02327_b200 import _lib
    src = open(os.path.join(ROOT, "include", "qsync_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    protos = re.findall(r"^\s*(?:int|const char\*|size_t|unsigned long long)\s+(qsync_\w+)\(([^)]*)\);", src,
                        re.M | re.S)
    assert len(protos) >= 40
    for name, params in protos:
        params = params.strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert len(_lib.SIGNATURES[name]) == n, (name, n, len(_lib.SIGNATURES[name]))


def test_library_error_names_mirror_error_kinds():
    from paper_2407_02327_b200 import _lib
    L = _lib.lib()
    assert [L.qsync_status_name(i + 1).decode() for i in range(14)] == _lib.ERROR_KINDS
    assert L.qsync_abi_version() == 1


def test_mt_jump_ahead_polynomials_host():
    """GF(2) jump-ahead identity vs a scalar mt19937_64 (host code of the .so)."""
    from paper_2407_02327_b200 import _lib
    _lib.check(_lib.lib().qsync_mt_jump_selftest())


def test_ops_refuse_cpu_tensors():
    import torch

    from paper_2407_02327_b200 import QsyncError, ops
    with pytest.raises(QsyncError) as e:
        ops.absmax(torch.zeros(4))
    assert e.value.kind == "validation"
