"""GPU parity tests: every kernel through the C ABI vs the oracle on identical
inputs.  Integer / byte / index results bit-exact; FP GEMMs within the stated
tolerance."""
import base64

import numpy as np
import pytest
import torch

from paper_2407_02327_b200 import QsyncError, ops

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _arr(s, dt):
    return np.frombuffer(base64.b64decode(s), dtype=dt)


def _t(a):
    return torch.from_numpy(np.array(a, copy=True)).to(DEV)


def _np(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _data(shape, seed, dist="uniform"):
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        return rng.uniform(-1, 1, size=shape).astype(np.float32)
    x = rng.normal(size=shape).astype(np.float32)
    flat = x.reshape(-1)
    if flat.size == 0:
        return x
    idx = rng.choice(flat.size, size=max(1, flat.size // 1000), replace=False)
    flat[idx] *= 100.0  # outliers stress absmax
    return x


# ------------------------------------------------------------------ K1 / K2 / K3
SHAPES = [(1, 1), (7, 13), (64, 1024), (129, 255), (4096, 768), (33, 4096), (1000, 1001)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dist", ["uniform", "normal"])
def test_quantize_per_tensor_bit_exact(shape, dist, cpuref):
    x = _data(shape, 11, dist)
    q_ref, s_ref = cpuref.quantize_per_tensor(x)
    q, scale, qt = ops.quantize_per_tensor(_t(x), transposed_f16=True)
    assert np.float32(_np(scale)[0]) == s_ref
    assert _np(scale)[1] == cpuref.absmax(x)
    assert np.array_equal(_np(q), q_ref)
    qt = _np(qt)
    rows = shape[0]
    assert qt.shape == (shape[1], (rows + 7) // 8 * 8)  # K-pitch padded to 8 for TMA
    assert np.array_equal(qt[:, :rows].astype(np.int32), q_ref.T.astype(np.int32))
    assert not qt[:, rows:].any()
    q2, scale2, _ = ops.quantize_per_tensor(_t(x))
    assert np.array_equal(_np(q2), q_ref) and _np(scale2)[0] == s_ref
    # the 1-byte transposed copy an INT8 op keeps for backward, and its exact FP16 view
    q3, _, qt8 = ops.quantize_per_tensor(_t(x), transposed_i8=True)
    assert np.array_equal(_np(q3), q_ref)
    qt8n = _np(qt8)
    assert qt8n.dtype == np.int8 and np.array_equal(qt8n[:, :rows], q_ref.T) and not qt8n[:, rows:].any()
    assert np.array_equal(_np(ops.cast(qt8, torch.float16)).astype(np.int32), qt8n.astype(np.int32))


def test_quantize_edge_cases(cpuref):
    # empty, all-zero, misaligned base pointer (vector path disabled), 16-bit inputs
    q, s, _ = ops.quantize_per_tensor(torch.empty((0, 5), device=DEV))
    assert q.numel() == 0 and _np(s)[0] == 1.0
    q, s, _ = ops.quantize_per_tensor(torch.zeros((3, 7), device=DEV))
    assert not _np(q).any() and _np(s)[0] == 1.0
    x = _data((1, 4099), 5)
    xt = _t(x)[:, 1:].contiguous()  # fresh buffer
    base = torch.empty(4100, device=DEV)
    base[1:].copy_(_t(x).reshape(-1)[:4099])
    mis = base[1:]  # 4-byte misaligned view, contiguous
    q_ref, s_ref = cpuref.quantize_per_tensor(x.reshape(-1)[:4099])
    q, s, _ = ops.quantize_per_tensor(mis)
    assert np.array_equal(_np(q), q_ref) and _np(s)[0] == s_ref
    del xt
    for dt in (torch.float16, torch.bfloat16):
        xh = torch.from_numpy(_data((257, 129), 6)).to(DEV).to(dt)
        q_ref, s_ref = cpuref.quantize_per_tensor(xh.float().cpu().numpy())
        q, s, _ = ops.quantize_per_tensor(xh)
        assert np.array_equal(_np(q), q_ref) and _np(s)[0] == s_ref


@pytest.mark.parametrize("shape", [(1, 1), (768, 768), (3072, 768), (5, 4097), (2304, 3)])
def test_quantize_per_channel_bit_exact(shape, cpuref):
    w = _data(shape, 3, "normal")
    w[min(1, shape[0] - 1)] = 0.0
    q_ref, s_ref = cpuref.quantize_per_channel(w)
    q, s, wt = ops.quantize_per_channel(_t(w), transposed_f16=True)
    assert np.array_equal(_np(s), s_ref)
    assert np.array_equal(_np(q), q_ref)
    assert np.array_equal(_np(wt).view(np.uint16), cpuref.cast_f32_f16(w).T.view(np.uint16))


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 65536, 1 << 20, 3_000_001])
def test_absmax_and_dequant(n, cpuref):
    x = _data((n,), 21, "normal")
    a = ops.absmax(_t(x))
    assert _np(a)[0] == (cpuref.absmax(x) if n else 0.0)
    q_ref, s_ref = cpuref.quantize_per_tensor(x)
    s = torch.tensor([s_ref], device=DEV)
    q = ops.quantize_with_scale(_t(x), s)
    assert np.array_equal(_np(q), q_ref)
    d = ops.dequantize_per_tensor(_t(q_ref), s)
    assert np.array_equal(_np(d), cpuref.dequantize_per_tensor(q_ref, s_ref))


def test_absmax_rows_and_dequant_per_channel(cpuref):
    w = _data((300, 517), 4, "normal")
    am = ops.absmax_rows(_t(w))
    assert np.array_equal(_np(am), np.abs(w).max(1))
    q_ref, s_ref = cpuref.quantize_per_channel(w)
    d = ops.dequantize_per_channel(_t(q_ref), _t(s_ref))
    assert np.array_equal(_np(d), cpuref.dequantize_per_channel(q_ref, s_ref))


# ------------------------------------------------------------------ K4
@pytest.mark.parametrize("n", [1, 7, 8, 1000003])
def test_casts_bit_exact(n, cpuref):
    x = _data((n,), 8, "normal") * 1000
    h = ops.cast(_t(x), torch.float16)
    assert np.array_equal(_np(h).view(np.uint16), cpuref.cast_f32_f16(x).view(np.uint16))
    b = ops.cast(_t(x), torch.bfloat16)
    assert torch.equal(b.cpu(), torch.from_numpy(x).to(torch.bfloat16))
    back = ops.cast(h, torch.float32)
    assert np.array_equal(_np(back), cpuref.cast_f32_f16(x).astype(np.float32))


@pytest.mark.parametrize("shape", [(1, 1), (4096, 768), (130, 33), (64, 3072)])
def test_cast_transpose(shape, cpuref):
    x = _data(shape, 9, "normal")
    o, t, s = ops.cast_transpose(_t(x), True, True, True)
    h = cpuref.cast_f32_f16(x)
    assert np.array_equal(_np(o).view(np.uint16), h.view(np.uint16))
    t = _np(t)
    assert np.array_equal(t[:, :shape[0]].view(np.uint16), h.T.view(np.uint16))
    assert not t[:, shape[0]:].astype(np.float32).any()
    np.testing.assert_allclose(_np(s), x.astype(np.float64).sum(0), rtol=1e-5, atol=1e-3)


# ------------------------------------------------------------------ K5
@pytest.mark.parametrize("n", [1, 1000, 4096 * 768, 10_000_019])
def test_tensor_stats(n, cpuref):
    x = _data((n,), 31, "normal")
    st = _np(ops.tensor_stats(_t(x)))
    ref = cpuref.tensor_stats(x)
    assert st[1] == ref[1] and st[2] == ref[2] and st[3] == ref[3] and st[4] == ref[4]
    # FP64 accumulation; only the summation order differs from the oracle
    assert abs(st[0] - ref[0]) <= 1e-10 * ref[0]
    sh = _np(ops.tensor_stats(_t(x).half()))
    refh = cpuref.tensor_stats(x.astype(np.float16).astype(np.float32))
    assert sh[1] == refh[1] and abs(sh[0] - refh[0]) <= 1e-10 * refh[0]


# ------------------------------------------------------------------ K9 SR
def test_mt64_draws_with_offsets(golden, cpuref):
    for seed, draws in golden["mt64"].items():
        d = _np(ops.mt64_draws(int(seed), 8)).view(np.uint64)
        assert d.tolist() == [int(v) for v in draws]
    ref = cpuref.mt64_draws(99, 2_000_000)
    for off, n in [(0, 2_000_000), (1, 1000), (311, 313), (312, 624), (123457, 500000)]:
        d = _np(ops.mt64_draws(99, n, offset=off)).view(np.uint64)
        assert np.array_equal(d, ref[off:off + n]), (off, n)


def test_stochastic_round_golden(golden):
    g = golden["G1"]
    u = _np(ops.mt64_draws(1, g["n"])).view(np.uint64)
    x = 2.0 * ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0
    q = float.fromhex(g["q"])
    r, _ = ops.stochastic_round(_t(x), q, 0.0, g["sr_seed"])
    r = _np(r)
    assert int(r.sum()) == g["sum"] and int((r * r).sum()) == g["sumsq"]
    assert r[:16].tolist() == g["first16"]
    import hashlib
    assert hashlib.sha256(r.astype(np.int8).tobytes()).hexdigest() == g["sha256_int8"]
    g2 = golden["G2"]
    x2 = np.array([float.fromhex(v) for v in g2["x"]])
    assert _np(ops.stochastic_round(_t(x2), g2["q"], 0.0, g2["seed"])[0]).tolist() == g2["rounded"]
    g3 = golden["G3"]
    x3 = np.array([float.fromhex(v) for v in g3["x"]])
    out = _np(ops.stochastic_round_float(_t(x3), g3["e"], g3["k"], g3["seed"]))
    assert [v.hex() for v in out] == g3["out"]


def test_stochastic_round_cases_bit_exact(golden):
    for c in golden["sr_cases"]:
        x = _arr(c["x"], np.float64)
        r, d = ops.stochastic_round(_t(x), c["q"], c["zp"], c["seed"])
        assert np.array_equal(_np(r), _arr(c["rounded"], np.int64))
        assert np.array_equal(_np(d).view(np.uint64), _arr(c["deq"], np.uint64))
    for c in golden["srf_cases"]:
        x = _arr(c["x"], np.float64)
        d = ops.stochastic_round_float(_t(x), c["e"], c["k"], c["seed"])
        assert np.array_equal(_np(d).view(np.uint64), _arr(c["out"], np.uint64))


def test_stochastic_round_domain_error():
    with pytest.raises(QsyncError) as e:
        ops.stochastic_round(torch.zeros(3, dtype=torch.float64, device=DEV), 0.0, 0.0, 1)
    assert e.value.kind == "domain" and "scaling factor" in str(e.value)
    with pytest.raises(QsyncError) as e:
        ops.stochastic_round_float(torch.zeros(3, dtype=torch.float64, device=DEV), 0, 0, 1)
    assert "mantissa" in str(e.value)


@pytest.mark.parametrize("n", [1, 5000, 1 << 20, 3_333_333])
def test_quantize_sr_bit_exact(n, cpuref):
    x = _data((n,), 41, "normal")
    _, s_ref = cpuref.quantize_per_tensor(x)
    q_ref = cpuref.quantize_sr_per_tensor(x, s_ref, 7)
    q = ops.quantize_sr(_t(x), torch.tensor([s_ref], device=DEV), 7)
    assert np.array_equal(_np(q), q_ref)


# ------------------------------------------------------------------ K6 / K7 GEMM
GEMM_SHAPES = [(128, 256, 128), (64, 1024, 1024), (200, 300, 64), (1, 16, 16), (4096, 768, 768),
               (257, 129, 3072), (512, 2304, 768)]


@pytest.mark.parametrize("cta_bn", [(1, 0), (1, 64), (1, 128), (1, 192), (1, 256), (2, 128), (2, 256), (0, 0)])
@pytest.mark.parametrize("mnk", GEMM_SHAPES)
def test_gemm_s8_int32_bit_exact(mnk, cta_bn, cpuref):
    """int32 accumulators bit-exact for single-CTA tiles and CTA-pair (cta_group::2) tiles."""
    cta, bn = cta_bn
    M, N, K = mnk
    rng = np.random.default_rng(M * 7 + N + K)
    a = rng.integers(-127, 128, size=(M, K), dtype=np.int8)
    b = rng.integers(-127, 128, size=(N, K), dtype=np.int8)
    ops.force_tile_n(bn)
    ops.force_cta(cta)
    try:
        ci, _ = ops.gemm_s8(_t(a), _t(b), out_i32=True, out_f32=False)
    finally:
        ops.force_tile_n(0)
        ops.force_cta(0)
    assert np.array_equal(_np(ci), cpuref.gemm_s8_tn(a, b))


@pytest.mark.parametrize("mnk", [(64, 1024, 1024), (300, 200, 128), (4096, 2304, 768)])
def test_gemm_s8_dequant_epilogue_bit_exact(mnk, cpuref):
    M, N, K = mnk
    rng = np.random.default_rng(5)
    x = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(N, K)) / np.sqrt(K)).astype(np.float32)
    bias = rng.normal(size=N).astype(np.float32)
    xq, sx = cpuref.quantize_per_tensor(x)
    wq, sw = cpuref.quantize_per_channel(w)
    acc = cpuref.gemm_s8_tn(xq, wq)
    y_ref = cpuref.dequant_epilogue(acc, sx, sw, bias)
    ci, y = ops.gemm_s8(_t(xq), _t(wq), torch.tensor([sx], device=DEV), _t(sw), _t(bias),
                        out_i32=True)
    assert np.array_equal(_np(ci), acc)
    assert np.array_equal(_np(y), y_ref)


def test_gemm_s8_rejects_bad_k():
    a = torch.zeros((16, 24), dtype=torch.int8, device=DEV)
    with pytest.raises(QsyncError) as e:
        ops.gemm_s8(a, a, out_i32=True, out_f32=False)
    assert e.value.kind == "domain"


@pytest.mark.parametrize("cta", [1, 2, "bn192"])
@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("mnk", [(128, 128, 64), (64, 1024, 1024), (333, 200, 72),
                                 (4096, 768, 3072), (768, 3072, 4096)])
def test_gemm_f16_within_tolerance(mnk, dt, cta, cpuref):
    M, N, K = mnk
    if cta == "bn192":
        ops.force_tile_n(192)
    else:
        ops.force_cta(cta)
    try:
        _check_f16(M, N, K, dt)
    finally:
        ops.force_cta(0)
        ops.force_tile_n(0)


def _check_f16(M, N, K, dt):
    rng = np.random.default_rng(M + N + K)
    a = torch.from_numpy(rng.normal(size=(M, K)).astype(np.float32)).to(dt)
    b = torch.from_numpy(rng.normal(size=(N, K)).astype(np.float32)).to(dt)
    ref = a.double() @ b.double().T  # exact products of the 16-bit inputs
    c = ops.gemm_f16(a.to(DEV), b.to(DEV), out_dtype=torch.float32, alpha=0.5)
    err = (torch.from_numpy(_np(c)).double() - 0.5 * ref).abs().max().item()
    # FP32 accumulation of K products: tolerance 1e-3 relative to the output scale
    assert err <= 1e-3 * (0.5 * ref).abs().max().item()
    c16 = ops.gemm_f16(a.to(DEV), b.to(DEV), out_dtype=torch.float16)
    rel = ((torch.from_numpy(_np(c16).astype(np.float32)).double() - ref).abs().max()
           / ref.abs().max()).item()
    assert rel <= 1e-2


def test_gemm_f16_bias_alpha_dev_accumulate():
    rng = np.random.default_rng(1)
    M, N, K = 256, 384, 128
    a = torch.from_numpy(rng.normal(size=(M, K)).astype(np.float16)).to(DEV)
    b = torch.from_numpy(rng.normal(size=(N, K)).astype(np.float16)).to(DEV)
    bias = torch.from_numpy(rng.normal(size=N).astype(np.float32)).to(DEV)
    s = torch.tensor([0.25], device=DEV)
    base = torch.ones((M, N), device=DEV)
    ops.gemm_f16(a, b, alpha=2.0, alpha_dev=s, bias=bias, out=base, accumulate=True)
    ref = 0.5 * (a.double() @ b.double().T) + bias.double() + 1.0
    assert (base.double() - ref).abs().max().item() < 1e-3 * ref.abs().max().item()


@pytest.mark.parametrize("cta", [1, 2, "bn192"])
@pytest.mark.parametrize("lay", ["b_mn", "ab_mn"])
@pytest.mark.parametrize("mnk", [(128, 128, 64), (4096, 768, 2304), (2304, 768, 4096), (768, 3072, 300),
                                 (200, 136, 77), (512, 512, 1000)])
def test_gemm_f16_mn_major_operands(mnk, lay, cta):
    """MN-major operands (no transposed copies): dgrad reads W [N_out, K_in] as B,
    wgrad reads dY [M, N_out] and X [M, K_in] as A and B; K need not be padded."""
    M, N, K = mnk
    if lay == "b_mn" and K % 8:
        pytest.skip("K-major A needs K % 8 == 0")
    rng = np.random.default_rng(M + 3 * N + K)
    a = torch.from_numpy(rng.normal(size=(M, K)).astype(np.float32)).half()
    b = torch.from_numpy(rng.normal(size=(N, K)).astype(np.float32)).half()
    ref = a.double() @ b.double().T
    if cta == "bn192":
        ops.force_tile_n(192)
    else:
        ops.force_cta(cta)
    try:
        if lay == "b_mn":
            c = ops.gemm_f16(a.cuda(), b.t().contiguous().cuda(), b_mn=True)
        else:
            c = ops.gemm_f16(a.t().contiguous().cuda(), b.t().contiguous().cuda(), a_mn=True, b_mn=True)
        base = torch.ones(M, N, device=DEV)
        ops.gemm_f16(a.t().contiguous().cuda(), b.t().contiguous().cuda(), a_mn=True, b_mn=True,
                     out=base, accumulate=True, alpha=0.5)
    finally:
        ops.force_cta(0)
        ops.force_tile_n(0)
    err = (torch.from_numpy(_np(c)).double() - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item()
    err2 = (torch.from_numpy(_np(base)).double() - (1.0 + 0.5 * ref)).abs().max().item()
    assert err2 <= 1e-3 * (1.0 + 0.5 * ref).abs().max().item()


def test_sr_rejects_graph_capture_and_streams_are_independent():
    """the SR jump-ahead workspace is per (device, stream) and SR is
    refused inside a CUDA-graph capture (its polynomials come from the host)."""
    import torch

    from paper_2407_02327_b200 import ops
    from paper_2407_02327_b200._lib import QsyncError
    x = torch.rand(1 << 20, device="cuda", dtype=torch.float32)
    sc = torch.tensor([0.01], device="cuda")
    ref = ops.quantize_sr(x, sc, 7)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for s in (s1, s2, s1, s2):  # interleaved on two streams, larger then smaller
        with torch.cuda.stream(s):
            outs.append(ops.quantize_sr(x, sc, 7))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with pytest.raises(QsyncError) as e:
            with torch.cuda.graph(g, stream=s):
                ops.quantize_sr(x, sc, 7)
    assert e.value.kind == "validation"
