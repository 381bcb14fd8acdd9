"""Stream-K scheduling of the tcgen05 GEMM (csrc/gemm.cu, EpiParams::streamk):
the tiles x k-blocks space cut evenly over the SMs, partial tiles fixed up
through the workspace (or reduce-added when the output accumulates).  INT8 is
bit-exact against the tile schedule (int32 partial sums are exact); FP16 /
accumulating FP32 agree to FP32 summation-order noise."""
import pytest
import torch

from paper_2407_02327_b200 import ops

pytestmark = pytest.mark.gpu

SHAPES = [(4096, 768, 768), (4096, 768, 3072), (4096, 3072, 768), (333, 520, 1024), (128, 256, 64),
          (1000, 1024, 4096)]


def _both(fn):
    out = {}
    try:
        for mode in (-1, 1, 1):  # twice with stream-K: the per-tile flags must reset
            ops.set_streamk(mode)
            out.setdefault(mode, []).append(fn())
            torch.cuda.synchronize()
    finally:
        ops.set_streamk(-1)
    return out[-1][0], out[1][0], out[1][1]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_streamk_int8_bit_exact(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda", generator=g)
    sa = torch.tensor([0.01], device="cuda")
    sb = torch.rand(N, device="cuda", generator=g) * 0.01
    bias = torch.randn(N, device="cuda", generator=g)
    for dt in (torch.float32, torch.float16):
        ref, y1, y2 = _both(lambda: ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=dt))
        assert torch.equal(y1, ref) and torch.equal(y2, ref), f"INT8 stream-K {M}x{N}x{K} {dt}"


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("b_mn", [False, True])
def test_streamk_f16(M, N, K, b_mn):
    g = torch.Generator(device="cuda").manual_seed(7 + M + K)
    a = torch.randn(M, K, device="cuda", generator=g).half()
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda", generator=g).half()
    bias = torch.randn(N, device="cuda", generator=g)
    for dt in (torch.float32, torch.float16):
        ref, y1, y2 = _both(lambda: ops.gemm_f16(a, b, out_dtype=dt, bias=bias, b_mn=b_mn))
        scale = ref.float().abs().max().item()
        tol = 1e-5 if dt == torch.float32 else 2e-3
        for y in (y1, y2):
            assert (y.float() - ref.float()).abs().max().item() <= tol * scale
        assert torch.equal(y1, y2), "stream-K is deterministic"


@pytest.mark.parametrize("M,N,K", [(2304, 768, 4096), (768, 3072, 4096), (4096, 768, 2304), (200, 136, 520)])
def test_streamk_accumulate(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.randn(K, M, device="cuda", generator=g).half()  # wgrad-like: both MN-major
    b = torch.randn(K, N, device="cuda", generator=g).half()
    base = torch.randn(M, N, device="cuda", generator=g)

    def run():
        out = base.clone()
        ops.gemm_f16(a, b, out=out, accumulate=True, a_mn=True, b_mn=True)
        return out
    ref, y1, y2 = _both(run)
    want = base.double() + a.double().t() @ b.double()
    scale = want.abs().max().item()
    for y in (ref, y1, y2):
        assert (y.double() - want).abs().max().item() <= 1e-5 * scale


def _dual_pair(fn):
    try:
        ops.set_dual_issue(False)
        ref = fn()
        ops.set_dual_issue(True)
        got = fn()
        torch.cuda.synchronize()
    finally:
        ops.set_dual_issue(True)
    return ref, got


@pytest.mark.parametrize("M,N,K", [(4096, 768, 768), (4096, 768, 3072), (1000, 768, 528), (4096, 768, 512)])
def test_dual_issue_int8_bit_exact(M, N, K):
    """Two MMA issuers splitting the k-blocks into two accumulators (kLay bit
    11): int32 partial sums are exact, so the INT8 output is bit-identical."""
    g = torch.Generator(device="cuda").manual_seed(N + K)
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda", generator=g)
    sa = torch.tensor([0.02], device="cuda")
    sb = torch.rand(N, device="cuda", generator=g) * 0.01
    bias = torch.randn(N, device="cuda", generator=g)
    for dt in (torch.float32, torch.float16):
        ref, got = _dual_pair(lambda: ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=dt))
        assert torch.equal(ref, got)


@pytest.mark.parametrize("M,N,K,lay", [(4096, 768, 768, 0), (4096, 768, 2304, 2), (4096, 768, 3072, 2),
                                       (2304, 768, 4096, 3), (768, 768, 4096, 3)])
def test_dual_issue_f16(M, N, K, lay):
    g = torch.Generator(device="cuda").manual_seed(M + 3 * K)
    a = torch.randn((K, M) if lay == 3 else (M, K), device="cuda", generator=g).half()
    b = torch.randn((K, N) if lay & 2 else (N, K), device="cuda", generator=g).half()
    acc = lay != 0
    base = torch.randn(M, N, device="cuda", generator=g)

    def run():
        out = base.clone() if acc else torch.empty(M, N, device="cuda")
        ops.gemm_f16(a, b, out=out, accumulate=acc, a_mn=lay == 3, b_mn=bool(lay & 2))
        return out
    ref, got = _dual_pair(run)
    A = a.double().t() if lay == 3 else a.double()
    B = b.double() if lay & 2 else b.double().t()
    want = (base.double() if acc else 0) + A @ B
    scale = want.abs().max().item()
    for y in (ref, got):
        assert (y.double() - want).abs().max().item() <= 1e-5 * scale
