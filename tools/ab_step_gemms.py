"""A/B timing of the exact GEMM configurations of one BERT step (run once per library)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops
from tools.bench_bwd_gemm import timeit
T, H, F = 4096, 768, 3072
tot = 0.0
rows = []
for (M, N, K) in [(T, 3 * H, H), (T, H, H), (T, F, H), (T, H, F)]:
    x = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    sa = torch.tensor([0.01], device="cuda"); sb = torch.rand(N, device="cuda"); bias = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    t8 = timeit(lambda: ops.gemm_s8(x, w, sa, sb, bias, out=out))
    xh = torch.randn(M, K, device="cuda").half(); wh = torch.randn(N, K, device="cuda").half()
    o16 = torch.empty(M, N, device="cuda").half()
    t16 = timeit(lambda: ops.gemm_f16(xh, wh, bias=bias, out=o16))
    dy = torch.randn(M, N, device="cuda").half(); wt = torch.randn(K, N, device="cuda").half()
    dx = torch.empty(M, K, device="cuda")
    tdg = timeit(lambda: ops.gemm_f16(dy, wt, out=dx))
    dyt = torch.randn(N, M, device="cuda").half(); xt = torch.randn(K, M, device="cuda").half()
    mg = torch.zeros(N, K, device="cuda"); s = torch.tensor([0.5], device="cuda")
    twg = timeit(lambda: ops.gemm_f16(dyt, xt, alpha_dev=s, out=mg, accumulate=True))
    rows.append((M, N, K, t8, t16, tdg, twg))
    tot += 6 * (t8 + t16) / 2 + 6 * (tdg + twg) * 2  # 6 INT8 + 6 FP16 layers; bwd for all 12
for r in rows:
    print("%5d %5d %5d  int8-fwd %6.1f  f16-fwd %6.1f  dgrad %6.1f  wgrad %6.1f" % r)
print(f"GEMM time per step (mixed plan) ~ {tot/1e3:.3f} ms  lib={ops._lib.LIB_PATH}")
