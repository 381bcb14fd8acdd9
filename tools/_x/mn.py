import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2407_02327_b200 import ops
from tools.gemm_overhead import graph_time_us
for (M, N, K) in [(2304, 768, 4096), (3072, 768, 4096), (768, 3072, 4096), (8192, 8192, 8192)]:
    res = {}
    for lay in (0, 2, 3):
        a = torch.randn((K, M) if lay == 3 else (M, K), device="cuda").half()
        b = torch.randn((K, N) if lay & 2 else (N, K), device="cuda").half()
        for acc in (False, True):
            out = torch.zeros(M, N, device="cuda")
            f = lambda: ops.gemm_f16(a, b, out=out, accumulate=acc, a_mn=lay == 3, b_mn=bool(lay & 2))
            t = graph_time_us(f, n=10)
            res[(lay, acc)] = t
    print(M, N, K, " ".join(f"lay{l}{'acc' if ac else ''}={t:.1f}" for (l, ac), t in res.items()), flush=True)
