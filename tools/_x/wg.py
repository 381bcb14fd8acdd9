import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2407_02327_b200 import ops
from tools.gemm_overhead import graph_time_us
T, H, F = 4096, 768, 3072
for nm, (M, N) in {"qkv": (3 * H, H), "o": (H, H), "ff1": (F, H), "ff2": (H, F)}.items():
    a = torch.randn(T, M, device="cuda").half()
    b = torch.randn(T, N, device="cuda").half()
    out = torch.zeros(M, N, device="cuda")
    t = graph_time_us(lambda: ops.gemm_f16(a, b, out=out, accumulate=True, a_mn=True, b_mn=True), n=10)
    print(os.environ.get("QSYNC_B200_LIB", "")[-8:], nm, f"{t:.1f} us", flush=True)
