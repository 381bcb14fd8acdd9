import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops, _lib
from tools.bench_bwd_gemm import timeit
for (M, N, K) in [(4096, 2304, 768), (4096, 3072, 768), (4096, 768, 3072), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").half(); b = torch.randn(N, K, device="cuda").half()
    out = torch.empty(M, N, device="cuda"); out16 = torch.empty(M, N, device="cuda").half()
    r = {}
    for dbg in (0, 1):
        _lib.call("qsync_gemm_debug_epilogue", dbg)
        for cta in (1, 2):
            ops.force_cta(cta)
            r[(dbg, cta, 'f32')] = timeit(lambda: ops.gemm_f16(a, b, out=out))
            r[(dbg, cta, 'f16')] = timeit(lambda: ops.gemm_f16(a, b, out=out16))
        ops.force_cta(0)
    _lib.call("qsync_gemm_debug_epilogue", 0)
    print(M, N, K, " ".join(f"{k}:{v:.1f}" for k, v in r.items()), flush=True)
