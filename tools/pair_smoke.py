import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2407_02327_b200 import ops
from oracle.cpu_ref import CpuRef
ref = CpuRef()
for (M, N, K) in [(256, 256, 128), (512, 256, 256), (300, 200, 64)]:
    rng = np.random.default_rng(1)
    a = rng.integers(-127, 128, size=(M, K), dtype=np.int8); b = rng.integers(-127, 128, size=(N, K), dtype=np.int8)
    ops.force_cta(2); ops.force_tile_n(256 if N >= 256 else 128)
    ci, _ = ops.gemm_s8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), out_i32=True, out_f32=False)
    torch.cuda.synchronize()
    ok = np.array_equal(ci.cpu().numpy(), ref.gemm_s8_tn(a, b))
    print(M, N, K, "pair int8 exact:", ok, flush=True)
    if not ok:
        d = ci.cpu().numpy() - ref.gemm_s8_tn(a, b); print("mismatch rows", np.unique(np.nonzero(d)[0])[:20], "cols", np.unique(np.nonzero(d)[1])[:20])
