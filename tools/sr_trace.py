import collections, sys, time
sys.path.insert(0, '.')
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2407_02327_b200 import ops
for n in (1 << 20, 1 << 24):
    x = torch.randn(n, device="cuda")
    sc = torch.tensor([0.01, 1.0], device="cuda")
    ops.quantize_sr(x, sc, 7); torch.cuda.synchronize()
    t0 = time.perf_counter(); ops.quantize_sr(x, sc, 7); torch.cuda.synchronize(); t1 = time.perf_counter()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        ops.quantize_sr(x, sc, 7); torch.cuda.synchronize()
    print("n", n, "wall us", (t1 - t0) * 1e6)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            print(f"  {e.time_range.end - e.time_range.start:9.1f} us  {e.name[:80]}")
