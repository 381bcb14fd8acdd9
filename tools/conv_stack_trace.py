"""Kernel breakdown (CUPTI) of the ResNet-50 conv stack fwd+bwd (bench_kernels
--conv's workload): device time per kernel, weighted by how many of the 53
layers share each shape, plus the per-layer top kernels.

    python tools/conv_stack_trace.py [INT8|FP16] [batch]
"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_kernels import resnet50_convs  # noqa: E402
from paper_2407_02327_b200.qconv import qconv2d  # noqa: E402

if os.environ.get("QSB_DGRAD_STRIDED_IMPLICIT"):  # A/B: strided dgrad on the gather lanes
    import paper_2407_02327_b200.ops as _ops
    _ops.implicit_dgrad_ok = lambda C, co, stride=(1, 1): co % 64 == 0 and C % 8 == 0
prec = sys.argv[1] if len(sys.argv) > 1 else "INT8"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
distinct = {}
for c in resnet50_convs(batch):
    distinct.setdefault(c[1:], []).append(c[0])
total = collections.defaultdict(float)
for key, names in distinct.items():
    N, H, W, C, Co, R, st, pd = key
    x = torch.randn(N, H, W, C, device="cuda")
    if prec == "FP16":
        x = x.half()
    x.requires_grad_(C != 3)
    w = (torch.randn(Co, R, R, C, device="cuda") / (R * R * C) ** 0.5).requires_grad_(True)
    b = torch.zeros(Co, device="cuda", requires_grad=True)
    wrt = [t for t in (x, w, b) if t.requires_grad]
    y = qconv2d(x, w, b, (st, st), (pd, pd), prec)
    g = torch.randn_like(y)
    torch.autograd.grad(y, wrt, g)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        y = qconv2d(x, w, b, (st, st), (pd, pd), prec)
        torch.autograd.grad(y, wrt, g)
        torch.cuda.synchronize()
    per = collections.defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.replace("(anonymous namespace)::", "").replace("qsb::", "").split("(")[0][:70]
            per[k] += e.time_range.end - e.time_range.start
    lay = sum(per.values())
    print(f"{names[0]:10s} x{len(names)} C={C:4d}->{Co:4d} R={R} s={st} H={H:3d}: {lay:8.1f} us  " +
          ", ".join(f"{k.split('<')[0]}{'<' + k.split('<')[1][:14] if '<' in k else ''} {v:.0f}"
                    for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:5]), flush=True)
    for k, v in per.items():
        total[k] += v * len(names)
    del x, w, b, y, g
    torch.cuda.empty_cache()
s = sum(total.values())
print(f"\nstack total {s / 1e3:.2f} ms ({prec}, batch {batch}, profiled: serialised kernels)")
for k, v in sorted(total.items(), key=lambda kv: -kv[1]):
    print(f"{v / 1e3:8.3f} ms {100 * v / s:5.1f}%  {k}")
