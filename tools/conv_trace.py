"""Kernel breakdown (CUPTI) of one planned Conv2d fwd+bwd at a ResNet-50 shape.

    python tools/conv_trace.py [N H C Cout R stride pad prec]
"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200.qconv import qconv2d  # noqa: E402

a = sys.argv[1:] or ["64", "224", "3", "64", "7", "2", "3", "FP16"]
N, H, C, Co, R, st, pd = map(int, a[:7])
prec = a[7]
x = torch.randn(N, H, H, C, device="cuda")
if prec == "FP16":
    x = x.half()
x.requires_grad_(True)
w = (torch.randn(Co, R, R, C, device="cuda") / (R * R * C) ** 0.5).requires_grad_(True)
b = torch.zeros(Co, device="cuda", requires_grad=True)
y = qconv2d(x, w, b, (st, st), (pd, pd), prec)
g = torch.randn_like(y)
y.backward(g)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    y = qconv2d(x, w, b, (st, st), (pd, pd), prec)
    y.backward(g)
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name.replace("(anonymous namespace)::", "").split("(")[0][:90]] += e.time_range.end - e.time_range.start
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.1f} us  {k}")
