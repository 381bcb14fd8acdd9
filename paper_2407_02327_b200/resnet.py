"""ResNet-50 (NHWC, 224x224) whose 53 convolutions and classifier follow a QSync plan.

BASELINE configs[2]: the paper's conv workload. Every Conv2d is a
`QConv2d` (implicit-GEMM INT8 / FP16 on tcgen05, FP32 for training ranks), the
classifier a `QLinear`; BatchNorm + ReLU and the residual adds are the graph's
fixed FP32 operators (the reference keeps normalisation out of the adjustable set,
graph.hpp:18-33 `OperatorKind`). Omitted plan entries run FP32 (replayer.cpp:86-94).

The op ids here are the ones `profiler_resnet.resnet50_graph` emits, so a plan the
reference `solve` writes for that bundle loads straight into this model.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from . import qlinear
from .qconv import QConv2d
from .qlinear import FP32, QLinear

# (stage width, blocks, first stride) of ResNet-50's four residual stages
STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))


def conv_specs(batch: int, image: int = 224):
    """The 53 convolutions in execution order:
    (op id, N, H, W, C, Cout, R, stride, pad, block id)."""
    h = image // 4
    out = [("conv1", batch, image, image, 3, 64, 7, 2, 3, "stem")]
    cin = 64
    for si, (width, blocks, stride) in enumerate(STAGES):
        for b in range(blocks):
            s = stride if b == 0 else 1
            blk = f"res{si + 2}.{b}"
            ho = h // s
            out.append((f"{blk}.a", batch, h, h, cin, width, 1, 1, 0, blk))
            out.append((f"{blk}.b", batch, h, h, width, width, 3, s, 1, blk))
            out.append((f"{blk}.c", batch, ho, ho, width, 4 * width, 1, 1, 0, blk))
            if b == 0:
                out.append((f"{blk}.ds", batch, h, h, cin, 4 * width, 1, s, 0, blk))
            cin, h = 4 * width, ho
    return out


class _Conv(QConv2d):
    """QConv2d that reports the K5 statistics of its input, weight and incoming
    gradient to the active `qlinear.STATS_RECORDER` (profile.hpp:95-108)."""

    def forward(self, x):
        rec = qlinear.STATS_RECORDER is not None
        if rec:
            qlinear._record(self.name, "act", x)
            qlinear._record(self.name, "w", self.weight.detach())
        y = super().forward(x)
        if rec and y.requires_grad:
            y.register_hook(lambda g, n=self.name: qlinear._record(n, "grad", g))
        return y


class _BN(torch.nn.Module):
    """BatchNorm over the channel axis of an NHWC tensor, computed in FP32."""

    def __init__(self, c):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.ones(c))
        self.bias = torch.nn.Parameter(torch.zeros(c))
        self.register_buffer("rm", torch.zeros(c))
        self.register_buffer("rv", torch.ones(c))

    def forward(self, x):
        y = F.batch_norm(x.float().permute(0, 3, 1, 2), self.rm, self.rv, self.weight, self.bias,
                         self.training, 0.1, 1e-5)
        return y.permute(0, 2, 3, 1)


class ResNet50(torch.nn.Module):
    def __init__(self, num_classes: int = 1000, image: int = 224):
        super().__init__()
        self.image = image
        self.convs = torch.nn.ModuleDict()
        self.bns = torch.nn.ModuleDict()
        self.specs = conv_specs(1, image)
        for name, _, _, _, c, cout, r, s, p, _ in self.specs:
            self.convs[name.replace(".", "_")] = _Conv(c, cout, r, name, stride=s, pad=p, bias=False)
            self.bns[name.replace(".", "_")] = _BN(cout)
        self.fc = QLinear(2048, num_classes, "fc")

    def qops(self) -> dict:
        d = {m.name: m for m in self.convs.values()}
        d["fc"] = self.fc
        return d

    def apply_plan(self, plan: dict[str, str]) -> None:
        for name, m in self.qops().items():
            m.precision = plan.get(name, FP32)

    def _cbr(self, name, x, relu=True):
        k = name.replace(".", "_")
        y = self.bns[k](self.convs[k](x))
        return F.relu(y) if relu else y

    def forward(self, images, labels):
        """images NHWC [N, H, W, 3] FP32, labels [N] -> mean cross-entropy."""
        x = self._cbr("conv1", images)
        x = F.max_pool2d(x.permute(0, 3, 1, 2), 3, 2, 1).permute(0, 2, 3, 1).contiguous()
        for si, (_, blocks, _) in enumerate(STAGES):
            for b in range(blocks):
                blk = f"res{si + 2}.{b}"
                y = self._cbr(f"{blk}.a", x)
                y = self._cbr(f"{blk}.b", y)
                y = self._cbr(f"{blk}.c", y, relu=False)
                sc = self._cbr(f"{blk}.ds", x, relu=False) if b == 0 else x
                x = F.relu(y + sc).contiguous()
        pooled = x.mean(dim=(1, 2))
        return F.cross_entropy(self.fc(pooled), labels)
