"""One device SR call (FP32 -> INT8 on the reference mt19937_64 stream) at 16M
elements, for ncu: `ncu --set full -k regex:'k_mt_jump|k_sr' python tools/sr_ncu_target.py`."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops  # noqa: E402

x = torch.randn(1 << 24, device="cuda")
sc = torch.tensor([0.01, 1.0], device="cuda")
ops.quantize_sr(x, sc, 7)
torch.cuda.synchronize()
