"""A/B the graphed BERT-base step under library switches (PDL on/off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import _lib  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, mixed_plan  # noqa: E402
from tools.replay_fidelity import measured_step_ms  # noqa: E402

cfg = BertConfig()
for pdl in (1, 0, 1, 0):
    _lib.call("qsync_gemm_set_pdl", pdl)
    print(f"pdl={pdl} step_ms={measured_step_ms(cfg, 32, mixed_plan(cfg), steps=30):.3f}", flush=True)
