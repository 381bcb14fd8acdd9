"""A/B the graphed BERT-base step across library builds:
    python tools/ab_libs.py lib_a.so lib_b.so ...   (each run in a fresh process)"""
import os
import subprocess
import sys

CODE = r"""
import os, sys, torch
sys.path.insert(0, %r)
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan
cfg = BertConfig(); torch.manual_seed(0)
m = BertEncoderStack(cfg).cuda(); m.apply_plan(mixed_plan(cfg))
st = TrainStep(m, batch=32, graph=True); st.tokens.random_(0, cfg.vocab); st.capture(warmup=3)
for _ in range(10): st()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): st()
e.record(); torch.cuda.synchronize()
print(s.elapsed_time(e) / 50)
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = sys.argv[1:]
for rep in range(3):
    for lib in libs:
        env = dict(os.environ)
        if lib != "default":
            env["QSYNC_B200_LIB"] = os.path.abspath(lib)
        out = subprocess.run([sys.executable, "-c", CODE % root], env=env, capture_output=True, text=True)
        print(f"{lib:28s} step_ms={float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else -1:.3f} {out.stderr.strip()[-200:] if out.returncode else ''}",
              flush=True)
