"""A/B the graphed BERT-base train step (batch 32 x 128, CUDA-graph replay,
CUDA-event timed, best of 3 x 40 steps) over one switch at a time.  Every
variant builds a fresh model and TrainStep; runs alternate so drift between
repetitions shows.

    python tools/ab_step.py plan=mixed,int8,fp16
    python tools/ab_step.py attn=0,1,2            attention core impl (csrc/attn.cu)
    python tools/ab_step.py pdl=1,0               programmatic dependent launch
    python tools/ab_step.py overlap=1,0           wgrad GEMMs on the side stream
    python tools/ab_step.py overlap_opt=0,1       bucket-wise AdamW on the comm stream
    python tools/ab_step.py wgrad_cap=0,98        side-stream wgrad grid cap (CTAs)
    python tools/ab_step.py lib=default,/tmp/x.so library build (fresh process each)
    python tools/ab_step.py ff1gelu=1,0           GELU in FF1's GEMM epilogue vs the operand kernel
    python tools/ab_step.py ff2recompute=1,0      INT8 FF2 operand: GELU twice vs stored GELU(h)
    python tools/ab_step.py head=1,0              classification head on csrc/head.cu vs torch
    python tools/ab_step.py attnq=1,0             INT8 O operand quantized in the attention kernel
    python tools/ab_step.py dual=1,0              two MMA issuers on 192-wide single-unit GEMMs
    python tools/ab_step.py wgradpdl=1,0          side-stream wgrad GEMMs launched with PDL
    python tools/ab_step.py zero=1,0              gradient reset overlapping the forward
    python tools/ab_step.py onepass=1,0           INT8 FF1 -> FF2 operand in one pass (GEMM ymax)
    QSB_AB_PLAN=int8 python tools/ab_step.py ...  plan for the non-plan knobs (default mixed)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def step_ms(knob: str, val: str, steps: int = 40) -> float:
    import torch

    from paper_2407_02327_b200 import _lib, fused
    from paper_2407_02327_b200.qlinear import FP16, INT8
    from paper_2407_02327_b200.train_step import (BertConfig, BertEncoderStack, TrainStep, mixed_plan,
                                                  uniform_plan)
    cfg = BertConfig()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    plan = val if knob == "plan" else os.environ.get("QSB_AB_PLAN", "mixed")
    fused.FF1_GELU_EPILOGUE = knob == "ff1gelu" and val == "1"
    fused.FF2_INT8_RECOMPUTE = knob == "ff2recompute" and val == "1"
    import paper_2407_02327_b200.train_step as _ts
    _ts.HEAD_KERNELS = not (knob == "head" and val == "0")
    _ts.ZERO_OVERLAP = not (knob == "zero" and val == "0")
    fused.ATTN_QUANT = not (knob == "attnq" and val == "0")
    fused.WGRAD_PDL = not (knob == "wgradpdl" and val == "0")
    fused.GELU_ONE_PASS = not (knob == "onepass" and val == "0")
    from paper_2407_02327_b200 import ops as _ops
    _ops.set_dual_issue(not (knob == "dual" and val == "0"))
    m.apply_plan({"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16)}[plan])
    kw = {}
    if knob == "overlap":
        kw["overlap_wgrad"] = val == "1"
    if knob == "overlap_opt":
        kw["overlap_opt"] = val == "1"
    if knob == "attn":
        _lib.call("qsync_attention_set_impl", int(val))
    if knob == "pdl":
        _lib.call("qsync_gemm_set_pdl", int(val))
    st = TrainStep(m, batch=32, graph=True, **kw)
    if knob == "wgrad_cap":
        fused.WGRAD_CTAS = int(val)  # after TrainStep, which sets its default
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    for _ in range(5):
        st()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            st()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / steps)
    return best


def main():
    knob, vals = sys.argv[1].split("=", 1)
    vals = vals.split(",")
    if knob == "--one":  # child process of the lib switch: --one=<knob>:<val>
        k, v = vals[0].split(":", 1)
        print(step_ms(k, v))
        return
    for rep in range(2):
        for v in vals:
            if knob == "lib":
                env = dict(os.environ)
                if v != "default":
                    env["QSYNC_B200_LIB"] = os.path.abspath(v)
                plan = os.environ.get("QSB_AB_PLAN", "mixed")
                r = subprocess.run([sys.executable, __file__, f"--one=plan:{plan}"], env=env, capture_output=True,
                                   text=True)
                ms = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else float("nan")
            else:
                ms = step_ms(knob, v)
            print(f"rep {rep} {knob}={v:24s} step_ms={ms:.3f}", flush=True)


if __name__ == "__main__":
    main()
