"""QSync mixed-precision DP training step on B200 -- the driver's benchmark.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json configs[1], configs[3]): BERT-base encoder stack, seq 128,
batch 32 per GPU, synthetic token ids (seed-fixed), random-init weights, a
heterogeneous per-rank INT8/FP16 plan (rank r runs plan variant r % 2), FP32
master weights + AdamW, NCCL bucketed FP32 gradient all-reduce for N > 1.
One "step" = forward + backward + all-reduce + optimizer on one batch.

Metric: train samples/s (whole job, all ranks).  ``value`` is device-timed with
CUDA events around exactly K captured steps (inputs already in HBM), max over
ranks; ``e2e`` times the same steps through the public TrainStep call with the
token/label batch copied host->device from pinned memory and the loss read back
device->host every step.  The dominant kernel's roofline (the INT8 tcgen05 GEMM)
is measured live with CUDA events on its launching stream during an eager step;
its peak is the INT8 dense rate measured in this run with cuBLASLt at 8192^3.

``--impl reference`` times the reference path on the host CPU: the oracle
restatement (oracle/cpu_ref.c, OpenMP over all host cores) of the planned
Linear layers' forward+backward for a bounded sample of the batch.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QSync mixed-precision train samples/s at 1/2/4/8 B200; INT8 GEMM TOPS vs peak"
BATCH, SEQ = 32, 128
PLAN_DESC = {"mixed": "mixed INT8/FP16 per layer (rank r%2 mirrored), pooler FP32",
             "int8": "all encoder Linears INT8", "fp16": "all encoder Linears FP16"}


def _peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


def _ncu_traffic(prefix: str, shapes) -> float | None:
    """Mean per-launch DRAM traffic (read + write bytes) of a kernel at the step's
    shapes, from the committed `ncu --set full` capture (profiles/*_ncu_metrics.json,
    written by tools/summarize_round.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_metrics.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        m = json.load(f)
    sc = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for s in shapes:
        d = m.get(f"{prefix}_{s}")
        if not d or "dram__bytes_read.sum" not in d:
            return None
        vals.append(d["dram__bytes_read.sum"] * sc.get(d.get("dram__bytes_read.sum.unit"), 1.0)
                    + d["dram__bytes_write.sum"] * sc.get(d.get("dram__bytes_write.sum.unit"), 1.0))
    return sum(vals) / len(vals)


def _config(world: int, plan_desc: str) -> dict:
    return {"workload": "BERT-base encoder stack train step (configs[1]; DP configs[3])",
            "model": "bert-base (12x768, ffn 3072, 12 heads), fused QKV",
            "global_batch": BATCH * world, "seq_len": SEQ, "batch_per_gpu": BATCH,
            "parallelism": f"dp{world}", "precision_plan": plan_desc,
            "l2": "step working set (~0.5 GB weights+optimizer, activations) > 126 MB L2"}


# --------------------------------------------------------------------------- CPU leg
def cpu_sample(plan: dict, cfg, seqs: int = 1, rep: int = 1) -> dict:
    """Oracle forward+backward of the plan's encoder Linears for `seqs` sequences."""
    import numpy as np

    from oracle.cpu_ref import CpuRef
    ref = CpuRef()
    M = seqs * SEQ
    h, f = cfg.hidden, cfg.ffn
    rng = np.random.default_rng(0)
    shapes = {"qkv": (3 * h, h), "o": (h, h), "ff1": (f, h), "ff2": (h, f)}
    weights = {k: (rng.uniform(-1, 1, size=s) / np.sqrt(s[1])).astype(np.float32)
               for k, s in shapes.items()}
    xs = {k: rng.normal(size=(M, s[1])).astype(np.float32) for k, s in shapes.items()}
    gs = {k: rng.normal(size=(M, s[0])).astype(np.float32) for k, s in shapes.items()}
    bias = {k: np.zeros(s[0], np.float32) for k, s in shapes.items()}
    t0 = time.perf_counter()
    for _ in range(rep):
        for i in range(cfg.layers):
            for op in ("qkv", "o", "ff1", "ff2"):
                p = plan.get(f"layer{i}.{op}", "FP32")
                if p == "INT8":
                    ref.qlinear_int8(xs[op], weights[op], bias[op], gs[op])
                else:  # FP16 (and FP32 rows, timed with the same wide-accumulation loops)
                    ref.qlinear_f16(xs[op], weights[op], bias[op], gs[op])
    dt = (time.perf_counter() - t0) / rep
    return {"seconds_per_rep": dt, "samples": seqs, "threads": ref.num_threads()}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # reference arm: rank 0 alone runs and prints
    from paper_2407_02327_b200.train_step import BertConfig, mixed_plan
    cfg = BertConfig()
    plan = mixed_plan(cfg)
    first = cpu_sample(plan, cfg)  # warm-up (page-in, thread pool)
    threads = first["threads"]
    # Bound the CPU leg to ~2 minutes: time min(K, budget / first) steps.
    budget_s = float(os.environ.get("QSYNC_REF_BUDGET_S", "120"))
    steps = max(1, min(args.steps, int(budget_s / max(first["seconds_per_rep"], 1e-3))))
    times = [cpu_sample(plan, cfg)["seconds_per_rep"] for _ in range(steps)]
    t = statistics.mean(times)
    value = 1.0 / t  # samples (sequences) per second
    sample = (f"1 sequence (128 tokens) of the 32-sequence batch: forward+dgrad+wgrad of the 48 "
              f"planned encoder Linears at the mixed INT8/FP16 plan (oracle/cpu_ref.c); "
              f"attention/LayerNorm/optimizer not included")
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "steps_timed": steps,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int8/fp16 (f64 accumulation on CPU)",
            "data": "synthetic", "config": _config(args.gpus, PLAN_DESC["mixed"]),
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.  NVML is read
    from a thread every ~4 ms, so even a 0.1 s region (the driver's 20 steps)
    yields ~25 samples; nvidia-smi -lms 100 is the fallback when NVML is absent."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index: int, pci_bus_id: str | None = None, period_s: float = 0.004):
        self.index = index
        self.pci = pci_bus_id
        self.period = period_s
        self.proc = None
        self.thread = None
        self.samples: list[tuple[float, float, int]] = []  # (sm MHz, max MHz, reason bits)
        self.out = ""

    def _nvml_loop(self, nv, h):
        import time as _t
        while not self._stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), int(rs)))
            except Exception:  # noqa: BLE001 -- a failed read is a missing sample
                pass
            _t.sleep(self.period)

    def __enter__(self):
        import threading
        self._stop = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
                except Exception:  # noqa: BLE001
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi fallback
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self._stop = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        if self.samples:
            for s, m, bits in self.samples:
                sm.append(s)
                mx = m
                for nm, bit in self.REASONS:
                    if bits & bit:
                        reasons.add(nm)
            src = f"NVML every {self.period * 1e3:.0f} ms"
        else:
            rows = [r.split(", ") for r in self.out.strip().splitlines() if r.strip()]
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for r in rows:
                try:
                    sm.append(float(r[1]))
                    mx = float(r[2])
                    for i, nm in enumerate(names):
                        if r[5 + i].strip().lower() == "active":
                            reasons.add(nm)
                except (ValueError, IndexError):
                    continue
            src = "nvidia-smi -lms 100"
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


def int8_peak(torch) -> float:
    n = 8192
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def gemm_durations(step, torch, ops, reps: int = 3):
    """Per-kind (gemm_s8 / gemm_f16) algorithmic flops and device time of one train
    step's GEMM launches, timed inside a captured copy of the step (see run_ours)."""
    n0 = ops.launch_count()
    ops.GEMM_TIMER = []
    try:
        s = torch.cuda.Stream(priority=-1)
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                step._body()
        rec = ops.GEMM_TIMER
    finally:
        ops.GEMM_TIMER = None
    launches = ops.launch_count() - n0  # this library's kernels in one step
    torch.cuda.current_stream().wait_stream(s)
    per = [[] for _ in rec]
    for _ in range(reps):
        g.replay()
        torch.cuda.synchronize()
        for i, (_, _, e0, e1) in enumerate(rec):
            per[i].append(e0.elapsed_time(e1))
    kern = {}
    for (kind, flops, _, _), ts in zip(rec, per):
        d = kern.setdefault(kind, {"flops": 0.0, "ms": 0.0, "launches": 0})
        d["flops"] += flops
        d["ms"] += statistics.median(ts)
        d["launches"] += 1
    del g
    return kern, launches


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2407_02327_b200 import ops
    from paper_2407_02327_b200.qlinear import FP16, INT8
    from paper_2407_02327_b200.train_step import (BertConfig, BertEncoderStack, TrainStep,
                                                  linear_flops_per_step, mixed_plan, uniform_plan)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}: launch through "
                         f"torch.distributed.run or let bench.py spawn the ranks")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.manual_seed(1234)  # identical initial weights on every rank
    cfg = BertConfig(seq=SEQ)
    model = BertEncoderStack(cfg).cuda()
    # Heterogeneous per-rank plans: rank r runs the mixed plan, odd ranks its
    # mirror (INT8 <-> FP16 per layer), as the allocator hands each device its own.
    plan = mixed_plan(cfg)
    if args.plan == "int8":
        plan = uniform_plan(cfg, INT8)
    elif args.plan == "fp16":
        plan = uniform_plan(cfg, FP16)
    elif rank % 2 == 1:
        plan = {k: ({INT8: FP16, FP16: INT8}.get(v, v)) for k, v in plan.items()}
    model.apply_plan(plan)
    plan_desc = PLAN_DESC[args.plan]

    step = TrainStep(model, BATCH, world=world, graph=not args.no_graph)
    g = torch.Generator().manual_seed(100 + rank)
    nb = max(1, min(args.steps, 8))
    host_tokens = [torch.randint(0, cfg.vocab, (BATCH, SEQ), generator=g).pin_memory() for _ in range(nb)]
    host_labels = [torch.randint(0, 2, (BATCH,), generator=g).pin_memory() for _ in range(nb)]
    step.tokens.copy_(host_tokens[0])
    step.labels.copy_(host_labels[0])

    launches_per_step = None
    step.capture(warmup=args.warmup)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-timed region: K captured steps, inputs resident in HBM ----
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()
    pr = torch.cuda.get_device_properties(local)
    try:
        pci = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
    except (AttributeError, TypeError, ValueError):
        pci = None
    barrier()
    # Clocks are sampled over both timed regions (device-timed and e2e).
    with ClockSampler(local, pci) as clk:
        t_s, t_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_s.record()
        for _ in range(args.steps):
            loss = step()
        t_e.record()
        barrier()
        ms = t_s.elapsed_time(t_e)

        # ---- e2e: H2D of each step's batch from pinned memory + D2H of the loss ----
        barrier()
        e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_s.record()
        for k in range(args.steps):
            step.tokens.copy_(host_tokens[k % nb], non_blocking=True)
            step.labels.copy_(host_labels[k % nb], non_blocking=True)
            loss = step()
            loss_host.copy_(loss, non_blocking=True)
        e_e.record()
        barrier()
        ms_e2e = e_s.elapsed_time(e_e)
    h2d = host_tokens[0].numel() * 8 + host_labels[0].numel() * 8
    d2h = 4

    # ---- dominant-kernel roofline, measured live on the step's own streams: the
    # step is captured once more with an event-record node around every GEMM
    # launch (ops.GEMM_TIMER; external events inside the capture) and replayed;
    # each GEMM's duration is its event pair on the stream it was launched on.
    # (Event nodes cut the PDL overlap a GEMM has in the timed graph, so these
    # durations include each GEMM's own launch and prologue: conservative.)
    kern, launches_per_step = gemm_durations(step, torch, ops, reps=3)

    if world > 1:
        t = torch.tensor([ms, ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = t.tolist()

    if rank == 0:
        pk = _peaks()
        i8 = int8_peak(torch)
        samples = BATCH * world * args.steps
        value = samples / (ms * 1e-3)
        e2e = samples / (ms_e2e * 1e-3)
        k8 = kern.get("gemm_s8", {"flops": 0.0, "ms": 1e-9, "launches": 1})
        k16 = kern.get("gemm_f16", {"flops": 0.0, "ms": 1e-9, "launches": 1})
        ach = k8["flops"] / (k8["ms"] * 1e-3) / 1e12 if k8["flops"] else 0.0
        ach16 = k16["flops"] / (k16["ms"] * 1e-3) / 1e12 if k16["flops"] else 0.0
        how = ("sum of 2MNK over the step's {n} {k} launches / their device durations: CUDA events "
               "recorded around each launch on its own stream inside a captured copy of the step "
               "(median of 3 replays; includes each launch's own prologue)")
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int8/fp16 (per-layer plan), fp32 master weights", "data": "synthetic",
            "config": _config(world, plan_desc),
            # the time-dominant kernel family of the step: the FP16 tcgen05 GEMMs
            # (every backward GEMM and the FP16 layers' forward)
            "roofline": {
                "bound": "tensor", "kernel": "k_gemm_tc<kI8=false> (tcgen05 kind::f16, fwd/dgrad/wgrad)",
                "achieved": ach16, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": ach16 / pk["bf16_tflops"],
                "traffic": _ncu_traffic("gemm_f16", ("ff1",)),
                "traffic_unit": "bytes per launch (DRAM read+write, ncu --set full, FF1 shape)",
                "peak_source": pk["source"] + " dense bf16/fp16 (burst)",
                "achieved_how": how.format(n=k16["launches"], k="FP16 GEMM"),
                "step_share_ms": k16["ms"],
            },
            # the metric's named quantity: INT8 GEMM TOPS vs the INT8 dense peak
            "roofline_int8": {
                "bound": "tensor", "kernel": "k_gemm_tc<kI8=true> (tcgen05 kind::i8, fused dequant)",
                "achieved": ach, "peak": i8, "unit": "TFLOP/s", "frac": ach / i8 if i8 else None,
                "traffic": _ncu_traffic("gemm_s8", ("qkv", "o", "ff1", "ff2")),
                "traffic_unit": "bytes per launch (DRAM read+write, ncu --set full, mean of the 4 step shapes)",
                "peak_source": "INT8 dense measured in this run: cuBLASLt torch._int_mm 8192^3 best of 10",
                "achieved_how": how.format(n=k8["launches"], k="INT8 GEMM"),
                "frac_vs_datasheet_4500": ach / 4500.0,
            },
            "kernels": {"gemm_s8": {**k8, "tflops": ach}, "gemm_f16": {**k16, "tflops": ach16,
                        "frac_vs_bf16_peak": ach16 / pk["bf16_tflops"]}},
            "linear_tflops_per_step_per_gpu": linear_flops_per_step(cfg, BATCH * SEQ) / 1e12,
            "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": (launches_per_step or 0) * args.steps,
            "clocks": clk.summary(),
            "loss": float(loss_host.item()),
        }
        if world == 1 and not args.no_cpu_baseline:
            cs = cpu_sample(plan, cfg)
            line["cpu_baseline"] = {
                "value": 1.0 / cs["seconds_per_rep"], "unit": "samples/s", "cores": cs["threads"],
                "kind": "port",
                "sample": ("1 sequence (128 tokens): forward+dgrad+wgrad of the 48 planned encoder "
                           "Linears, oracle/cpu_ref.c with OpenMP")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args) -> int:
    """``python bench.py --gpus N`` with N > 1 and no torchrun environment:
    re-launch this script as N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1, exactly as the driver does.  NCCL INIT
    logging is on so every communicator reports its nranks (on stderr)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_selftest(args) -> None:
    """Rank plumbing without a GPU (tests/test_bench_spawn.py): gloo rendezvous,
    per-rank timing, MAX over ranks, one JSON line from rank 0."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    x = torch.full((1024,), float(rank + 1))
    for _ in range(args.steps):
        if world > 1:
            dist.all_reduce(x)
    ms = (time.perf_counter() - t0) * 1e3
    t = torch.tensor([ms, float(rank)])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "selftest": True, "n_gpus": world, "steps": args.steps,
                          "ms_max_over_ranks": float(t[0]), "max_rank": int(t[1]),
                          "allreduce_value": float(x[0])}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)  # ~1 s timed: ~10 clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--plan", choices=["mixed", "int8", "fp16"], default="mixed")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--selftest", action="store_true", help="rank plumbing only (CPU, gloo)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.selftest:
        run_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
