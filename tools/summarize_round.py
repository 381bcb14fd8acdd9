"""Run on the GPU box after tools/profile_round.sh: summarise every
gpurun_out/prof_*.ncu-rep into gpurun_out/ncu_<target>.md and collect the raw
per-launch metrics (duration, DRAM bytes, pipe utilisation) into
gpurun_out/ncu_metrics.json, so the large reports need not travel back.

    python tools/summarize_round.py [--keep-reps]
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.summarize_ncu import WANT, launches, report  # noqa: E402

T, H, F = 4096, 768, 3072
ALG = {  # algorithmic flops (GEMM) or bytes (streaming) per launch
    "gemm_s8_qkv": (2.0 * T * 3 * H * H, "flops"), "gemm_s8_o": (2.0 * T * H * H, "flops"),
    "gemm_s8_ff1": (2.0 * T * F * H, "flops"), "gemm_s8_ff2": (2.0 * T * H * F, "flops"),
    "gemm_s8_8192": (2.0 * 8192 ** 3, "flops"), "gemm_f16_8192": (2.0 * 8192 ** 3, "flops"),
    "gemm_f16_ff1": (2.0 * T * F * H, "flops"),
    "attn_fwd": (32 * 12 * (3 * 128 * 64 * 2 + 128 * 64 * 2 + 128 * 4), "bytes"),
    "attn_bwd": (32 * 12 * (5 * 128 * 64 * 2 + 128 * 4 + 3 * 128 * 64 * 2), "bytes"),
    "ln_bwd": (T * H * (4 + 4 + 4 + 2), "bytes"), "act_bwd": (T * F * (2 + 2 + 2), "bytes"),
    "conv_fwd": (2.0 * 64 * 28 * 28 * 128 * 9 * 128, "flops"), "conv_wgrad": (2.0 * 64 * 28 * 28 * 128 * 9 * 128, "flops"),
    "conv_dgrad": (2.0 * 64 * 28 * 28 * 128 * 9 * 128, "flops"),
    "quantize_with_scale": ((1 << 28) * 5, "bytes"), "quantize_per_channel": ((1 << 28) * 5, "bytes"),
    "absmax": ((1 << 28) * 4, "bytes"), "stats": ((1 << 28) * 4, "bytes"), "cast": ((1 << 28) * 6, "bytes"),
    "dequantize": ((1 << 28) * 5, "bytes"), "quantize_f16": ((1 << 28) * 3, "bytes"),
    "quantize_per_tensor": ((1 << 28) * 5, "bytes"),
}


def raw_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, units = rows[0], rows[1]
    d = dict(zip(h, rows[2]))
    res = {"kernel": d.get("Kernel Name", "?")[:160]}
    for w in WANT:
        if w in d:
            try:
                res[w] = float(d[w].replace(",", ""))
                res[w + ".unit"] = units[h.index(w)]
            except ValueError:
                pass
    return res


def main():
    keep = "--keep-reps" in sys.argv
    metrics = {}
    for rep in sorted(glob.glob("gpurun_out/prof_*.ncu-rep")):
        t = os.path.basename(rep)[len("prof_"):-len(".ncu-rep")]
        alg, unit = ALG.get(t, (None, None))
        report(rep, f"gpurun_out/ncu_{t}.md", alg, unit)
        metrics[t] = raw_metrics(rep)
        if alg:
            metrics[t]["algorithmic_" + unit] = alg
        if not keep and "ff1" not in t:
            os.remove(rep)
    if os.path.exists("gpurun_out/launches_bench.csv"):
        launches("gpurun_out/launches_bench.csv", "gpurun_out/launches_step.md")
    with open("gpurun_out/ncu_metrics.json", "w") as f:
        json.dump(metrics, f, indent=1)
    print(f"summarised {len(metrics)} reports")


if __name__ == "__main__":
    main()
