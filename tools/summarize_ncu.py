"""Summarise ncu outputs into profiles/ (run here, on the CPU side).

    python tools/summarize_ncu.py launches <launches.csv> <out.md>
    python tools/summarize_ncu.py report <prof.ncu-rep> <out.md> [algorithmic_bytes_or_flops unit]
"""
import collections
import csv
import io
import subprocess
import sys


def _launch_rows(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) > 5]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")

    def ns(r):
        v = float(r[mi].replace(",", ""))
        return v * 1e3 if r[ui] == "usecond" else (v * 1e6 if r[ui] == "msecond" else v)

    return [(r[ki], ns(r)) for r in data]


def launches(path, out):
    rows = _launch_rows(path)
    # One step starts with the reset of the flat gradient buffer (k_zero16 of
    # qsync_zero; a framework FillFunctor before round 2) and ends with the
    # optimizer; take the last complete step.
    fills = [i for i, (k, v) in enumerate(rows) if ("FillFunctor" in k or "k_zero16" in k) and v > 20e3]
    seg = rows
    for a, b in zip(fills[-2::-1], fills[:0:-1]):
        if any("multi_tensor_apply" in k or "k_adamw" in k for k, _ in rows[a:b]):
            seg = rows[a:b]
            break
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v in seg:
        short = k.split("(")[0][:90]
        tot[short] += v
        cnt[short] += 1
    T = sum(tot.values())
    ours = sum(v for k, v in tot.items() if "qsb::" in k)
    lines = [f"# ncu launch list -- one training step ({len(seg)} kernels)\n",
             f"Source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none;",
             "cold-cache, serialised: compare SHARES, not absolutes).\n",
             f"Sum of kernel durations: {T/1e3:.1f} us; this package's kernels (qsb::): "
             f"{ours/T*100:.1f}%.\n",
             "| share | total us | launches | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {v/T*100:.2f}% | {v/1e3:.1f} | {cnt[k]} | `{k}` |")
    open(out, "w").write("\n".join(lines) + "\n")
    print(f"wrote {out}")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def report(path, out, alg=None, unit=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{path}`\n"]
    for r in rows[2:]:
        d = dict(zip(h, r))
        lines.append(f"## `{d.get('Kernel Name', '?')[:120]}`\n")
        lines.append("| metric | value | unit |")
        lines.append("|---|---:|---|")
        for w in WANT:
            if w in h:
                lines.append(f"| {w} | {d[w]} | {units[h.index(w)]} |")
        if alg:
            dur = float(d["gpu__time_duration.sum"].replace(",", ""))
            dur_s = dur * (1e-6 if units[h.index('gpu__time_duration.sum')] == "us" else 1e-9)
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
            lines.append(f"\nAlgorithmic {unit} per launch: {alg:.4g}; achieved (cold, under ncu): "
                         f"{alg / dur_s / (1e9 if unit == 'bytes' else 1e12):.1f} "
                         f"{'GB/s' if unit == 'bytes' else 'TFLOP/s'}\n")
            _ = rd
    open(out, "w").write("\n".join(lines) + "\n")
    print(f"wrote {out}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
        report(sys.argv[2], sys.argv[3], alg, sys.argv[5] if len(sys.argv) > 5 else None)
