"""Per-stream exclusive time of a measured step trace (tools/step_trace.py output).

Kernels on one stream overlap under programmatic dependent launch (a kernel's
recorded start includes its griddepcontrol.wait), so each kernel is charged
only [max(start, previous end on its stream), end]: the stream's critical-path
share by kernel.

    python tools/stream_breakdown.py gpurun_out/step_trace.trace.json.gz [--steps 5]
"""
import argparse
import collections
import gzip
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--top", type=int, default=25)
    args = ap.parse_args()
    with gzip.open(args.trace, "rt") as f:
        evs = json.load(f)["traceEvents"]
    by_tid = collections.defaultdict(list)
    for e in evs:
        by_tid[e["tid"]].append(e)
    for tid, es in sorted(by_tid.items(), key=lambda kv: -sum(e["dur"] for e in kv[1])):
        es.sort(key=lambda e: e["ts"])
        excl = collections.Counter()
        cnt = collections.Counter()
        prev = None
        span0, span1 = es[0]["ts"], max(e["ts"] + e["dur"] for e in es)
        for e in es:
            s, t = e["ts"], e["ts"] + e["dur"]
            if prev is not None:
                s = max(s, prev)
            excl[e["name"]] += max(0.0, t - s)
            cnt[e["name"]] += 1
            prev = max(prev or t, t)
        tot = sum(excl.values())
        print(f"== stream {tid}: {len(es) // args.steps} launches/step, exclusive busy {tot / args.steps:.1f} us/step,"
              f" span {(span1 - span0) / args.steps:.1f} us/step")
        for n, v in excl.most_common(args.top):
            print(f"   {v / args.steps:9.1f} us  {cnt[n] // args.steps:4d}x  {n}")


if __name__ == "__main__":
    main()
