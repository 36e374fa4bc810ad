"""Kernel-level timeline of one eager training step from CUPTI (torch.profiler's CUDA
activity trace), per CUDA stream: proves (or disproves) that PaReprop's recompute lane and
gradient lane execute kernels concurrently. This stands in for an nsys timeline (the
image's nsys cannot import its own .qdstrm captures).

    python tools/cupti_timeline.py [preset=revvit-b] [batch=256] [out=gpurun_out/timeline]

Writes <out>_<mode>.json (Chrome trace, loadable in chrome://tracing / Perfetto) and prints
per-stream kernel busy time, the backward window, and the time during which kernels of
the two lanes' streams were resident on the GPU at the same time.
"""
import json
import sys

sys.path.insert(0, ".")

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig  # noqa: E402


def union(iv):
    iv = sorted(iv)
    out = []
    for s, e in iv:
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


def inter(a, b):
    i = j = 0
    tot = 0.0
    while i < len(a) and j < len(b):
        lo, hi = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if hi > lo:
            tot += hi - lo
        if a[i][1] < b[j][1]:
            i += 1
        else:
            j += 1
    return tot


def main():
    kw = dict(preset="revvit-b", batch=None, out="gpurun_out/timeline")
    for a in sys.argv[1:]:
        k, v = a.split("=")
        kw[k] = v
    p = dict(PRESETS[kw["preset"]])
    if kw["batch"]:
        p["batch"] = int(kw["batch"])
    eng = Engine(ModelConfig(**p))
    for mode, name in ((REPROP, "reprop"), (PAREPROP, "pareprop")):
        for _ in range(2):
            eng.step(mode, graph=False)
        eng.sync()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            eng.step(mode, graph=False)
            eng.sync()
        path = f"{kw['out']}_{name}.json"
        prof.export_chrome_trace(path)
        with open(path) as f:
            ev = json.load(f)["traceEvents"]
        k = [e for e in ev if e.get("cat") == "kernel"]
        by_stream = {}
        for e in k:
            sid = e["args"].get("stream", e.get("tid"))
            by_stream.setdefault(sid, []).append((e["ts"], e["ts"] + e["dur"]))
        t0 = min(s for v in by_stream.values() for s, _ in v)
        t1 = max(e for v in by_stream.values() for _, e in v)
        print(f"== {name}, {kw['preset']} batch {p['batch']}: {len(k)} kernels, step "
              f"{(t1 - t0) / 1e3:.3f} ms (eager)")
        streams = sorted(by_stream, key=lambda s: -len(by_stream[s]))
        for s in streams:
            u = union(by_stream[s])
            busy = sum(e - b for b, e in u)
            print(f"   stream {s}: {len(by_stream[s])} kernels, busy {busy / 1e3:.3f} ms")
        if len(streams) >= 2:
            a, b = union(by_stream[streams[0]]), union(by_stream[streams[1]])
            ov = inter(a, b)
            print(f"   streams {streams[0]} and {streams[1]} concurrently executing: "
                  f"{ov / 1e3:.3f} ms ({100 * ov / (t1 - t0):.1f}% of the step)")
    eng.close()


if __name__ == "__main__":
    main()
