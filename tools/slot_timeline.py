"""Lane timeline of one PaReprop (and Reprop) backward from the engine's CUDA-event slot
log: per block, the recompute slot (lane R) and the gradient slot (lane G),
and how much of the backward the two lanes spend executing concurrently.

    python tools/slot_timeline.py [batch=256] [preset=revvit-b]

(nsys is present in the image but its importer is not, so the overlap evidence is taken
from CUDA events recorded on each lane's stream around every slot.)
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig  # noqa


def union_len(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for s, e in iv:
        if cur is None or s > cur[1]:
            if cur is not None:
                tot += cur[1] - cur[0]
            cur = [s, e]
        else:
            cur[1] = max(cur[1], e)
    if cur is not None:
        tot += cur[1] - cur[0]
    return tot


def overlap(a, b):
    tot = 0.0
    for s1, e1 in a:
        for s2, e2 in b:
            tot += max(0.0, min(e1, e2) - max(s1, s2))
    return tot


def main():
    kw = dict(batch=256, preset="revvit-b")
    for a in sys.argv[1:]:
        k, v = a.split("=")
        kw[k] = v
    p = dict(PRESETS[kw["preset"]])
    p["batch"] = int(kw["batch"])
    eng = Engine(ModelConfig(**p))
    eng.set_instrument(True)
    for mode, name in ((REPROP, "reprop"), (PAREPROP, "pareprop")):
        for _ in range(2):
            eng.step(mode, graph=False)
        eng.sync()
        eng.step(mode, graph=False)
        eng.sync()
        log = eng.slot_log()  # [lane][block][start, end] ms, relative to the first R slot
        r = [(float(log[0, b, 0]), float(log[0, b, 1])) for b in range(p["depth"])]
        g = [(float(log[1, b, 0]), float(log[1, b, 1])) for b in range(p["depth"])]
        t0 = min(s for s, _ in r + g)
        t1 = max(e for _, e in r + g)
        ov = overlap(r, g)
        print(f"== {name}, batch {p['batch']}: backward {t1 - t0:.3f} ms, lane R busy "
              f"{union_len(r):.3f} ms, lane G busy {union_len(g):.3f} ms, R and G concurrent "
              f"{ov:.3f} ms ({100 * ov / (t1 - t0):.1f}% of the backward)")
        print("   block   R slot [start, end] ms      G slot [start, end] ms")
        for b in range(p["depth"] - 1, -1, -1):
            print(f"   {b:5d}   [{r[b][0] - t0:8.3f}, {r[b][1] - t0:8.3f}]   "
                  f"[{g[b][0] - t0:8.3f}, {g[b][1] - t0:8.3f}]")
    eng.close()


if __name__ == "__main__":
    main()
