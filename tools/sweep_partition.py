"""PaReprop SM-partition sweep: step time of Reprop and of PaReprop with the recompute
lane's GEMMs capped at r CTAs and the gradient lane's at g CTAs (device-timed, CUDA graphs).

    python tools/sweep_partition.py [--steps 10]
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import argparse
import json

import torch

from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig


def time_steps(eng, mode, K):
    s = torch.cuda.ExternalStream(eng.stream_ptr)
    for _ in range(3):
        eng.step(mode)
    eng.sync()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        eng.step(mode)
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / K


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--preset", default="revvit-b")
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args(argv)
    p = dict(PRESETS[a.preset])
    if a.batch:
        p["batch"] = a.batch
    eng = Engine(ModelConfig(**p))
    eng.set_lr(1e-4)
    B = p["batch"]
    res = {"reprop_ms": time_steps(eng, REPROP, a.steps)}
    print(json.dumps({"mode": "reprop", "ms": res["reprop_ms"], "img_s": B * 1e3 / res["reprop_ms"]}))
    for r, g in [(0, 0), (48, 100), (64, 84), (74, 74), (32, 116), (100, 48)]:
        eng.set_partition(r, g)
        ms = time_steps(eng, PAREPROP, a.steps)
        print(json.dumps({"mode": "pareprop", "r_ctas": r, "g_ctas": g, "ms": ms,
                          "img_s": B * 1e3 / ms, "gain_pct": 100 * (res["reprop_ms"] / ms - 1)}))


if __name__ == "__main__":
    main()
