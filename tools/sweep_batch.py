"""Reprop vs PaReprop step time across per-GPU batch sizes (§3.3: the gain comes
from GPU under-utilisation, largest at small batch).

    python tools/sweep_batch.py [--batches 8,16,32,64,128,256]
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import argparse
import json

from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig
from sweep_partition import time_steps


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="revvit-b")
    ap.add_argument("--batches", default="8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--priorities", default="1,0")
    a = ap.parse_args(argv)
    for B in [int(x) for x in a.batches.split(",")]:
        for prio in [int(x) for x in a.priorities.split(",")]:
            p = dict(PRESETS[a.preset], batch=B)
            eng = Engine(ModelConfig(lane_priority=prio, **p))
            eng.set_lr(1e-4)
            r = time_steps(eng, REPROP, a.steps)
            q = time_steps(eng, PAREPROP, a.steps)
            print(json.dumps({"batch": B, "lane_priority": prio, "reprop_ms": r,
                              "pareprop_ms": q, "reprop_img_s": B * 1e3 / r,
                              "pareprop_img_s": B * 1e3 / q,
                              "gain_pct": 100 * (r / q - 1)}), flush=True)
            eng.close()


if __name__ == "__main__":
    main()
