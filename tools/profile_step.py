"""One RevViT-B training step under cudaProfilerStart/Stop, for ncu:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/profile_step.py --mode reprop
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import argparse

import torch

from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["reprop", "pareprop"], default="reprop")
    ap.add_argument("--preset", default="revvit-b")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--depth", type=int, default=0)
    a = ap.parse_args(argv)
    p = dict(PRESETS[a.preset])
    if a.batch:
        p["batch"] = a.batch
    if a.depth:
        p["depth"] = a.depth
    eng = Engine(ModelConfig(**p))
    mode = REPROP if a.mode == "reprop" else PAREPROP
    for _ in range(2):
        eng.step(mode, graph=False)
    eng.sync()
    torch.cuda.cudart().cudaProfilerStart()
    eng.step(mode, graph=False)
    eng.sync()
    torch.cuda.cudart().cudaProfilerStop()
    print("loss", eng.loss())


if __name__ == "__main__":
    main()
