"""Same-process A/B of whole-step time: Reprop / PaReprop x PDL on / off, or x window-attention
kernels 0 / 1 with --window (device-timed, CUDA graphs), so clock / power-cap drift between
boxes does not enter the comparison.

    python tools/ab_step.py [--rounds 3]
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import argparse
import json

from paper_2306_09342_b200 import _capi
from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig
from sweep_partition import time_steps


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="revvit-b")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--window", action="store_true",
                    help="A/B the window-attention kernels (variant 0 vs 1) instead of PDL")
    a = ap.parse_args(argv)
    p = dict(PRESETS[a.preset])
    if a.batch:
        p["batch"] = a.batch
    eng = Engine(ModelConfig(**p))
    eng.set_lr(1e-4)
    res = {}
    for r in range(a.rounds):
        for v in (1, 0):
            if a.window:
                _capi.lib().rp_set_attention_window_variant(v)
                tag = f"win{v}"
            else:
                _capi.lib().rp_set_pdl(v)
                tag = f"pdl{v}"
            eng.invalidate_graphs()
            for mode, name in ((REPROP, "reprop"), (PAREPROP, "pareprop")):
                ms = time_steps(eng, mode, a.steps)
                res.setdefault(f"{name}_{tag}", []).append(ms)
    _capi.lib().rp_set_pdl(0)
    _capi.lib().rp_set_attention_window_variant(0)
    B = p["batch"]
    out = {k: {"ms": min(v), "img_s": B * 1e3 / min(v)} for k, v in res.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
