"""BASELINE.json configs[0]: RevViT-Ti (depth 12, dim 192, 3 heads, 197 tokens), fp32, batch 8,
Reprop vs PaReprop on the CPU reference itself (oracle/_ref: the reference's ops.cpp /
layers.cpp compiled in place + the SPEC engines; PaReprop runs its recompute lane on a
second thread).

    python tools/cpu_reference_ti.py [steps]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ref as R  # noqa: E402
from oracle import revprop_oracle as O  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    mc = O.ModelConfig(12, 192, 3, 768, 197, 768, 1000)
    p = O.init_params(mc, 0, np.float32)
    x, lab = O.synthetic_batch(mc, 8, seed=1)
    x = x.astype(np.float32)
    out = {"config": "RevViT-Ti fp32 batch 8 (BASELINE configs[0])", "cpu": os.cpu_count()}
    for engine in ("reprop", "pareprop"):
        R.step(mc, p, x, lab, engine)  # warm-up
        t0 = time.perf_counter()
        for _ in range(steps):
            loss, _, _, _ = R.step(mc, p, x, lab, engine)
        dt = (time.perf_counter() - t0) / steps
        out[engine] = {"s_per_step": dt, "img_per_s": 8 / dt, "threads": 1 if engine == "reprop" else 2,
                       "loss": loss}
    out["pareprop_gain_pct"] = 100 * (out["reprop"]["s_per_step"] / out["pareprop"]["s_per_step"] - 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
