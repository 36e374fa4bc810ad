"""Diagnostic: run-to-run determinism of one engine mode (lr = 0).

    python tools/diag_determinism.py [mode=1] [depth=2] [width=192] [batch=2] [reps=4] [graph=0] [seq=1212]

Runs `reps` steps of one mode and prints, per parameter tensor, whether its gradient
differs from the first step's (count, index range, max diff).
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from oracle import revprop_oracle as O  # noqa: E402
from paper_2306_09342_b200.engine import Engine, ModelConfig, bf16_bits  # noqa: E402

kw = dict(mode=1, depth=2, width=192, batch=2, reps=4, graph=0, classes=100, seq="")
for a in sys.argv[1:]:
    k, v = a.split("=")
    kw[k] = v if k == "seq" else int(v)
# seq=1212 runs modes 1,2,1,2 (one step each) and compares every step with the first
modes = [int(c) for c in kw["seq"]] if kw["seq"] else [kw["mode"]] * kw["reps"]
d = kw["width"]
heads = d // 64
mc = O.ModelConfig(kw["depth"], d, heads, 4 * d, 197, 768, kw["classes"])
eng = Engine(ModelConfig(depth=kw["depth"], width=d, heads=heads, hidden=4 * d, seq_len=197,
                         num_classes=kw["classes"], batch=kw["batch"]))
p0 = O.init_params(mc, 0, np.float32)
eng.set_params(p0)
x, lab = O.synthetic_batch(mc, kw["batch"], seed=1)
eng.set_batch(bf16_bits(x), lab)
eng.set_lr(0.0)
names = [n for n, _ in O.tensor_shapes(mc)]
off, numel = eng.tensor_table()
ref = None
for r, mode in enumerate(modes):
    eng.step(mode, graph=bool(kw["graph"]))
    eng.sync()
    g = eng.grads().copy()
    if ref is None:
        ref = g
        continue
    bad = []
    for i, (o, n) in enumerate(zip(off, numel)):
        a, b = g[o:o + n], ref[o:o + n]
        nd = int(np.count_nonzero(a != b))
        if nd:
            idx = np.nonzero(a != b)[0]
            bad.append(f"{names[i]}: {nd}/{n} idx[{idx[0]}..{idx[-1]}] "
                       f"maxdiff {np.max(np.abs(a - b)):.3e} scale {np.max(np.abs(b)):.3e}")
    print(f"rep {r} (mode {mode}) vs rep 0 (mode {modes[0]}): {'IDENTICAL' if not bad else ''}", flush=True)
    for line in bad[:60]:
        print("   ", line)
print("done")
