"""Diagnostic: step-to-step determinism of the engine across mode switches (lr = 0).

Prints, for each pair of consecutive steps, which parameter tensors' gradients differ and by
how much. Used to localise state carried from one step into the next.
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from oracle import revprop_oracle as O  # noqa: E402
from paper_2306_09342_b200.engine import (REPROP, VANILLA, Engine, ModelConfig,  # noqa: E402
                                          bf16_bits)

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mc = O.ModelConfig(depth, 192, 3, 768, 197, 768, 1000)
eng = Engine(ModelConfig(depth=depth, width=192, heads=3, hidden=768, seq_len=197,
                         num_classes=1000, batch=4))
p0 = O.init_params(mc, 0, np.float32)
eng.set_params(p0)
x, lab = O.synthetic_batch(mc, 4, seed=21)
eng.set_batch(bf16_bits(x), lab)
eng.set_lr(0.0)
eng.enable_vanilla()
names = [n for n, _ in O.tensor_shapes(mc)]
off, numel = eng.tensor_table()
seq = [("r1", REPROP), ("r2", REPROP), ("v1", VANILLA), ("v2", VANILLA), ("v3", VANILLA),
       ("r3", REPROP), ("r4", REPROP), ("v4", VANILLA)]
prev = {}
for tag, mode in seq:
    eng.step(mode, graph=False)
    eng.sync()
    g = eng.grads().copy()
    assert np.array_equal(eng.params(), p0), "params changed with lr = 0"
    key = "r" if mode == REPROP else "v"
    if key in prev:
        ptag, pg = prev[key]
        bad = []
        for i, (o, n) in enumerate(zip(off, numel)):
            a, b = g[o:o + n], pg[o:o + n]
            nd = int(np.count_nonzero(a != b))
            if nd:
                idx = np.nonzero(a != b)[0]
                bad.append(f"{names[i]}: {nd}/{n} idx[{idx[0]}..{idx[-1]}] "
                           f"maxdiff {np.max(np.abs(a - b)):.3e} scale {np.max(np.abs(b)):.3e}")
        print(f"{tag} vs {ptag}: {'IDENTICAL' if not bad else ''}")
        for line in bad[:40]:
            print("   ", line)
    prev[key] = (tag, g)
print("done")
