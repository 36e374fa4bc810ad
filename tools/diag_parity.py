"""Diagnostic: per-tensor gradient error of one engine step vs the f64 oracle.

    python tools/diag_parity.py depth=2 width=128 heads=2 hidden=512 seq_len=64 in_dim=256 \
        num_classes=7 window=16 batch=4
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from oracle import revprop_oracle as O  # noqa: E402
from paper_2306_09342_b200.engine import (REPROP, Engine, ModelConfig, bf16_bits,  # noqa: E402
                                          bf16_round)

kw = dict(depth=2, width=128, heads=2, hidden=512, seq_len=64, in_dim=256, num_classes=7,
          window=0, batch=4, seed=8)
for a in sys.argv[1:]:
    k, v = a.split("=")
    kw[k] = int(v)
B, seed = kw.pop("batch"), kw.pop("seed")
cfg = ModelConfig(**kw, batch=B)
eng = Engine(cfg)
mc = O.ModelConfig(cfg.depth, cfg.width, cfg.heads, cfg.hidden, cfg.seq_len, cfg.in_dim,
                   cfg.num_classes, cfg.window or None)
p32 = O.init_params(mc, 0, np.float32)
eng.set_params(p32)
pref = p32.astype(np.float64)
off = 0
for name, shape in O.tensor_shapes(mc):
    n = int(np.prod(shape))
    if len(shape) == 2:
        pref[off:off + n] = bf16_round(p32[off:off + n])
    off += n
x, lab = O.synthetic_batch(mc, B, seed=seed)
eng.set_batch(bf16_bits(x), lab)
eng.set_lr(0.0)
eng.step(REPROP, graph=False)
g = eng.grads()
r = O.step(mc, pref, bf16_round(x).astype(np.float64), lab)
print(f"loss gpu {eng.loss():.7f} oracle {r.loss:.7f}")
off = 0
for name, shape in O.tensor_shapes(mc):
    n = int(np.prod(shape))
    a, b = g[off:off + n].astype(np.float64), r.grads[off:off + n]
    mr = np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)
    l2 = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    print(f"{name:24s} maxrel {mr:.3e} l2rel {l2:.3e} scale {np.max(np.abs(b)):.3e}")
    off += n
