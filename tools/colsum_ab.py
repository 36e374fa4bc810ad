"""Device-timed column-sum reductions at the engine's shapes (RevViT-B, batch 256):
the d_u GEMM's per-32-row partials -> db1 (1576 x 3072) and the LayerNorm backward's
per-64-row dgamma|dbeta partials (788 x 1536); Rev-Swin-B (batch 128) stage shapes after. Prints one JSON line of us per call.

    RP_LIB=... python tools/colsum_ab.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2306_09342_b200 import kernels as K


def t(fn, iters=200):
    for _ in range(10):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / iters


res = {}
for n, c in ((1576, 3072), (788, 1536), (12544, 512), (3136, 1024), (6272, 256), (784, 2048)):
    part = torch.randn(n, c, device="cuda")
    out = torch.zeros(c, device="cuda")
    res[f"{n}x{c}"] = round(t(lambda: K.colsum_parts(part, out=out)), 2)
print(json.dumps(res))
