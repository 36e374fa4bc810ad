"""Device-timed LayerNorm backward (single pass, fused dgamma | dbeta | dx column sums) at
the model shapes: RevViT-B (50432 x 768), G48 (12608 x 1664), RevViT-L (50432 x 1024),
Rev-Swin-B stages 1 / 3 (401408 x 128, 25088 x 512). us per call, one JSON line.

    RP_LIB=... python tools/ln_ab.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2306_09342_b200 import kernels as K


def t(fn, iters=30):
    for _ in range(3):
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
for rows, cols in ((50432, 768), (12608, 1664), (50432, 1024), (401408, 128), (100352, 256),
                   (25088, 512)):
    x = torch.randn(rows, cols, device="cuda")
    g = torch.rand(cols, device="cuda") + 0.5
    y = torch.empty(rows, cols, device="cuda", dtype=torch.bfloat16)
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    K.layer_norm_fwd(x, g, torch.zeros(cols, device="cuda"), 1e-5, y=y, mean=mean, rstd=rstd)
    dy = torch.randn(rows, cols, device="cuda").bfloat16()
    dres = torch.randn(rows, cols, device="cuda")
    dx = torch.empty_like(x)
    dxb = torch.empty_like(y)
    cs = torch.empty(cols, device="cuda")
    res[f"{rows}x{cols}"] = round(t(lambda: K.layer_norm_bwd(x, mean, rstd, g, dy, dres=dres, dx=dx,
                                                             dx_bf16=dxb, dx_colsum=cs)), 1)
print(json.dumps(res))
