"""A/B of the tcgen05 attention forward kernels at the BASELINE shapes (CUDA events).

    python tools/attn_fwd_ab.py          # current default kernel
    RP_ATTN_FWD_DUAL=1 python tools/attn_fwd_ab.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import kernels as K  # noqa: E402


def t(fn, it=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / it * 1e3


for (B, N, H) in [(256, 197, 12), (256, 197, 16), (64, 128, 12), (128, 224, 12)]:
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, N, H)
    us = t(lambda: K.attention_fwd(qkv, B, N, H, out=out, lse=lse))
    q, k, v = qkv.float().view(B, N, 3, H, 64).permute(2, 0, 3, 1, 4)
    s = (q @ k.transpose(-1, -2)) / 8.0
    ref = (torch.softmax(s, -1) @ v).permute(0, 2, 1, 3).reshape(B * N, H * 64)
    err = ((out.float() - ref).norm() / ref.norm()).item()
    lerr = ((lse / 1.4426950408889634 - torch.logsumexp(s, -1)).abs().max()).item()
    print(f"{B} {N} {H}: {us:.1f} us  rel err {err:.2e}  lse err {lerr:.2e}")
