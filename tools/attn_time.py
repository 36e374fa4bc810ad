"""CUDA-event time of the attention forward / backward at the RevViT-B/L shapes with the
library in RP_LIB (for interleaved A/B of two builds: tools/ab_libs.sh)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import kernels as K  # noqa: E402


def t(fn, it=30):
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


out = []
for (B, N, H) in [(256, 197, 12), (256, 197, 16)]:
    torch.manual_seed(0)
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    o, lse = K.attention_fwd(qkv, B, N, H)
    dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
    dq = torch.empty_like(qkv)
    tf = t(lambda: K.attention_fwd(qkv, B, N, H, out=o, lse=lse))
    tb = t(lambda: K.attention_bwd(qkv, o, lse, dout, B, N, H, dqkv=dq))
    out.append(f"{B}x{N}x{H} fwd {tf:.1f} bwd {tb:.1f}")
print(" | ".join(out))
