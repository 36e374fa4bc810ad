"""A/B of the tcgen05 attention forward variants at the BASELINE shapes (CUDA events,
interleaved per shape so both variants see the same clocks).

    python tools/attn_fwd_ab.py [reps]
variant 0 = ping-pong softmax groups with the split P V (default), 2 = ping-pong with one
P V issuer, 1 = lockstep persistent kernel.
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi  # noqa: E402
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


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L = _capi.lib()
for (B, N, H) in [(256, 197, 12), (256, 197, 16), (64, 128, 12), (128, 224, 12), (64, 256, 12),
                  (8, 197, 3), (3, 1, 2), (2, 130, 3)]:
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    q, k, v = qkv.float().view(B, N, 3, H, 64).permute(2, 0, 3, 1, 4)
    s = (q @ k.transpose(-1, -2)) / 8.0
    ref = (torch.softmax(s, -1) @ v).permute(0, 2, 1, 3).reshape(B * N, H * 64)
    res = {}
    for _ in range(reps):
        for var in (0, 2, 1):
            if var == 1 and N > 224:
                continue
            L.rp_set_attention_fwd_variant(var)
            out, lse = K.attention_fwd(qkv, B, N, H)
            us = t(lambda: K.attention_fwd(qkv, B, N, H, out=out, lse=lse))
            err = ((out.float() - ref).norm() / ref.norm()).item()
            lerr = ((lse / 1.4426950408889634 - torch.logsumexp(s, -1)).abs().max()).item()
            res.setdefault(var, []).append((us, err, lerr))
    L.rp_set_attention_fwd_variant(0)
    flops = 4 * B * H * N * N * 64
    line = f"{B:4d} {N:4d} {H:3d}:"
    for var, r in sorted(res.items()):
        us = min(x[0] for x in r)
        line += f"  v{var} {us:7.1f} us ({flops / us / 1e6:6.1f} TF/s) err {r[0][1]:.1e} lse {r[0][2]:.1e}"
    print(line, flush=True)
