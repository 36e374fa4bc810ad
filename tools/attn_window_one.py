"""Window attention at a Rev-Swin-B shape (default stage 3 at batch 128: 512 windows of 49
tokens, 16 heads of 32): `python tools/attn_window_one.py [S N H hd] [--time]`.
--variant=1: the general mma.sync kernels; --impl=1: mma.sync only. Without --time: two forward + backward calls (for ncu -k). With --time: CUDA-event
microseconds per forward and per backward, and the HBM floors of both (Q, K, V read +
O written; Q, K, V, dO read + dQ, dK, dV written)."""
import json
import sys

import torch

sys.path.insert(0, '.')
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--variant="):  # window kernels: 0 single-tile (default), 1 general
        _capi.lib().rp_set_attention_window_variant(int(a.split("=")[1]))
    if a.startswith("--impl="):  # rp_set_attention_impl: 0 tcgen05 where it applies, 1 mma.sync
        _capi.lib().rp_set_attention_impl(int(a.split("=")[1]))

args = [a for a in sys.argv[1:] if not a.startswith("--")]
S, N, H, hd = (int(x) for x in args) if args else (512, 49, 16, 32)
qkv = torch.randn(S * N, 3 * H * hd, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, S, N, H, head_dim=hd)
dout = torch.randn(S * N, H * hd, device="cuda").bfloat16()
dq = torch.empty_like(qkv)
if "--time" not in sys.argv:
    for _ in range(2):
        K.attention_fwd(qkv, S, N, H, head_dim=hd, out=out, lse=lse)
        K.attention_bwd(qkv, out, lse, dout, S, N, H, head_dim=hd, dqkv=dq)
    torch.cuda.synchronize()
    sys.exit(0)


def t(fn, it=50):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / it * 1e3


e = S * N * H * hd * 2  # bytes of one [tokens, H*hd] bf16 tensor
f = t(lambda: K.attention_fwd(qkv, S, N, H, head_dim=hd, out=out, lse=lse))
b = t(lambda: K.attention_bwd(qkv, out, lse, dout, S, N, H, head_dim=hd, dqkv=dq))
print(json.dumps({"shape": [S, N, H, hd], "fwd_us": round(f, 1), "bwd_us": round(b, 1),
                  "fwd_floor_us": round(4 * e / 6.55e6, 1), "bwd_floor_us": round(7 * e / 6.55e6, 1)}))
