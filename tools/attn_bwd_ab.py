"""Interleaved same-box A/B of the attention backward implementations (CUDA events, us per
call) at the model shapes, with the max |difference| between implementations' d_qkv.
    python tools/attn_bwd_ab.py [impl ...]     (default: 3 0, i.e. dS^T round trip vs fused)"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

lib = _capi.lib()
impls = [int(x) for x in sys.argv[1:]] or [3, 0]


def t(fn, it=20):
    for _ in range(3):
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


for (B, N, H) in [(256, 197, 12), (256, 197, 16), (64, 197, 12), (64, 512, 12)]:
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, N, H)
    dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
    dq = torch.empty_like(qkv)
    res = {i: [] for i in impls}
    outs = {}
    for rep in range(3):  # interleaved
        for impl in impls:
            lib.rp_set_attention_impl(impl)
            res[impl].append(t(lambda: K.attention_bwd(qkv, out, lse, dout, B, N, H, dqkv=dq)))
            outs[impl] = dq.clone()
    lib.rp_set_attention_impl(0)
    ref = outs[impls[0]].float()
    line = " ".join("impl%d %.1f us (maxdiff %.3g)" % (i, min(res[i]), (outs[i].float() - ref).abs().max().item())
                    for i in impls)
    print(B, N, H, line, flush=True)
