import torch, sys
sys.path.insert(0, '.')
from paper_2306_09342_b200 import _capi, kernels as K
lib = _capi.lib()
def t(fn, it=20):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / it * 1e3
for (B, N, H) in [(256, 197, 12), (64, 512, 12), (256, 197, 16)]:
    qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, N, H)
    dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
    dq = torch.empty_like(qkv)
    res = {}
    for impl in (2, 0):
        lib.rp_set_attention_impl(impl)
        res[impl] = t(lambda: K.attention_bwd(qkv, out, lse, dout, B, N, H, dqkv=dq))
        r = dq.clone()
        if impl == 0:
            print(B, N, H, "two-pass %.1f us, fused %.1f us" % (res[2], res[0]),
                  "max|diff| vs two-pass", (r.float() - r2.float()).abs().max().item())
        r2 = r
    lib.rp_set_attention_impl(0)
