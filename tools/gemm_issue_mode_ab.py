"""Same-process A/B of the GEMM MMA issue form (rp_set_mma_issue 1 converged / 0 one lane)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

L = _capi.lib()


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


T, d, h = 256 * 197, 768, 3072
dev = "cuda"
x = torch.randn(T, d, device=dev).bfloat16()
w1 = (torch.randn(d, h, device=dev) * 0.03).bfloat16()
b1 = torch.randn(h, device=dev) * 0.1
o1 = torch.empty(T, h, device=dev, dtype=torch.bfloat16)
o2 = torch.empty_like(o1)
cases = {
    "gelu_slope": lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BIAS_GELU_SLOPE, out=o1,
                                 out2=o2, bias=b1, bn=512),
    "bias_gelu": lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BIAS_GELU, out=o1, bias=b1,
                                bn=512),
    "bf16": lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BF16, out=o1, bn=512),
}
res = {}
for rep in range(3):
    for m in (1, 0):
        L.rp_set_mma_issue(m)
        for k, fn in cases.items():
            res.setdefault((k, m), []).append(t(fn))
L.rp_set_mma_issue(1)
print(" | ".join(f"{k}: converged {min(res[(k, 1)]):.1f} / one lane {min(res[(k, 0)]):.1f} us" for k in cases))
