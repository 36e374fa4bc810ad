"""CUDA-event timing of one CTA-pair GEMM per fused epilogue at the RevViT-B MLP shapes
(T = 256 x 197 tokens), for same-box A/B of epilogue plans (RP_LIB alternation)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402


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


T, d, h = 256 * 197, 768, 3072
dev = "cuda"
x = torch.randn(T, d, device=dev).bfloat16()
w1 = (torch.randn(d, h, device=dev) * 0.03).bfloat16()
b1 = torch.randn(h, device=dev) * 0.1
o1 = torch.empty(T, h, device=dev, dtype=torch.bfloat16)
o2 = torch.empty_like(o1)
res = {}
x3 = torch.randn(T, h, device=dev).bfloat16()
w2 = (torch.randn(h, d, device=dev) * 0.03).bfloat16()
dy = torch.randn(T, d, device=dev).bfloat16()
part = torch.empty((T + 31) // 32, h, device=dev)
res["bias_gelu_slope"] = t(lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BIAS_GELU_SLOPE,
                                         out=o1, out2=o2, bias=b1, bn=512))
res["bias_gelu"] = t(lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BIAS_GELU,
                                   out=o1, bias=b1, bn=512))
res["slope_mul"] = t(lambda: K.gemm(dy, w2, T, h, d, b_mn=False, epi=_capi.RP_EPI_MUL, out=o1, aux=o2,
                                   colsum_part=part, bn=512))
res["bf16"] = t(lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BF16, out=o1, bn=512))
wo = (torch.randn(d, d, device=dev) * 0.03).bfloat16()
xr = torch.randn(T, d, device=dev)
res["resid_proj"] = t(lambda: K.gemm(x, wo, T, d, d, b_mn=True, epi=_capi.RP_EPI_RESID, out=xr,
                                    aux=xr, bn=512))
res["resid_w2"] = t(lambda: K.gemm(x3, w2, T, d, h, b_mn=True, epi=_capi.RP_EPI_RESID, out=xr,
                                  aux=xr, bn=512))
print(" ".join(f"{k} {v:.1f}us" for k, v in res.items()))
