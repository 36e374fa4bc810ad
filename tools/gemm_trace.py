"""clock64 timeline of the CTA-pair GEMM's cluster 0 at the RevViT-B shapes
(rp_set_gemm_trace): per tile, whether the MMA warp waited for the accumulator (epilogue-
bound) or for operand stages (load-bound), and how long the epilogue took.

    python tools/gemm_trace.py
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

L = _capi.lib()
T, d, h = 256 * 197, 768, 3072
dev = "cuda"
torch.manual_seed(0)
x = torch.randn(T, d, device=dev).bfloat16()
w1 = (torch.randn(d, h, device=dev) * 0.03).bfloat16()
wq = (torch.randn(d, 3 * d, device=dev) * 0.03).bfloat16()
w2 = (torch.randn(h, d, device=dev) * 0.03).bfloat16()
x3 = torch.randn(T, h, device=dev).bfloat16()
b1 = torch.randn(h, device=dev) * 0.1
o1 = torch.empty(T, h, device=dev, dtype=torch.bfloat16)
o2 = torch.empty_like(o1)
oq = torch.empty(T, 3 * d, device=dev, dtype=torch.bfloat16)
od = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
res = torch.randn(T, d, device=dev)
dyb = torch.randn(T, h, device=dev).bfloat16()
ws = torch.empty(8 * d * h, device=dev)
dW = torch.empty(d, h, device=dev)
cases = {
    "resid fp32 K=3072": lambda: K.gemm(x3, w2, T, d, h, b_mn=True, epi=_capi.RP_EPI_RESID, out=res,
                                         aux=res, bn=512),
    "resid fp32 K=768": lambda: K.gemm(x, wq[:, :d].contiguous(), T, d, d, b_mn=True,
                                        epi=_capi.RP_EPI_RESID, out=res, aux=res, bn=512),
    "wgrad split-K": lambda: K.gemm(x, dyb, d, h, T, a_mn=True, b_mn=True, epi=_capi.RP_EPI_F32,
                                    out=dW, splits=4, workspace=ws, bn=512),
    "qkv_bf16 K=768": lambda: K.gemm(x, wq, T, 3 * d, d, b_mn=True, epi=_capi.RP_EPI_BF16, out=oq, bn=512),
    "gelu_slope K=768": lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=_capi.RP_EPI_BIAS_GELU_SLOPE,
                                       out=o1, out2=o2, bias=b1, bn=512),
    "dgrad bf16 K=3072": lambda: K.gemm(x3, w1, T, d, h, b_mn=False, epi=_capi.RP_EPI_BF16, out=od, bn=512),
}
buf = torch.zeros(64 * 8, dtype=torch.int64, device=dev)
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    buf.zero_()
    L.rp_set_gemm_trace(C.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    L.rp_set_gemm_trace(None)
    t = buf.view(64, 8).cpu().numpy().astype(np.int64)
    n = int((t[:, 1] > 0).sum())
    t = t[2:n - 1]
    per = np.diff(t[:, 1])
    acc_wait = t[:, 1] - t[:, 0]
    mma_span = t[:, 3] - t[:, 1]
    full_wait = t[:, 2]
    epi = t[:, 5] - t[:, 4]
    print(f"{name}: tiles {n}, median cycles per tile {np.median(per):.0f} | MMA warp: waits for "
          f"accumulator {np.median(acc_wait):.0f}, issue span {np.median(mma_span):.0f} of which "
          f"waiting for operands {np.median(full_wait):.0f} | epilogue {np.median(epi):.0f}")
