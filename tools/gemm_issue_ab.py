"""A/B of the GEMM MMA issue form (rp_set_mma_issue: 1 warp-converged predicated issue,
0 one diverged lane) on the RevViT-B GEMM shapes, interleaved on one box; outputs compared
bit for bit between the two forms.

    python tools/gemm_issue_ab.py [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402


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


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L = _capi.lib()
T, d, h = 256 * 197, 768, 3072
dev = "cuda"
x = torch.randn(T, d, device=dev).bfloat16()
a = torch.randn(T, h, device=dev).bfloat16()
w1 = (torch.randn(d, h, device=dev) * 0.03).bfloat16()
w2 = (torch.randn(h, d, device=dev) * 0.03).bfloat16()
wq = (torch.randn(d, 3 * d, device=dev) * 0.03).bfloat16()
b1 = torch.randn(h, device=dev) * 0.1
b2 = torch.randn(d, device=dev) * 0.1
res = torch.randn(T, d, device=dev)
o_h = torch.empty(T, h, device=dev, dtype=torch.bfloat16)
o_h2 = torch.empty_like(o_h)
o_q = torch.empty(T, 3 * d, device=dev, dtype=torch.bfloat16)
o_d = torch.empty(T, d, device=dev)
o_db = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
g_w1 = torch.empty(d, h, device=dev)
ws = torch.empty(8 * d * h, device=dev)
E = _capi
cases = {
    "qkv bf16 (K=768)": (2 * T * d * 3 * d, lambda: K.gemm(x, wq, T, 3 * d, d, b_mn=True, epi=E.RP_EPI_BF16, out=o_q, bn=512), o_q),
    "w1 bias+gelu+slope": (2 * T * d * h, lambda: K.gemm(x, w1, T, h, d, b_mn=True, epi=E.RP_EPI_BIAS_GELU_SLOPE, out=o_h, out2=o_h2, bias=b1, bn=512), o_h),
    "w2 resid (K=3072)": (2 * T * h * d, lambda: K.gemm(a, w2, T, d, h, b_mn=True, epi=E.RP_EPI_RESID, out=o_d, aux=res, bias=b2, bn=512), o_d),
    "dgrad du.W1^T bf16": (2 * T * h * d, lambda: K.gemm(a, w1, T, d, h, b_mn=False, epi=E.RP_EPI_BF16, out=o_db, bn=512), o_db),
    "wgrad x^T a split4": (2 * T * d * h, lambda: K.gemm(x, a, d, h, T, a_mn=True, b_mn=True, epi=E.RP_EPI_F32, out=g_w1, splits=4, workspace=ws, bn=512), g_w1),
}
out = {}
for _ in range(reps):
    for name, (fl, fn, o) in cases.items():
        for mode in (0, 1):
            L.rp_set_mma_issue(mode)
            us = t(fn)
            r = out.setdefault(name, {}).setdefault(mode, [1e9, None])
            r[0] = min(r[0], us)
            r[1] = o.clone()
L.rp_set_mma_issue(1)
for name, (fl, fn, o) in cases.items():
    r0, r1 = out[name][0], out[name][1]
    same = torch.equal(r0[1], r1[1])
    print(f"{name:24s} lane {r0[0]:7.1f} us {fl / r0[0] / 1e6:6.0f} TF/s | converged {r1[0]:7.1f} us "
          f"{fl / r1[0] / 1e6:6.0f} TF/s | bit-identical {same}", flush=True)
