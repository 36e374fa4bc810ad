"""Launch each hot kernel once at the RevViT-B block shapes (T = 256*197), for ncu:

    ncu --set full -k regex:<kernel> -c 1 python tools/ncu_targets.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch

from paper_2306_09342_b200 import _capi, kernels as K
from paper_2306_09342_b200._capi import (RP_EPI_BF16, RP_EPI_BIAS_GELU, RP_EPI_BIAS_GELU_SLOPE, RP_EPI_F32, RP_EPI_MUL,
                    RP_EPI_RESID)


def main():
    _capi.lib()
    B, N, d, h, H = 256, 197, 768, 3072, 12
    T = B * N
    bf = torch.bfloat16
    dev = "cuda"
    qkv = torch.randn(T, 3 * d, device=dev).to(bf)
    att = torch.empty(T, d, device=dev, dtype=bf)
    lse = torch.empty(B, H, N, device=dev)
    dO = torch.randn(T, d, device=dev).to(bf)
    x = torch.randn(T, d, device=dev).to(bf)
    x3 = torch.randn(T, h, device=dev).to(bf)
    W1 = (0.02 * torch.randn(d, h, device=dev)).to(bf)
    W2 = (0.02 * torch.randn(h, d, device=dev)).to(bf)
    res = torch.randn(T, d, device=dev)
    a = torch.empty(T, h, device=dev, dtype=bf)
    u = torch.empty(T, h, device=dev, dtype=bf)
    b1 = torch.zeros(h, device=dev)
    xf = torch.randn(T, d, device=dev)
    g = torch.ones(d, device=dev)
    bt = torch.zeros(d, device=dev)
    qkv_out = torch.empty(T, 3 * d, device=dev, dtype=bf)
    Wqkv = (0.02 * torch.randn(d, 3 * d, device=dev)).to(bf)
    part = torch.empty((T + 31) // 32, h, device=dev)
    dW = torch.empty(d, h, device=dev)
    ws = torch.empty(8 * d * h, device=dev)
    for _ in range(2):  # second iteration is the profiled one under -s/-c filters
        K.attention_fwd(qkv, B, N, H, out=att, lse=lse)
        K.attention_bwd(qkv, att, lse, dO, B, N, H)
        # the engine's GEMM set (CTA-pair 256 x 256 tiles, bn=512)
        K.gemm(x, Wqkv, T, 3 * d, d, a_mn=0, b_mn=1, epi=RP_EPI_BF16, out=qkv_out, bn=512)
        K.gemm(x, W1, T, h, d, a_mn=0, b_mn=1, epi=RP_EPI_BIAS_GELU, out=a, bias=b1, bn=512)
        K.gemm(x, W1, T, h, d, a_mn=0, b_mn=1, epi=RP_EPI_BIAS_GELU_SLOPE, out=a, out2=u,
               bias=b1, bn=512)
        K.gemm(x3, W2, T, d, h, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=res, aux=res, bn=512)
        K.gemm(x, W2, T, h, d, a_mn=0, b_mn=0, epi=RP_EPI_MUL, out=a, aux=u, colsum_part=part,
               bn=512)
        K.gemm(x3, W1, T, d, h, a_mn=0, b_mn=0, epi=RP_EPI_BF16, out=x, bn=512)
        K.gemm(x, a, d, h, T, a_mn=1, b_mn=1, epi=RP_EPI_F32, out=dW, splits=4, workspace=ws,
               bn=512)
        y, mean, rstd = K.layer_norm_fwd(xf, g, bt)
        K.layer_norm_bwd(xf, mean, rstd, g, y, dres=res, dx=res)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
