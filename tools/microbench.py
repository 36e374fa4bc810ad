"""Per-kernel timing of the RevViT-B block shapes (T = 256*197 rows, d = 768, h = 3072).

    python tools/microbench.py [--json out.json]

Times every sm_100a kernel of one reversible block with CUDA events (warm-up, then the
median of repeated launches on one stream) and reports TFLOP/s or GB/s against
MEASURED_PEAKS.json. torch.matmul (cuBLAS) on the same shapes is printed beside the GEMMs
as a library yardstick only; it is never on the product path.
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import argparse
import json
import os

import torch

from paper_2306_09342_b200 import _capi, kernels as K
from paper_2306_09342_b200._capi import RP_EPI_BF16, RP_EPI_BIAS_GELU, RP_EPI_F32, RP_EPI_GELU_BWD, RP_EPI_RESID


def _peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["bf16_tflops"], d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 6650.0, "fallback"


def timeit(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args(argv)
    _capi.lib()
    torch.backends.cuda.matmul.allow_tf32 = False
    tf_peak, gbs_peak, src = _peaks()
    dev = "cuda"
    B, N, d, h, H = a.batch, 197, 768, 3072, 12
    T = B * N
    bf = torch.bfloat16
    x = torch.randn(T, d, device=dev).to(bf)
    x3 = torch.randn(T, h, device=dev).to(bf)
    Wqkv = (0.02 * torch.randn(d, 3 * d, device=dev)).to(bf)
    Wo = (0.02 * torch.randn(d, d, device=dev)).to(bf)
    W1 = (0.02 * torch.randn(d, h, device=dev)).to(bf)
    W2 = (0.02 * torch.randn(h, d, device=dev)).to(bf)
    b1 = torch.zeros(h, device=dev)
    b2 = torch.zeros(d, device=dev)
    res = torch.randn(T, d, device=dev)
    rows = []

    def gemm_row(name, M, Nn, Kk, fn, torch_fn=None):
        ms = timeit(fn)
        tf = 2.0 * M * Nn * Kk / ms / 1e9
        r = {"kernel": name, "M": M, "N": Nn, "K": Kk, "ms": ms, "tflops": tf,
             "frac": tf / tf_peak}
        if torch_fn is not None:
            tms = timeit(torch_fn)
            r["cublas_ms"] = tms
            r["cublas_tflops"] = 2.0 * M * Nn * Kk / tms / 1e9
        rows.append(r)
        print(json.dumps(r))

    # forward / recompute
    qkv = torch.empty(T, 3 * d, device=dev, dtype=bf)
    gemm_row("fwd_qkv", T, 3 * d, d,
             lambda: K.gemm(x, Wqkv, T, 3 * d, d, a_mn=0, b_mn=1, epi=RP_EPI_BF16, out=qkv),
             lambda: torch.matmul(x, Wqkv))
    yo = torch.empty(T, d, device=dev)
    gemm_row("fwd_proj_resid", T, d, d,
             lambda: K.gemm(x, Wo, T, d, d, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=yo, aux=res),
             lambda: torch.matmul(x, Wo))
    aa = torch.empty(T, h, device=dev, dtype=bf)
    uu = torch.empty(T, h, device=dev, dtype=bf)
    gemm_row("fwd_w1_gelu", T, h, d,
             lambda: K.gemm(x, W1, T, h, d, a_mn=0, b_mn=1, epi=RP_EPI_BIAS_GELU, out=aa,
                            out2=uu, bias=b1),
             lambda: torch.matmul(x, W1))
    gemm_row("fwd_w2_resid", T, d, h,
             lambda: K.gemm(x3, W2, T, d, h, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=yo, aux=res,
                            bias=b2),
             lambda: torch.matmul(x3, W2))
    # the same forward shapes on CTA pairs (cta_group::2, 256x256 tiles)
    gemm_row("fwd_qkv_2sm", T, 3 * d, d,
             lambda: K.gemm(x, Wqkv, T, 3 * d, d, a_mn=0, b_mn=1, epi=RP_EPI_BF16, out=qkv, bn=512))
    gemm_row("fwd_w1_gelu_2sm", T, h, d,
             lambda: K.gemm(x, W1, T, h, d, a_mn=0, b_mn=1, epi=RP_EPI_BIAS_GELU, out=aa,
                            out2=uu, bias=b1, bn=512))
    gemm_row("fwd_w2_resid_2sm", T, d, h,
             lambda: K.gemm(x3, W2, T, d, h, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=yo, aux=res,
                            bias=b2, bn=512))
    gemm_row("fwd_proj_resid_2sm", T, d, d,
             lambda: K.gemm(x, Wo, T, d, d, a_mn=0, b_mn=1, epi=RP_EPI_RESID, out=yo, aux=res,
                            bn=512))
    # dgrad
    du = torch.empty(T, h, device=dev, dtype=bf)
    gemm_row("dgrad_w2_gelu", T, h, d,
             lambda: K.gemm(x, W2, T, h, d, a_mn=0, b_mn=0, epi=RP_EPI_GELU_BWD, out=du, aux=uu),
             lambda: torch.matmul(x, W2.t()))
    dh = torch.empty(T, d, device=dev, dtype=bf)
    gemm_row("dgrad_w1", T, d, h,
             lambda: K.gemm(x3, W1, T, d, h, a_mn=0, b_mn=0, epi=RP_EPI_BF16, out=dh),
             lambda: torch.matmul(x3, W1.t()))
    gemm_row("dgrad_qkv", T, d, 3 * d,
             lambda: K.gemm(qkv, Wqkv, T, d, 3 * d, a_mn=0, b_mn=0, epi=RP_EPI_BF16, out=dh),
             lambda: torch.matmul(qkv, Wqkv.t()))
    # wgrad (split-K)
    gemm_row("dgrad_w2_gelu_2sm", T, h, d,
             lambda: K.gemm(x, W2, T, h, d, a_mn=0, b_mn=0, epi=RP_EPI_GELU_BWD, out=du, aux=uu,
                            bn=512))
    gemm_row("dgrad_w1_2sm", T, d, h,
             lambda: K.gemm(x3, W1, T, d, h, a_mn=0, b_mn=0, epi=RP_EPI_BF16, out=dh, bn=512))
    for name, A_, B_, M, Nn, splits, bnn in [
            ("wgrad_w1", x, x3, d, h, 2, 256), ("wgrad_w2", x3, x, h, d, 2, 256),
            ("wgrad_qkv", x, qkv, d, 3 * d, 8, 256), ("wgrad_proj", x, x, d, d, 8, 256),
            ("wgrad_w1_2sm", x, x3, d, h, 4, 512), ("wgrad_w2_2sm", x3, x, h, d, 4, 512),
            ("wgrad_qkv_2sm", x, qkv, d, 3 * d, 8, 512), ("wgrad_proj_2sm", x, x, d, d, 16, 512)]:
        o = torch.empty(M, Nn, device=dev)
        ws = torch.empty(splits * M * Nn, device=dev)
        gemm_row(f"{name}_s{splits}", M, Nn, T,
                 lambda A_=A_, B_=B_, M=M, Nn=Nn, o=o, ws=ws, s=splits, bnn=bnn: K.gemm(
                     A_, B_, M, Nn, T, a_mn=1, b_mn=1, epi=RP_EPI_F32, out=o, splits=s,
                     workspace=ws, bn=bnn),
                 lambda A_=A_, B_=B_: torch.matmul(A_.t(), B_))

    # memory-bound kernels
    def mem_row(name, nbytes, fn):
        ms = timeit(fn)
        gbs = nbytes / ms / 1e6
        r = {"kernel": name, "ms": ms, "gbs": gbs, "frac": gbs / gbs_peak, "bytes": nbytes}
        rows.append(r)
        print(json.dumps(r))

    xf = torch.randn(T, d, device=dev)
    gamma = torch.ones(d, device=dev)
    beta = torch.zeros(d, device=dev)
    hb = torch.empty(T, d, device=dev, dtype=bf)
    mean = torch.empty(T, device=dev)
    rstd = torch.empty(T, device=dev)
    mem_row("ln_fwd", T * d * 6 + T * 8,
            lambda: K.layer_norm_fwd(xf, gamma, beta, 1e-5, y=hb, mean=mean, rstd=rstd))
    dx = torch.empty(T, d, device=dev)
    dxb = torch.empty(T, d, device=dev, dtype=bf)
    mem_row("ln_bwd", T * d * (4 + 2 + 4 + 4 + 2) + T * 8,
            lambda: K.layer_norm_bwd(xf, mean, rstd, gamma, hb, dres=res, dx=dx, dx_bf16=dxb))
    mem_row("colsum_bf16_h", T * h * 2, lambda: K.colsum(du))
    # attention
    att = torch.empty(T, d, device=dev, dtype=bf)
    lse = torch.empty(B, H, N, device=dev)
    fl = 4.0 * B * H * N * N * 64
    ms = timeit(lambda: K.attention_fwd(qkv, B, N, H, out=att, lse=lse))
    r = {"kernel": "attn_fwd", "ms": ms, "tflops": fl / ms / 1e9}
    rows.append(r)
    print(json.dumps(r))
    dq = torch.empty_like(qkv)
    ms = timeit(lambda: K.attention_bwd(qkv, att, lse, hb, B, N, H, dqkv=dq))
    r = {"kernel": "attn_bwd", "ms": ms, "tflops": 2.5 * fl / ms / 1e9}
    rows.append(r)
    print(json.dumps(r))
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"peaks": {"bf16_tflops": tf_peak, "hbm_gbs": gbs_peak, "source": src},
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
