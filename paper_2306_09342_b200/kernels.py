"""Thin torch-tensor front end over the C ABI kernels (device memory comes from torch;
the arithmetic is the sm_100a library's). Used by the parity tests and the layer-level
Python mirror; the training engine itself calls the same launchers from C++.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi
from ._capi import GemmDesc, check, lib


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _req(t, dtype, name):
    if t.device.type != "cuda":
        raise _capi.ContractError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise _capi.ShapeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise _capi.ShapeError(f"{name}: expected a contiguous tensor")


def gemm(A, B, M, N, K, *, a_mn=False, b_mn=False, epi=_capi.RP_EPI_BF16, out=None,
         out2=None, aux=None, bias=None, sign=1.0, splits=1, workspace=None, max_ctas=0,
         bn=256, lda=None, ldb=None, ldo=None, ldo2=None, ldaux=None, colsum_part=None,
         rowdot=None, rd_seq=0, stream=None):
    """C[M,N] = A.B on the tcgen05 path. A is [M,K] (a_mn=False) or [K,M] (a_mn=True);
    B is [N,K] (b_mn=False) or [K,N] (b_mn=True)."""
    d = GemmDesc()
    d.A, d.B = A.data_ptr(), B.data_ptr()
    d.lda = lda if lda is not None else A.shape[-1]
    d.ldb = ldb if ldb is not None else B.shape[-1]
    d.a_mn, d.b_mn = int(a_mn), int(b_mn)
    d.M, d.N, d.K = M, N, K
    d.epi = epi
    d.out = out.data_ptr()
    d.ldo = ldo if ldo is not None else N
    d.out2 = out2.data_ptr() if out2 is not None else None
    d.ldo2 = ldo2 if ldo2 is not None else N
    d.aux = aux.data_ptr() if aux is not None else None
    d.ldaux = ldaux if ldaux is not None else N
    d.bias = bias.data_ptr() if bias is not None else None
    d.sign = sign
    d.splits = splits
    d.workspace = workspace.data_ptr() if workspace is not None else None
    d.rowdot = rowdot.data_ptr() if rowdot is not None else None
    d.rd_seq = rd_seq
    d.max_ctas = max_ctas
    d.bn = bn
    d.colsum_part = colsum_part.data_ptr() if colsum_part is not None else None
    check(lib().rp_gemm(C.byref(d), _stream(stream)), "gemm")
    return out


def colsum_parts(part, out=None, accumulate=False, stream=None):
    """Second stage of a column sum: out[c] (+)= sum_p part[p][c] (fixed order)."""
    nparts, cols = part.shape
    if out is None:
        out = torch.zeros(cols, dtype=torch.float32, device=part.device)
    check(lib().rp_colsum_parts(_p(part), nparts, cols, _p(out), int(accumulate),
                                _stream(stream)), "colsum_parts")
    return out


def layer_norm_fwd(x, gamma, beta, eps=1e-5, y=None, mean=None, rstd=None, stream=None):
    """ref:proj/core/src/ops.cpp:264-304 -> (y bf16, mean, rstd)."""
    _req(x, torch.float32, "layer_norm x")
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    if y is None:
        y = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    if mean is None:
        mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    if rstd is None:
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    check(lib().rp_layer_norm_fwd(_p(x), _p(gamma), _p(beta), rows, cols, eps, _p(y), _p(mean),
                                  _p(rstd), _stream(stream)), "layer_norm")
    return y, mean, rstd


def layer_norm_bwd(x, mean, rstd, gamma, dy, dres=None, dx=None, dx_bf16=None, dgamma=None,
                   dbeta=None, dx_colsum=None, accumulate=False, stream=None):
    """ref:proj/core/src/ops.cpp:306-345 (+ fused residual cotangent add; optional column sum
    of the produced dx, the next block's MLP output-bias gradient)."""
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    dev = x.device
    if dx is None:
        dx = torch.empty(x.shape, dtype=torch.float32, device=dev)
    if dgamma is None:
        dgamma = torch.zeros(cols, dtype=torch.float32, device=dev)
    if dbeta is None:
        dbeta = torch.zeros(cols, dtype=torch.float32, device=dev)
    ws = torch.empty(lib().rp_layer_norm_bwd_workspace_floats(rows, cols), dtype=torch.float32,
                     device=dev)
    check(lib().rp_layer_norm_bwd_ex(_p(x), _p(mean), _p(rstd), _p(gamma), _p(dy), _p(dres), rows,
                                     cols, _p(dx), _p(dx_bf16), _p(dgamma), _p(dbeta),
                                     _p(dx_colsum), _p(ws), int(accumulate), _stream(stream)),
          "layer_norm_vjp")
    return dx, dgamma, dbeta


def colsum(x, out=None, accumulate=False, stream=None):
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    if out is None:
        out = torch.zeros(cols, dtype=torch.float32, device=x.device)
    ws = torch.empty(lib().rp_colsum_workspace_floats(rows, cols), dtype=torch.float32,
                     device=x.device)
    check(lib().rp_colsum(_p(x), int(x.dtype == torch.bfloat16), rows, cols, _p(out), _p(ws),
                          int(accumulate), _stream(stream)), "col_sum")
    return out


def attention_fwd(qkv, B, N, H, head_dim=64, out=None, lse=None, stream=None):
    """qkv [B*N, 3*H*hd] bf16 -> (out [B*N, H*hd] bf16, lse [B,H,N] fp32 log2-domain)."""
    _req(qkv, torch.bfloat16, "attention qkv")
    if out is None:
        out = torch.empty(B * N, H * head_dim, dtype=torch.bfloat16, device=qkv.device)
    if lse is None:
        lse = torch.empty(B, H, N, dtype=torch.float32, device=qkv.device)
    check(lib().rp_attention_fwd(_p(qkv), B, N, H, head_dim, _p(out), _p(lse), _stream(stream)),
          "attention_forward")
    return out, lse


def attention_bwd(qkv, out, lse, dout, B, N, H, head_dim=64, dqkv=None, stream=None):
    if dqkv is None:
        dqkv = torch.empty_like(qkv)
    ws = torch.empty(lib().rp_attention_bwd_workspace_floats(B, N, H), dtype=torch.float32,
                     device=qkv.device)
    check(lib().rp_attention_bwd(_p(qkv), _p(out), _p(lse), _p(dout), B, N, H, head_dim,
                                 _p(dqkv), _p(ws), _stream(stream)), "attention_vjp")
    return dqkv
