"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/librevprop_ref.so, i.e. the
reference's own ops.cpp / layers.cpp compiled in place plus the SPEC restatement in
oracle/ref_shim.cpp. Used to pin oracle/revprop_oracle.py, to generate tests/golden/, and as
bench.py's CPU baseline (`--impl reference`, `cpu_baseline.kind = "reference"`).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "librevprop_ref.so"
REFERENCE = Path("/root/reference/proj/core")


class RefCfg(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("depth", "width", "heads", "hidden", "seq_len", "in_dim",
                                         "num_classes", "window")]


class RefHierCfg(C.Structure):
    _fields_ = [("stages", C.c_int64), ("depths", C.c_int64 * 8), ("widths", C.c_int64 * 8),
                ("heads", C.c_int64 * 8)] + [(n, C.c_int64) for n in (
                    "ratio", "seq_len", "in_dim", "num_classes", "window", "reduction", "fusion")]


_lib = None


def build(force: bool = False) -> bool:
    """Compile oracle/_ref from /root/reference (only possible where the reference exists)."""
    if LIB.exists() and not force:
        return True
    if not REFERENCE.exists():
        return False
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB.exists()


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise FileNotFoundError(f"{LIB} not built (make -C oracle)")
        L = C.CDLL(str(LIB))
        P, I64, I = C.c_void_p, C.c_int64, C.c_int
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_param_count": (I64, [C.POINTER(RefCfg)]),
            "ref_block_param_count": (I64, [C.POINTER(RefCfg)]),
            "ref_rng": (I, [C.c_uint64, C.c_uint64, I64, P, P, P]),
            "ref_layer_norm": (I, [I, P, I64, I64, P, P, C.c_double, P, P, P, P, P, P]),
            "ref_attention": (I, [I, C.POINTER(RefCfg), I64, P, P, P, P, P, P]),
            "ref_mlp": (I, [I, C.POINTER(RefCfg), I64, P, P, P, P, P, P]),
            "ref_rev_forward": (I, [I, C.POINTER(RefCfg), I64, P, P, P, P, P]),
            "ref_rev_inverse": (I, [I, C.POINTER(RefCfg), I64, P, P, P, P, P]),
            "ref_rev_backward_local": (I, [I, C.POINTER(RefCfg), I64, P, P, P, P, P, P, P, P, P,
                                           P]),
            "ref_step": (I, [I, C.POINTER(RefCfg), I, I64, P, P, P, P, P, P, P]),
            "ref_step_dp": (I, [I, C.POINTER(RefCfg), I, I64, I, P, P, P, P, P]),
            "ref_hier_param_count": (I64, [C.POINTER(RefHierCfg)]),
            "ref_hier_step": (I, [I, C.POINTER(RefHierCfg), I64, P, P, P, P, P]),
            "ref_boundary": (I, [I, I64, I64, I64, I64, I64, I] + [P] * 10),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def cfg_of(mc) -> RefCfg:
    return RefCfg(mc.depth, mc.width, mc.heads, mc.hidden, mc.seq_len, mc.in_dim,
                  mc.num_classes, mc.window or 0)


def _dt(f64):
    return np.float64 if f64 else np.float32


def rng(seed, stream, n):
    u = np.empty(n, np.uint64)
    z = np.empty(n, np.float64)
    t = np.empty(n, np.float64)
    _chk(lib().ref_rng(seed, stream, n, _p(u), _p(z), _p(t)))
    return u, z, t


def layer_norm(x, g, b, eps=1e-5, dy=None):
    f64 = x.dtype == np.float64
    R, Cc = x.reshape(-1, x.shape[-1]).shape
    y = np.empty_like(x)
    inv = np.empty(R, x.dtype)
    dx = np.empty_like(x) if dy is not None else None
    dg = np.empty(Cc, x.dtype) if dy is not None else None
    db = np.empty(Cc, x.dtype) if dy is not None else None
    _chk(lib().ref_layer_norm(int(f64), _p(x), R, Cc, _p(g), _p(b), eps, _p(dy), _p(y), _p(inv),
                              _p(dx), _p(dg), _p(db)))
    return y, inv, dx, dg, db


def attention(mc, pf, x, dy=None):
    f64 = x.dtype == np.float64
    B = x.shape[0]
    y = np.empty_like(x)
    dx = np.empty_like(x) if dy is not None else None
    dp = np.empty_like(pf) if dy is not None else None
    c = cfg_of(mc)
    _chk(lib().ref_attention(int(f64), C.byref(c), B, _p(pf), _p(x), _p(dy), _p(y), _p(dx),
                             _p(dp)))
    return y, dx, dp


def mlp(mc, pg, x, dy=None):
    f64 = x.dtype == np.float64
    B = x.shape[0]
    y = np.empty_like(x)
    dx = np.empty_like(x) if dy is not None else None
    dp = np.empty_like(pg) if dy is not None else None
    c = cfg_of(mc)
    _chk(lib().ref_mlp(int(f64), C.byref(c), B, _p(pg), _p(x), _p(dy), _p(y), _p(dx), _p(dp)))
    return y, dx, dp


def rev_forward(mc, pb, i1, i2):
    c = cfg_of(mc)
    o1, o2 = np.empty_like(i1), np.empty_like(i2)
    _chk(lib().ref_rev_forward(int(i1.dtype == np.float64), C.byref(c), i1.shape[0], _p(pb),
                               _p(i1), _p(i2), _p(o1), _p(o2)))
    return o1, o2


def rev_inverse(mc, pb, o1, o2):
    c = cfg_of(mc)
    i1, i2 = np.empty_like(o1), np.empty_like(o2)
    _chk(lib().ref_rev_inverse(int(o1.dtype == np.float64), C.byref(c), o1.shape[0], _p(pb),
                               _p(o1), _p(o2), _p(i1), _p(i2)))
    return i1, i2


def rev_backward_local(mc, pb, o1, o2, d_o1, d_o2):
    c = cfg_of(mc)
    outs = [np.empty_like(o1) for _ in range(4)]
    dpb = np.empty_like(pb)
    _chk(lib().ref_rev_backward_local(int(o1.dtype == np.float64), C.byref(c), o1.shape[0],
                                      _p(pb), _p(o1), _p(o2), _p(d_o1), _p(d_o2),
                                      *[_p(o) for o in outs], _p(dpb)))
    return (outs[0], outs[1]), (outs[2], outs[3]), dpb


def step(mc, params, x, labels, engine="reprop", slots=False):
    """ref_step: returns (loss, grads, peak_bytes, slot_log or None)."""
    c = cfg_of(mc)
    f64 = params.dtype == np.float64
    loss = C.c_double()
    grads = np.empty_like(params)
    peak = C.c_int64()
    sl = np.zeros((2 * mc.depth, 4), np.int64) if slots else None
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    _chk(lib().ref_step(int(f64), C.byref(c), 1 if engine == "reprop" else 2, x.shape[0],
                        _p(params), _p(np.ascontiguousarray(x)), _p(lab), C.byref(loss), _p(grads),
                        C.byref(peak), _p(sl)))
    return loss.value, grads, peak.value, sl


def step_dp(mc, params, x, labels, threads, engine="reprop"):
    c = cfg_of(mc)
    f64 = params.dtype == np.float64
    loss = C.c_double()
    grads = np.empty_like(params)
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    _chk(lib().ref_step_dp(int(f64), C.byref(c), 1 if engine == "reprop" else 2, x.shape[0],
                           threads, _p(params), _p(np.ascontiguousarray(x)), _p(lab),
                           C.byref(loss), _p(grads)))
    return loss.value, grads


def block_slice(mc, flat, b):
    d, h, i = mc.width, mc.hidden, mc.in_dim
    bs = 4 * d * d + 2 * d * h + h + 5 * d
    off = i * d + b * bs
    return flat[off:off + bs]


def split_block(mc, pb):
    """block params -> (F params [w_qkv|w_out|g|b], G params [w1|b1|w2|b2|g|b])."""
    d = mc.width
    nf = 3 * d * d + d * d + 2 * d
    return pb[:nf], pb[nf:]


def hier_cfg_of(mc) -> RefHierCfg:
    S = len(mc.depths)
    c = RefHierCfg()
    c.stages = S
    for s in range(S):
        c.depths[s], c.widths[s], c.heads[s] = mc.depths[s], mc.widths[s], mc.stage_heads[s]
    c.ratio = mc.hidden // mc.width
    c.seq_len, c.in_dim, c.num_classes = mc.seq_len, mc.in_dim, mc.num_classes
    c.window, c.reduction = mc.window or 0, mc.reduction
    c.fusion = 1 if mc.fusion == "mlp" else 0
    return c


def hier_param_count(mc) -> int:
    return int(lib().ref_hier_param_count(C.byref(hier_cfg_of(mc))))


def hier_step(mc, params, x, labels):
    """ref_hier_step (Reprop order): (loss, flat grads)."""
    c = hier_cfg_of(mc)
    f64 = params.dtype == np.float64
    loss = C.c_double()
    grads = np.empty_like(params)
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    _chk(lib().ref_hier_step(int(f64), C.byref(c), x.shape[0], _p(params),
                             _p(np.ascontiguousarray(x)), _p(lab), C.byref(loss), _p(grads)))
    return loss.value, grads


def boundary(i1, i2, merge_w, fusion_w, r, d_y):
    """The reference's fuse -> patch_merge and its VJP: (y, d_i1, d_i2, d_merge_w, d_fusion_w)."""
    B, N, d = i1.shape
    dn = merge_w.shape[1]
    dt = i1.dtype
    y = np.empty((B, N // r, dn), dt)
    d1, d2 = np.empty_like(i1), np.empty_like(i1)
    dmw = np.empty_like(merge_w)
    dfw = None if fusion_w is None else np.empty_like(fusion_w)
    _chk(lib().ref_boundary(int(dt == np.float64), B, N, d, dn, r, int(fusion_w is not None),
                            _p(i1), _p(i2), _p(merge_w), _p(fusion_w), _p(d_y), _p(y), _p(d1),
                            _p(d2), _p(dmw), _p(dfw)))
    return y, d1, d2, dmw, dfw
