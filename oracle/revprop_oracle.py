"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference algorithm (the oracle).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.
The product path never does: it runs the sm_100a library and fails if that is missing.

Pinned against the reference itself: tests/test_oracle.py checks every function here
against the reference's own code compiled in place (oracle/_ref/librevprop_ref.so, built
by oracle/Makefile from /root/reference/proj/core/src/{ops,layers}.cpp) and against the
golden fixtures in tests/golden/ generated from it (tests/golden/make_golden.py), plus
the SPEC's known-answer examples.

Every function cites the reference file:line it restates. Arithmetic is numpy (f64 by
default); the reference accumulates left-to-right, numpy's BLAS does not, so f64 results
agree to ~1e-13 relative, not bit-for-bit.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

LN_EPS = 1e-5  # ref:proj/core/include/revprop/layers.hpp:18
GELU_C = 0.7978845608028654  # ref:proj/core/src/ops.cpp:11
GELU_A = 0.044715  # ref:proj/core/src/ops.cpp:12

# ------------------------------------------------------------------ counter RNG
# ref:proj/core/include/revprop/rng.hpp:13-71, vectorised over (stream, counter).
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix(z):
    """rng.hpp:59-66 murmur finalizer."""
    z = z ^ (z >> np.uint64(33))
    z = z * np.uint64(0xFF51AFD7ED558CCD)
    z = z ^ (z >> np.uint64(33))
    z = z * np.uint64(0xC4CEB9FE1A85EC53)
    z = z ^ (z >> np.uint64(33))
    return z


def rng_u64(seed, stream, counter):
    """Rng(seed, stream).next_u64() at `counter` (rng.hpp:27-33)."""
    with np.errstate(over="ignore"):
        seed = np.asarray(seed, dtype=np.uint64)
        stream = np.asarray(stream, dtype=np.uint64)
        counter = np.asarray(counter, dtype=np.uint64)
        h = _mix(seed ^ np.uint64(0x9E3779B97F4A7C15))
        h = _mix(h ^ (stream * np.uint64(0xBF58476D1CE4E5B9) + np.uint64(0x94D049BB133111EB)))
        h = _mix(h ^ (counter * np.uint64(0x2545F4914F6CDD1D) + np.uint64(0xD6E8FEB86659FD93)))
    return h


def rng_normal(seed, stream, counter):
    """next_normal at counters (c, c+1): Box-Muller, no caching (rng.hpp:38-42)."""
    u1 = ((rng_u64(seed, stream, counter) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (rng_u64(seed, stream, counter + np.uint64(1)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * 3.14159265358979323846 * u2)


def trunc_normal_streams(seed, streams, sigma):
    """Per-stream next_trunc_normal(sigma): reject outside +-2 (rng.hpp:45-50)."""
    streams = np.asarray(streams, dtype=np.uint64)
    out = np.empty(streams.shape, dtype=np.float64)
    todo = np.arange(streams.size)
    c = np.zeros(streams.size, dtype=np.uint64)
    flat = streams.reshape(-1)
    res = out.reshape(-1)
    while todo.size:
        z = rng_normal(seed, flat[todo], c[todo])
        ok = (z >= -2.0) & (z <= 2.0)
        res[todo[ok]] = z[ok] * sigma
        todo = todo[~ok]
        c[todo] += np.uint64(2)
    return out


# ------------------------------------------------------------------ tensor-core ops
def layer_norm(x, gamma, beta, eps=LN_EPS):
    """ops.cpp:264-304: two-pass mean / population variance; returns (y, (x_hat, inv_std))."""
    mean = x.mean(-1, keepdims=True)
    var = ((x - mean) ** 2).mean(-1, keepdims=True)
    inv_std = 1.0 / np.sqrt(var + eps)
    xh = (x - mean) * inv_std
    return xh * gamma + beta, (xh, inv_std[..., 0])


def layer_norm_vjp(cache, gamma, dy):
    """ops.cpp:306-345."""
    xh, inv_std = cache
    g = dy * gamma
    gm = g.mean(-1, keepdims=True)
    ghm = (g * xh).mean(-1, keepdims=True)
    dx = (g - gm - xh * ghm) * inv_std[..., None]
    lead = tuple(range(dy.ndim - 1))
    return dx, (dy * xh).sum(lead), dy.sum(lead)


def gelu(x):
    """ops.cpp:227-241 tanh-GELU."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + GELU_A * x ** 3)))


def gelu_vjp(x, dy):
    """ops.cpp:243-262."""
    t = np.tanh(GELU_C * (x + GELU_A * x ** 3))
    slope = 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * GELU_C * (1 + 3 * GELU_A * x * x)
    return slope * dy


def row_softmax(x):
    """ops.cpp:182-204."""
    e = np.exp(x - x.max(-1, keepdims=True))
    return e * (1.0 / e.sum(-1, keepdims=True))


def row_softmax_vjp(y, dy):
    """ops.cpp:206-225: y * (dy - <y, dy>)."""
    return y * (dy - (y * dy).sum(-1, keepdims=True))


# ------------------------------------------------------------------ layers (F, G)
@dataclass
class AttentionParams:  # layers.hpp:43-52
    w_qkv: np.ndarray
    w_out: np.ndarray
    ln_gamma: np.ndarray
    ln_beta: np.ndarray
    heads: int = 1
    window: int | None = None


@dataclass
class MlpParams:  # layers.hpp:94-103
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    ln_gamma: np.ndarray
    ln_beta: np.ndarray


def _heads(t, B, N, H, hd, W):
    # [B, N, H*hd] -> [B, H, nW, W, hd]  (gather_block, layers.cpp:54-70)
    return t.reshape(B, N // W, W, H, hd).transpose(0, 3, 1, 2, 4)


def _unheads(t, B, N, H, hd, W):
    # inverse of _heads (scatter_block, layers.cpp:72-84)
    return t.transpose(0, 2, 3, 1, 4).reshape(B, N, H * hd)


def attention_forward(x, p: AttentionParams):
    """layers.cpp:134-169: y = (softmax(q k^T * 1/sqrt(hd)) v) W_out, per (b, head, window)."""
    B, N, d = x.shape
    H = p.heads
    hd = d // H
    W = p.window or N
    assert N % W == 0 and d % H == 0
    h, ln_cache = layer_norm(x, p.ln_gamma, p.ln_beta)
    qkv = h @ p.w_qkv
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    qh, kh, vh = (_heads(t, B, N, H, hd, W) for t in (q, k, v))
    scores = (qh @ kh.swapaxes(-1, -2)) * (1.0 / np.sqrt(hd))  # scale after QK^T (:159)
    probs = row_softmax(scores)
    att = _unheads(probs @ vh, B, N, H, hd, W)
    y = att @ p.w_out
    return y, dict(ln=ln_cache, h=h, q=qh, k=kh, v=vh, probs=probs, att=att)


def attention_vjp(c, p: AttentionParams, dy):
    """layers.cpp:171-220."""
    B, N, d = dy.shape
    H = p.heads
    hd = d // H
    W = p.window or N
    d_att = dy @ p.w_out.T
    d_w_out = c["att"].reshape(-1, d).T @ dy.reshape(-1, d)
    doh = _heads(d_att, B, N, H, hd, W)
    da = doh @ c["v"].swapaxes(-1, -2)
    dvh = c["probs"].swapaxes(-1, -2) @ doh
    ds = row_softmax_vjp(c["probs"], da) * (1.0 / np.sqrt(hd))
    dqh = ds @ c["k"]
    dkh = ds.swapaxes(-1, -2) @ c["q"]
    d_qkv = np.concatenate([_unheads(t, B, N, H, hd, W) for t in (dqh, dkh, dvh)], -1)
    d_h = d_qkv @ p.w_qkv.T
    d_w_qkv = c["h"].reshape(-1, d).T @ d_qkv.reshape(-1, 3 * d)
    dx, dg, db = layer_norm_vjp(c["ln"], p.ln_gamma, d_h)
    return dx, dict(d_w_qkv=d_w_qkv, d_w_out=d_w_out, d_ln_gamma=dg, d_ln_beta=db)


def mlp_forward(x, p: MlpParams):
    """layers.cpp:222-239: y = gelu(LN(x) W1 + b1) W2 + b2."""
    h, ln_cache = layer_norm(x, p.ln_gamma, p.ln_beta)
    u = h @ p.w1 + p.b1
    a = gelu(u)
    y = a @ p.w2 + p.b2
    return y, dict(ln=ln_cache, h=h, u=u, a=a)


def mlp_vjp(c, p: MlpParams, dy):
    """layers.cpp:241-259."""
    d, hdim = p.w1.shape
    d_a = dy @ p.w2.T
    d_w2 = c["a"].reshape(-1, hdim).T @ dy.reshape(-1, d)
    d_b2 = dy.reshape(-1, d).sum(0)
    d_u = gelu_vjp(c["u"], d_a)
    d_h = d_u @ p.w1.T
    d_w1 = c["h"].reshape(-1, d).T @ d_u.reshape(-1, hdim)
    d_b1 = d_u.reshape(-1, hdim).sum(0)
    dx, dg, db = layer_norm_vjp(c["ln"], p.ln_gamma, d_h)
    return dx, dict(d_w1=d_w1, d_b1=d_b1, d_w2=d_w2, d_b2=d_b2, d_ln_gamma=dg, d_ln_beta=db)


# ------------------------------------------------------------------ revcore
@dataclass
class RevBlock:
    f: AttentionParams
    g: MlpParams


def rev_forward(b: RevBlock, i1, i2):
    """o2 = i2 + F(i1); o1 = i1 + G(o2)."""
    o2 = i2 + attention_forward(i1, b.f)[0]
    o1 = i1 + mlp_forward(o2, b.g)[0]
    return o1, o2


def rev_inverse(b: RevBlock, o1, o2):
    """i1 = o1 - G(o2); i2 = o2 - F(i1)."""
    i1 = o1 - mlp_forward(o2, b.g)[0]
    i2 = o2 - attention_forward(i1, b.f)[0]
    return i1, i2


def recompute(b: RevBlock, o1, o2):
    """Lane-R half of rev_backward_local: inverse retaining the F/G caches."""
    gy, cg = mlp_forward(o2, b.g)
    i1 = o1 - gy
    fy, cf = attention_forward(i1, b.f)
    i2 = o2 - fy
    return (i1, i2), cf, cg


def recompute_from_input(b: RevBlock, i1, i2):
    """First block of a stage: caches from the stored stage input."""
    fy, cf = attention_forward(i1, b.f)
    o2 = i2 + fy
    _, cg = mlp_forward(o2, b.g)
    return (i1, i2), cf, cg


def vjp_half(b: RevBlock, cf, cg, d_o1, d_o2):
    """d_o2t = d_o2 + VJP_G(d_o1); d_i1 = d_o1 + VJP_F(d_o2t); d_i2 = d_o2t."""
    gx, gg = mlp_vjp(cg, b.g, d_o1)
    d_o2t = d_o2 + gx
    fx, fg = attention_vjp(cf, b.f, d_o2t)
    return (d_o1 + fx, d_o2t), (fg, gg)


# ------------------------------------------------------------------ stage boundary
# ref:proj/core/src/layers.cpp:261-303, ops.cpp:393-406 (group_tokens / ungroup_tokens)
def fuse(i1, i2, fusion_w=None):
    """layers.cpp:276-287: average -> (i1 + i2) * 0.5 (ops::scale(ops::add)); mlp ->
    concat(i1, i2) . fusion_w. Returns (y, concat or None)."""
    if fusion_w is None:
        return (i1 + i2) * 0.5, None
    concat = np.concatenate([i1, i2], -1)
    return concat @ fusion_w, concat


def fuse_vjp(concat, fusion_w, d_y):
    """layers.cpp:289-303: (d_i1, d_i2, d_fusion_w or None)."""
    if fusion_w is None:
        half = d_y * 0.5
        return half, half, None
    d = d_y.shape[-1]
    d_concat = d_y @ fusion_w.T
    d_fw = concat.reshape(-1, 2 * d).T @ d_y.reshape(-1, d)
    return d_concat[..., :d], d_concat[..., d:], d_fw


def patch_merge(x, merge_w, r):
    """layers.cpp:261-267: group r adjacent tokens ([B, N, d] -> [B, N/r, r*d], a reshape of
    row-major data, ops.cpp:393-399) and project by merge_w [(r*d), d_next]."""
    B, N, d = x.shape
    assert N % r == 0, "group_tokens: token count not divisible by r"
    grouped = x.reshape(B, N // r, r * d)
    return grouped @ merge_w, grouped


def patch_merge_vjp(grouped, merge_w, r, d_y):
    """layers.cpp:269-274: (d_x [B, N, d], d_merge_w)."""
    B, G, rd = grouped.shape
    d_grouped = d_y @ merge_w.T
    d_merge_w = grouped.reshape(-1, rd).T @ d_y.reshape(-1, d_y.shape[-1])
    return d_grouped.reshape(B, G * r, rd // r), d_merge_w


def rev_backward_local(b: RevBlock, o1, o2, d_o1, d_o2):
    """SPEC.md:231-239."""
    inp, cf, cg = recompute(b, o1, o2)
    d_inp, grads = vjp_half(b, cf, cg, d_o1, d_o2)
    return inp, d_inp, grads


# ------------------------------------------------------------------ models
@dataclass
class ModelConfig:  # SPEC.md:275-278 (isotropic)
    depth: int
    width: int
    heads: int
    hidden: int
    seq_len: int
    in_dim: int
    num_classes: int
    window: int | None = None
    # hierarchical (Rev-Swin): blocks / width / heads per stage; the MLP
    # ratio hidden/width is kept in every stage; stage s has seq_len / r^s tokens and
    # attends in windows of min(window, tokens) (full attention when window is None).
    depths: tuple | None = None
    widths: tuple | None = None
    stage_heads: tuple | None = None
    reduction: int = 2
    fusion: str = "average"  # BoundaryParams.fusion_kind (layers.hpp:142-149)


@dataclass
class StageGeom:
    depth: int
    d: int
    heads: int
    hidden: int
    tokens: int
    window: int | None
    first: int  # global index of the stage's first block


def stages(cfg: ModelConfig):
    """Per-stage geometry; an isotropic model is one stage."""
    if not cfg.depths:
        return [StageGeom(cfg.depth, cfg.width, cfg.heads, cfg.hidden, cfg.seq_len, cfg.window, 0)]
    assert len(cfg.depths) >= 2 and cfg.hidden % cfg.width == 0
    ratio = cfg.hidden // cfg.width
    out, first, n = [], 0, cfg.seq_len
    for s, L in enumerate(cfg.depths):
        if s:
            assert n % cfg.reduction == 0, "seq_len not divisible by r^(stages-1)"
            n //= cfg.reduction
        d = cfg.widths[s]
        w = None if cfg.window is None else min(cfg.window, n)
        out.append(StageGeom(L, d, cfg.stage_heads[s], ratio * d, n, w, first))
        first += L
    return out


BLOCK_TENSORS = ("w_qkv", "w_out", "lnF_g", "lnF_b", "w1", "b1", "w2", "b2", "lnG_g", "lnG_b")


def tensor_shapes(cfg: ModelConfig):
    """Flat parameter order shared with the GPU engine (include/revprop_b200.h)."""
    st = stages(cfg)
    shapes = [("embed_w", (cfg.in_dim, st[0].d))]
    for s, g in enumerate(st):
        d, h = g.d, g.hidden
        per = dict(w_qkv=(d, 3 * d), w_out=(d, d), lnF_g=(d,), lnF_b=(d,), w1=(d, h), b1=(h,),
                   w2=(h, d), b2=(d,), lnG_g=(d,), lnG_b=(d,))
        for b in range(g.first, g.first + g.depth):
            shapes += [(f"blocks.{b}.{n}", per[n]) for n in BLOCK_TENSORS]
        if s + 1 < len(st):  # BoundaryParams (layers.hpp:144-149): merge_w, fusion_w
            shapes.append((f"boundary.{s}.merge_w", (cfg.reduction * d, st[s + 1].d)))
            if cfg.fusion == "mlp":
                shapes.append((f"boundary.{s}.fusion_w", (2 * d, d)))
    shapes.append(("head_w", (st[-1].d, cfg.num_classes)))
    return shapes


def param_count(cfg):
    return sum(int(np.prod(s)) for _, s in tensor_shapes(cfg))


def init_params(cfg: ModelConfig, seed: int, dtype=np.float64):
    """build_model: weights trunc-normal(sigma 0.02) at +-2 sigma, biases 0,
    LayerNorm gamma 1 / beta 0. Element e of flat tensor j draws from the counter RNG
    stream (1<<56)|(j<<32)|e (same definition as the GPU engine's init kernel)."""
    out = []
    for j, (name, shape) in enumerate(tensor_shapes(cfg)):
        n = int(np.prod(shape))
        base = name.split(".")[-1]
        if base in ("b1", "b2", "lnF_b", "lnG_b"):
            v = np.zeros(n)
        elif base in ("lnF_g", "lnG_g"):
            v = np.ones(n)
        else:
            streams = (np.uint64(1) << np.uint64(56)) | (np.uint64(j) << np.uint64(32)) | np.arange(
                n, dtype=np.uint64)
            v = trunc_normal_streams(np.uint64(seed), streams, 0.02)
        out.append(v)
    return np.concatenate(out).astype(dtype)


def synthetic_batch(cfg: ModelConfig, batch: int, seed: int):
    """Inputs N(0,1) from streams (2<<56)|e (counter 0); labels Rng(seed, 3<<56).next_int(0, C)
    in batch order (rng.hpp:38-42, 53-57)."""
    n = batch * cfg.seq_len * cfg.in_dim
    streams = (np.uint64(2) << np.uint64(56)) | np.arange(n, dtype=np.uint64)
    x = rng_normal(np.uint64(seed), streams, np.uint64(0)).reshape(batch, cfg.seq_len, cfg.in_dim)
    lab = rng_u64(np.uint64(seed), np.uint64(3) << np.uint64(56), np.arange(batch, dtype=np.uint64))
    labels = (lab % np.uint64(cfg.num_classes)).astype(np.int64)
    return x, labels


def unflatten(cfg: ModelConfig, flat):
    out, off = {}, 0
    for name, shape in tensor_shapes(cfg):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    return out


def blocks_of(cfg: ModelConfig, flat):
    t = unflatten(cfg, flat)
    blocks = []
    for st in stages(cfg):
        for b in range(st.first, st.first + st.depth):
            g = lambda n: t[f"blocks.{b}.{n}"]
            blocks.append(RevBlock(
                AttentionParams(g("w_qkv"), g("w_out"), g("lnF_g"), g("lnF_b"), st.heads,
                                st.window),
                MlpParams(g("w1"), g("b1"), g("w2"), g("b2"), g("lnG_g"), g("lnG_b"))))
    return t["embed_w"], blocks, t["head_w"]


def boundaries_of(cfg: ModelConfig, flat):
    """[(merge_w, fusion_w or None)] for the boundaries after stages 0..S-2."""
    t = unflatten(cfg, flat)
    return [(t[f"boundary.{s}.merge_w"], t.get(f"boundary.{s}.fusion_w"))
            for s in range(len(stages(cfg)) - 1)]


def loss_and_grad_head(logits, labels):
    """mean CE (log-sum-exp); d_logits = (softmax - onehot) / B."""
    B = logits.shape[0]
    mx = logits.max(-1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(-1))
    loss = float(np.mean(lse - logits[np.arange(B), labels]))
    p = np.exp(logits - lse[:, None])
    p[np.arange(B), labels] -= 1.0
    return loss, p / B


# ------------------------------------------------------------------ engines
@dataclass
class StepResult:
    loss: float
    grads: np.ndarray
    slots: list = field(default_factory=list)  # (lane, block 1-based) in issue order
    recomputed: list = field(default_factory=list)  # recomputed X_b (i1, i2), b = L-1..0


def _backward_stage(blocks, first, stage_in, o, d_out, engine, bgrads, slots, recomputed,
                    keep_recomputed):
    """One stage's backward: blocks last -> first, lane R recomputing the
    block input + caches from its output, lane G running the VJP. pareprop runs lane R on a
    second thread with a capacity-1 rendezvous; the arithmetic is
    identical, so the grads are identical. Returns the stage input's cotangent pair."""
    L = len(blocks)

    def do_r(i, out):
        if i == 0:
            return recompute_from_input(blocks[0], *stage_in)
        return recompute(blocks[i], *out)

    if engine == "reprop":
        out = o
        for i in range(L - 1, -1, -1):
            inp, cf, cg = do_r(i, out)
            slots.append(("R", first + i + 1))
            if keep_recomputed:
                recomputed.append(inp)
            d_out, bgrads[first + i] = vjp_half(blocks[i], cf, cg, *d_out)
            slots.append(("G", first + i + 1))
            out = inp
    elif engine == "pareprop":
        cv = threading.Condition()
        box = []
        err = []

        def lane_r():
            try:
                out = o
                for i in range(L - 1, -1, -1):
                    with cv:
                        cv.wait_for(lambda: not box or err)
                    item = do_r(i, out)
                    with cv:
                        slots.append(("R", first + i + 1))
                        box.append((i, item))
                        cv.notify_all()
                    out = item[0]
            except Exception as ex:  # pragma: no cover
                with cv:
                    err.append(ex)
                    cv.notify_all()

        t = threading.Thread(target=lane_r)
        t.start()
        for i in range(L - 1, -1, -1):
            with cv:
                cv.wait_for(lambda: box or err)
                if err:
                    break
                j, (inp, cf, cg) = box.pop()
                cv.notify_all()
            assert j == i
            if keep_recomputed:
                recomputed.append(inp)
            d_out, bgrads[first + i] = vjp_half(blocks[i], cf, cg, *d_out)
            with cv:
                slots.append(("G", first + i + 1))
        t.join()
        if err:
            raise RuntimeError(f"pipeline lane failed: {err[0]}")
    else:
        raise ValueError(engine)
    return d_out


def step(cfg: ModelConfig, flat, x, labels, engine="reprop", keep_recomputed=False):
    """step_reprop / step_pareprop over the isotropic or
    hierarchical model (forward_full: embed, duplicate, each stage's blocks,
    at each boundary fuse -> patch_merge -> duplicate; head on fuse-average of the last
    stage's output). Only each stage's input and output pairs are kept;
    the backward recomputes the boundary's fuse from the stored stage output."""
    embed_w, blocks, head_w = blocks_of(cfg, flat)
    bnds = boundaries_of(cfg, flat)
    st = stages(cfg)
    e = x @ embed_w
    stage_in, stage_out = [], []
    o = (e, e)  # duplication
    for s, g in enumerate(st):
        stage_in.append(o)
        for b in blocks[g.first:g.first + g.depth]:
            o = rev_forward(b, *o)
        stage_out.append(o)
        if s + 1 < len(st):
            f, _ = fuse(*o, bnds[s][1])
            y, _ = patch_merge(f, bnds[s][0], cfg.reduction)
            o = (y, y)
    fused = (o[0] + o[1]) * 0.5  # fuse average (layers.cpp:276-280)
    pooled = fused.mean(1)  # mean_tokens (ops.cpp:408-427)
    logits = pooled @ head_w
    loss, d_logits = loss_and_grad_head(logits, labels)
    grads = {"head_w": pooled.T @ d_logits}
    d_pooled = d_logits @ head_w.T
    n_last = st[-1].tokens
    d_fused = np.repeat(d_pooled[:, None, :] * (1.0 / n_last), n_last, 1)  # spread_tokens
    d_out = (d_fused * 0.5, d_fused * 0.5)  # fuse_vjp average (layers.cpp:289-293)
    bgrads = [None] * len(blocks)
    slots, recomputed = [], []
    for s in range(len(st) - 1, -1, -1):
        g = st[s]
        d_out = _backward_stage(blocks[g.first:g.first + g.depth], g.first, stage_in[s],
                                stage_out[s], d_out, engine, bgrads, slots, recomputed,
                                keep_recomputed)
        if s > 0:
            mw, fw = bnds[s - 1]
            d_y = d_out[0] + d_out[1]  # both halves of the next stage's input are y
            f, concat = fuse(*stage_out[s - 1], fw)
            grouped = f.reshape(f.shape[0], -1, cfg.reduction * f.shape[-1])
            d_f, grads[f"boundary.{s - 1}.merge_w"] = patch_merge_vjp(grouped, mw,
                                                                       cfg.reduction, d_y)
            d1, d2, d_fw = fuse_vjp(concat, fw, d_f)
            if d_fw is not None:
                grads[f"boundary.{s - 1}.fusion_w"] = d_fw
            d_out = (d1, d2)
    d_e = d_out[0] + d_out[1]
    grads["embed_w"] = x.reshape(-1, x.shape[-1]).T @ d_e.reshape(-1, d_e.shape[-1])
    names = {"d_w_qkv": "w_qkv", "d_w_out": "w_out", "d_ln_gamma": "lnF_g", "d_ln_beta": "lnF_b"}
    gnames = {"d_w1": "w1", "d_b1": "b1", "d_w2": "w2", "d_b2": "b2", "d_ln_gamma": "lnG_g",
              "d_ln_beta": "lnG_b"}
    for b, (fg, gg) in enumerate(bgrads):
        for k, v in fg.items():
            grads[f"blocks.{b}.{names[k]}"] = v
        for k, v in gg.items():
            grads[f"blocks.{b}.{gnames[k]}"] = v
    flat_g = np.concatenate([np.asarray(grads[n]).reshape(-1) for n, _ in tensor_shapes(cfg)])
    return StepResult(loss, flat_g, slots, recomputed)


def sgd_update(flat, grads, lr):
    """theta <- theta - lr * g."""
    return flat - lr * grads


def makespan(L, t_r, t_g, pipelined):
    """Discrete-event makespan of the backward: Reprop runs R,G per block in
    sequence; PaReprop's slots are [R_L], [G_L || R_{L-1}], ..., [G_1]."""
    if not pipelined:
        return L * (t_r + t_g)
    return t_r + (L - 1) * max(t_r, t_g) + t_g
