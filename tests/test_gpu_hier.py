"""Hierarchical (Rev-Swin-style) engine on the B200 against the CPU oracle: stages of
RevBlocks joined by fuse + patch_merge boundaries (ref:proj/core/src/
layers.cpp:261-303; the oracle's hierarchical step is pinned to the reference's boundary
layers in tests/test_oracle.py). Same stated tolerances as tests/test_gpu_engine.py: per
tensor max|gpu - ref| / max|ref| <= 5e-2 for parameter gradients, relative L2 <= 2e-2,
loss within 1e-3 relative; PaReprop vs Reprop bit-identical.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import revprop_oracle as O  # noqa: E402

TOL_GRAD = 5e-2
TOL_L2 = 2e-2

# two stages, average fusion, r = 4, head_dim 32 (mma.sync attention), windows 16 / 16
HA = dict(width=64, heads=2, hidden=128, seq_len=64, in_dim=64, num_classes=10, window=16,
          depths=(2, 2), widths=(64, 128), stage_heads=(2, 4), reduction=4)
# three stages, mlp fusion, r = 2, head_dim 64 (tcgen05 attention), windows 24
HM = dict(width=64, heads=1, hidden=128, seq_len=96, in_dim=32, num_classes=7, window=24,
          depths=(1, 2, 1), widths=(64, 128, 192), stage_heads=(1, 2, 3), reduction=2,
          fusion="mlp")
# Rev-Swin-B geometry (56x56 tokens of 48 features, 7x7 windows, widths 128..1024) with
# fewer blocks per stage so the f64 oracle finishes in seconds
SWIN = dict(width=128, heads=4, hidden=512, seq_len=3136, in_dim=48, num_classes=10,
            window=49, depths=(1, 1, 2, 1), widths=(128, 256, 512, 1024),
            stage_heads=(4, 8, 16, 32), reduction=4)


def maxrel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def l2rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def oracle_cfg(cfg):
    return O.ModelConfig(cfg.depth, cfg.width, cfg.heads, cfg.hidden, cfg.seq_len, cfg.in_dim,
                         cfg.num_classes, cfg.window or None, depths=cfg.depths,
                         widths=cfg.widths, stage_heads=cfg.stage_heads,
                         reduction=cfg.reduction, fusion=cfg.fusion)


def make(kw, batch, seed=0):
    from paper_2306_09342_b200.engine import Engine, ModelConfig, bf16_round
    cfg = ModelConfig(**dict(kw, batch=batch))
    eng = Engine(cfg)
    mc = oracle_cfg(cfg)
    assert eng.n_params == O.param_count(mc)
    p32 = O.init_params(mc, seed, np.float32)
    eng.set_params(p32)
    pref = p32.astype(np.float64)
    off = 0
    for name, shape in O.tensor_shapes(mc):
        n = int(np.prod(shape))
        if len(shape) == 2:  # the GPU computes with bf16 matrices
            pref[off:off + n] = bf16_round(p32[off:off + n])
        off += n
    return eng, mc, p32, pref


def test_tensor_table_matches_oracle_layout():
    eng, mc, _, _ = make(HM, batch=2)
    off, num = eng.tensor_table()
    shapes = O.tensor_shapes(mc)
    assert len(off) == len(shapes)
    o = 0
    for (name, shape), a, n in zip(shapes, off, num):
        assert a == o and n == int(np.prod(shape)), name
        o += n


@pytest.mark.parametrize("kw,batch", [(HA, 4), (HM, 4), (SWIN, 1)], ids=["avg-r4", "mlp-r2",
                                                                         "swin-b-geometry"])
def test_hier_step_grads_match_oracle(kw, batch):
    from paper_2306_09342_b200.engine import REPROP, bf16_bits, bf16_round
    eng, mc, p32, pref = make(kw, batch=batch)
    x, lab = O.synthetic_batch(mc, batch, seed=11)
    eng.set_batch(bf16_bits(x), lab)
    eng.set_lr(0.0)
    eng.step(REPROP, graph=False)
    loss = eng.loss()
    g = eng.grads()
    r = O.step(mc, pref, bf16_round(x).astype(np.float64), lab)
    assert abs(loss - r.loss) / abs(r.loss) < 1e-3
    off = 0
    for name, shape in O.tensor_shapes(mc):
        n = int(np.prod(shape))
        assert maxrel(g[off:off + n], r.grads[off:off + n]) <= TOL_GRAD, name
        off += n
    assert l2rel(g, r.grads) < TOL_L2
    np.testing.assert_array_equal(eng.params(), p32)


@pytest.mark.parametrize("kw", [HA, HM], ids=["avg", "mlp"])
def test_hier_pareprop_bit_identical_to_reprop(kw):
    from paper_2306_09342_b200.engine import PAREPROP, REPROP, bf16_bits
    eng, mc, _, _ = make(kw, batch=4)
    x, lab = O.synthetic_batch(mc, 4, seed=3)
    eng.set_batch(bf16_bits(x), lab)
    eng.set_lr(0.0)
    res = []
    for mode, graph in [(REPROP, False), (PAREPROP, False), (REPROP, True), (PAREPROP, True)]:
        eng.step(mode, graph=graph)
        res.append((eng.loss(), eng.grads()))
    for l, g in res[1:]:
        assert l == res[0][0]
        np.testing.assert_array_equal(g, res[0][1])


def test_hier_vanilla_and_descent():
    """Vanilla (stored activations) agrees with Reprop; SGD lowers the loss with identical
    Reprop / PaReprop trajectories."""
    from paper_2306_09342_b200.engine import PAREPROP, REPROP, VANILLA, bf16_bits
    eng, mc, _, _ = make(HM, batch=4)
    x, lab = O.synthetic_batch(mc, 4, seed=5)
    eng.set_batch(bf16_bits(x), lab)
    eng.set_lr(0.0)
    eng.step(REPROP, graph=False)
    gr = eng.grads()
    eng.enable_vanilla()
    eng.step(VANILLA, graph=False)
    assert l2rel(eng.grads(), gr) < 1e-2
    losses = {}
    for mode in (REPROP, PAREPROP):
        e2, _, _, _ = make(HM, batch=4)
        e2.set_batch(bf16_bits(x), lab)
        e2.set_lr(0.1)  # 0.2 overshoots on this 4-sample batch
        ls = []
        for _ in range(12):
            e2.step(mode)
            ls.append(e2.loss())
        losses[mode] = ls
        e2.close()
    assert losses[REPROP][-1] < 0.8 * losses[REPROP][0], losses[REPROP]
    assert losses[REPROP] == losses[PAREPROP]


def test_hier_activation_ledger():
    """Stored activations: every stage's input + output pair plus one
    (Reprop) or two (PaReprop) block footprints; Vanilla stores every block's input."""
    from paper_2306_09342_b200.engine import (PAREPROP, REPROP, VANILLA, ModelConfig,
                                              activation_bytes)
    cfg = ModelConfig(**dict(SWIN, batch=8, depths=(2, 2, 18, 2)))
    pr, blk = activation_bytes(cfg, REPROP)
    pp, _ = activation_bytes(cfg, PAREPROP)
    pv, _ = activation_bytes(cfg, VANILLA)
    assert pp - pr == blk
    assert pv > pr


@pytest.mark.parametrize("kw", [HA, HM], ids=["avg-r4", "mlp-r2"])
def test_boundary_entry_points_match_oracle(kw):
    """rp_engine_boundary_forward / _vjp (layers.cpp:261-303) vs the oracle's fuse +
    patch_merge and their VJPs on the same bf16-rounded weights; inputs random."""
    from paper_2306_09342_b200.engine import bf16_round
    eng, mc, p32, pref = make(kw, batch=2)
    st = O.stages(mc)
    bnd = O.boundaries_of(mc, pref)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    rng = np.random.default_rng(3)
    B = 2
    mw_off = dict((n, None) for n, _ in O.tensor_shapes(mc))
    for s in range(len(st) - 1):
        g0, g1 = st[s], st[s + 1]
        o1 = rng.standard_normal((B, g0.tokens, g0.d)).astype(np.float32)
        o2 = rng.standard_normal((B, g0.tokens, g0.d)).astype(np.float32)
        y = torch.empty(B * g1.tokens, g1.d, device="cuda")
        eng.boundary_forward(s, t(o1), t(o2), y)
        mw, fw = bnd[s]
        # the GPU fuses in fp32, rounds the fused tensor to bf16 for the merge GEMM
        f, _ = O.fuse(o1.astype(np.float64), o2.astype(np.float64), fw)
        yr, grouped = O.patch_merge(bf16_round(f.astype(np.float32)).astype(np.float64), mw,
                                    mc.reduction)
        assert maxrel(y.cpu().numpy().reshape(yr.shape), yr) < 2e-2
        d1 = rng.standard_normal((B, g1.tokens, g1.d)).astype(np.float32) * 1e-2
        d2 = rng.standard_normal((B, g1.tokens, g1.d)).astype(np.float32) * 1e-2
        do1 = torch.empty(B * g0.tokens, g0.d, device="cuda")
        do2 = torch.empty_like(do1)
        eng.boundary_vjp(s, t(o1), t(o2), t(d1), t(d2), do1, do2)
        dy = bf16_round((d1 + d2).astype(np.float32)).astype(np.float64)
        d_f, d_mw = O.patch_merge_vjp(grouped, mw, mc.reduction, dy)
        _, concat = O.fuse(o1.astype(np.float64), o2.astype(np.float64), fw)
        if concat is not None:
            concat = bf16_round(concat.astype(np.float32)).astype(np.float64)
        r1, r2, d_fw = O.fuse_vjp(concat, fw, d_f)
        assert maxrel(do1.cpu().numpy().reshape(r1.shape), r1) < 2e-2
        assert maxrel(do2.cpu().numpy().reshape(r2.shape), r2) < 2e-2
        g = eng.grads()
        off = 0
        for name, shape in O.tensor_shapes(mc):
            n = int(np.prod(shape))
            if name == f"boundary.{s}.merge_w":
                assert maxrel(g[off:off + n].reshape(shape), d_mw) < 5e-2, name
            if name == f"boundary.{s}.fusion_w":
                assert maxrel(g[off:off + n].reshape(shape), d_fw) < 5e-2, name
            off += n


def test_rev_inverse_round_trip():
    """rp_engine_rev_inverse on a block inside a later stage: recovers the
    block input at the SPEC's f32 round-trip bound and matches the oracle's inverse."""
    eng, mc, p32, pref = make(HM, batch=2)
    st = O.stages(mc)
    g1 = st[1]  # depth 2: block g1.first + 1 is not the stage's first
    b = g1.first + 1
    _, blocks, _ = O.blocks_of(mc, pref)
    rng = np.random.default_rng(5)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    i1 = rng.standard_normal((2, g1.tokens, g1.d)).astype(np.float32)
    i2 = rng.standard_normal((2, g1.tokens, g1.d)).astype(np.float32)
    rows = 2 * g1.tokens
    o1, o2, r1, r2 = (torch.empty(rows, g1.d, device="cuda") for _ in range(4))
    eng.rev_forward(b, t(i1), t(i2), o1, o2)
    eng.rev_inverse(b, o1, o2, r1, r2)
    assert maxrel(r1.cpu().numpy().reshape(i1.shape), i1) < 1e-4
    assert maxrel(r2.cpu().numpy().reshape(i2.shape), i2) < 1e-4
    ri1, ri2 = O.rev_inverse(blocks[b], o1.cpu().numpy().reshape(i1.shape).astype(np.float64),
                             o2.cpu().numpy().reshape(i1.shape).astype(np.float64))
    assert maxrel(r1.cpu().numpy().reshape(i1.shape), ri1) < 2e-2
    assert maxrel(r2.cpu().numpy().reshape(i2.shape), ri2) < 2e-2


def test_hier_adamw_trajectories_identical():
    """AdamW on the hierarchical model: the boundary buckets step with the
    blocks'; Reprop and PaReprop (graph-captured) give the same loss trajectory and the same
    parameters bit for bit, and the loss falls."""
    from paper_2306_09342_b200.engine import PAREPROP, REPROP, Engine, ModelConfig, bf16_bits
    runs = {}
    for mode in (REPROP, PAREPROP):
        cfg = ModelConfig(**dict(HM, batch=4, optimizer=1, weight_decay=0.01))
        eng = Engine(cfg)
        mc = oracle_cfg(cfg)
        eng.set_params(O.init_params(mc, 0, np.float32))
        x, lab = O.synthetic_batch(mc, 4, seed=5)
        eng.set_batch(bf16_bits(x), lab)
        eng.set_lr(2e-3)
        ls = []
        for _ in range(8):
            eng.step(mode)
            ls.append(eng.loss())
        runs[mode] = (ls, eng.params())
        eng.close()
    assert runs[REPROP][0] == runs[PAREPROP][0]
    np.testing.assert_array_equal(runs[REPROP][1], runs[PAREPROP][1])
    assert runs[REPROP][0][-1] < runs[REPROP][0][0]
