"""CPU suite: pins the numpy oracle to the reference (compiled in place, oracle/_ref) and to
the committed golden fixtures, and checks the SPEC's known answers and invariants
(SPEC.md:40-505). No GPU needed."""
import os

import numpy as np
import pytest

from oracle import revprop_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))

TINY = O.ModelConfig(depth=3, width=16, heads=2, hidden=32, seq_len=8, in_dim=16, num_classes=5)
TINY_WIN = O.ModelConfig(depth=2, width=16, heads=2, hidden=64, seq_len=8, in_dim=16,
                         num_classes=5, window=4)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def have_ref():
    try:
        from oracle import ref as R
        return R.available() or R.build()
    except Exception:
        return False


needs_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")


# ---------------------------------------------------------------- golden fixtures
def test_rng_matches_reference_vectors():
    for key in [k for k in GOLD.files if k.startswith("rng_") and k.endswith("_u64")]:
        _, seed, stream, _ = key.split("_")
        seed, stream = np.uint64(int(seed)), np.uint64(int(stream))
        n = GOLD[key].size
        u = O.rng_u64(seed, stream, np.arange(n, dtype=np.uint64))
        assert np.array_equal(u, GOLD[key])
        z = O.rng_normal(seed, stream, np.arange(0, 2 * n, 2, dtype=np.uint64))
        assert np.array_equal(z, GOLD[key.replace("_u64", "_normal")])


def test_layer_norm_golden():
    y, cache = O.layer_norm(GOLD["ln_x"], GOLD["ln_g"], GOLD["ln_b"])
    assert rel(y, GOLD["ln_y"]) < 1e-13
    assert rel(cache[1], GOLD["ln_inv"]) < 1e-13
    dx, dg, db = O.layer_norm_vjp(cache, GOLD["ln_g"], GOLD["ln_dy"])
    assert rel(dx, GOLD["ln_dx"]) < 1e-12
    assert rel(dg, GOLD["ln_dg"]) < 1e-13 and rel(db, GOLD["ln_db"]) < 1e-13


@pytest.mark.parametrize("name,mc", [("full", TINY), ("win", TINY_WIN)])
def test_layers_revcore_step_golden(name, mc):
    G = lambda k: GOLD[f"{name}_{k}"]
    params = G("params")
    assert np.array_equal(params, O.init_params(mc, 3))  # build_model is deterministic
    _, blocks, _ = O.blocks_of(mc, params)
    b = blocks[1]
    y, c = O.attention_forward(G("x"), b.f)
    assert rel(y, G("attn_y")) < 1e-12
    dx, dp = O.attention_vjp(c, b.f, G("dy"))
    assert rel(dx, G("attn_dx")) < 1e-11
    dpf = np.concatenate([np.ravel(dp[k]) for k in ("d_w_qkv", "d_w_out", "d_ln_gamma",
                                                     "d_ln_beta")])
    assert rel(dpf, G("attn_dp")) < 1e-11
    y, c = O.mlp_forward(G("x"), b.g)
    assert rel(y, G("mlp_y")) < 1e-12
    dx, dp = O.mlp_vjp(c, b.g, G("dy"))
    assert rel(dx, G("mlp_dx")) < 1e-11
    o1, o2 = O.rev_forward(b, G("i1"), G("i2"))
    assert rel(o1, G("o1")) < 1e-12 and rel(o2, G("o2")) < 1e-12
    (i1, i2), (d1, d2), (fg, gg) = O.rev_backward_local(b, G("o1"), G("o2"), G("d1"), G("d2"))
    assert rel(i1, G("ri1")) < 1e-12 and rel(i2, G("ri2")) < 1e-12
    assert rel(d1, G("di1")) < 1e-11 and rel(d2, G("di2")) < 1e-11
    r = O.step(mc, params, G("step_x"), G("step_labels"))
    assert abs(r.loss - float(G("step_loss"))) < 1e-12
    assert rel(r.grads, G("step_grads")) < 1e-10
    # the f32 reference run agrees with the f64 oracle to f32 rounding
    assert rel(G("step_grads32"), G("step_grads")) < 1e-4


# ---------------------------------------------------------------- live reference pins
@needs_ref
@pytest.mark.parametrize("mc", [TINY, TINY_WIN,
                                O.ModelConfig(2, 64, 1, 128, 12, 32, 7),
                                O.ModelConfig(2, 192, 3, 768, 20, 64, 10)],
                         ids=["tiny", "window", "one-head", "ti-width"])
def test_oracle_matches_compiled_reference(mc):
    from oracle import ref as R
    params = O.init_params(mc, 11)
    x, lab = O.synthetic_batch(mc, 2, seed=4)
    loss, grads, _, _ = R.step(mc, params, x, lab, "reprop")
    r = O.step(mc, params, x, lab)
    assert abs(r.loss - loss) < 1e-12
    assert rel(r.grads, grads) < 1e-10


@needs_ref
def test_reference_pareprop_bit_identical_to_reprop_50_seeds():
    """Acceptance 3 on the CPU reference: f32, 50 seeded trials."""
    from oracle import ref as R
    mc = O.ModelConfig(depth=4, width=16, heads=2, hidden=32, seq_len=6, in_dim=16, num_classes=5)
    for seed in range(50):
        p = O.init_params(mc, seed, np.float32)
        x, lab = O.synthetic_batch(mc, 2, seed=100 + seed)
        x = x.astype(np.float32)
        l1, g1, _, _ = R.step(mc, p, x, lab, "reprop")
        l2, g2, _, _ = R.step(mc, p, x, lab, "pareprop")
        assert l1 == l2 and np.array_equal(g1, g2)


@needs_ref
def test_reference_pareprop_memory_and_slots():
    """Acceptance 5 and 7: extra peak <= 2 block footprints; slot order per lane."""
    from oracle import ref as R
    mc = O.ModelConfig(depth=3, width=64, heads=1, hidden=256, seq_len=64, in_dim=32,
                       num_classes=5)
    p = O.init_params(mc, 0)
    x, lab = O.synthetic_batch(mc, 2, seed=1)
    _, _, peak_r, _ = R.step(mc, p, x, lab, "reprop")
    _, _, peak_p, sl = R.step(mc, p, x, lab, "pareprop", slots=True)
    T = 2 * mc.seq_len
    d, h = mc.width, mc.hidden
    # one block's recomputed set: inputs (2) + attention cache (x_hat, h, q, k, v, att,
    # probs) + MLP cache (x_hat, h, u, a), f64
    footprint = 8 * (2 * T * d + 6 * T * d + 2 * mc.heads * mc.seq_len ** 2 + T + 2 * T * d
                     + 2 * T * h + T)
    assert peak_r <= peak_p <= peak_r + 2 * footprint
    R_ = {int(b): (t0, t1) for lane, b, t0, t1 in sl if lane == 0}
    G_ = {int(b): (t0, t1) for lane, b, t0, t1 in sl if lane == 1}
    assert sorted(R_) == [1, 2, 3] and sorted(G_) == [1, 2, 3]
    for b in (1, 2, 3):
        assert G_[b][0] >= R_[b][1]  # G_b consumes R_b
    for b in (1, 2):
        assert R_[b][0] >= G_[b + 1][0] or R_[b][0] >= R_[b + 1][1]  # R runs <= 1 block ahead


# ---------------------------------------------------------------- SPEC known answers
def test_spec_known_answers():
    c = 3.7
    assert np.allclose(O.row_softmax(np.array([c, c + np.log(2.0)])), [1 / 3, 2 / 3], atol=1e-15)
    assert np.allclose(O.row_softmax(np.zeros(4)), 0.25)
    assert O.gelu(np.array(0.0)) == 0.0
    assert abs(O.gelu(np.array(10.0)) - 10.0) < 1e-4
    assert O.gelu_vjp(np.array(0.0), np.array(1.0)) == 0.5
    y, _ = O.layer_norm(np.ones((1, 4)), np.ones(4), np.zeros(4))
    assert np.all(y == 0.0)
    y, _ = O.layer_norm(np.array([[-1.0, 1.0]]), np.ones(2), np.zeros(2), eps=1e-300)
    assert np.allclose(y, [[-1, 1]])
    logits = np.zeros((3, 7))
    loss, _ = O.loss_and_grad_head(logits, np.array([0, 3, 6]))
    assert abs(loss - np.log(7)) < 1e-14
    assert np.array_equal(O.sgd_update(np.arange(5.0), np.ones(5), 0.0), np.arange(5.0))
    assert abs(O.sgd_update(np.array([1.0]), np.array([2.0]), 0.1)[0] - 0.8) < 1e-15


def test_scalar_surrogate_coupling():
    """SPEC.md:220, 229, 238 with F(x) = 2x, G(x) = 3x."""
    F = lambda x: 2 * x
    G = lambda x: 3 * x
    i1, i2 = 1.0, 2.0
    o2 = i2 + F(i1)
    o1 = i1 + G(o2)
    assert (o1, o2) == (13.0, 4.0)
    j1 = o1 - G(o2)
    assert (j1, o2 - F(j1)) == (1.0, 2.0)
    d_o1 = d_o2 = 1.0
    d_o2t = d_o2 + 3 * d_o1  # VJP_G
    d_i1 = d_o1 + 2 * d_o2t  # VJP_F
    assert (d_o2t, d_i1) == (4.0, 9.0)


def test_zero_params_are_zero_maps_and_identity_blocks():
    mc = TINY
    p = np.zeros(O.param_count(mc))
    _, blocks, _ = O.blocks_of(mc, p)
    x = np.random.default_rng(0).standard_normal((2, mc.seq_len, mc.width))
    assert np.all(O.attention_forward(x, blocks[0].f)[0] == 0)
    assert np.all(O.mlp_forward(x, blocks[0].g)[0] == 0)
    o1, o2 = O.rev_forward(blocks[0], x, 2 * x)
    assert np.array_equal(o1, x) and np.array_equal(o2, 2 * x)


def test_window_equal_to_n_is_full_attention():
    p = O.init_params(TINY, 1)
    _, blocks, _ = O.blocks_of(TINY, p)
    f = blocks[0].f
    x = np.random.default_rng(2).standard_normal((2, TINY.seq_len, TINY.width))
    y_full = O.attention_forward(x, f)[0]
    f.window = TINY.seq_len
    assert np.array_equal(O.attention_forward(x, f)[0], y_full)


def test_round_trip_f64_and_f32():
    """Acceptance 1: rev_inverse(rev_forward(x)) == x within 1e-12 (f64) / 1e-5 (f32)."""
    rng = np.random.default_rng(5)
    for trial in range(20):
        mc = O.ModelConfig(1, 16, 2, 32, 8, 16, 5)
        p = O.init_params(mc, trial) * 5  # non-trivial blocks
        _, blocks, _ = O.blocks_of(mc, p)
        i1, i2 = rng.standard_normal((2, 2, 8, 16))
        j1, j2 = O.rev_inverse(blocks[0], *O.rev_forward(blocks[0], i1, i2))
        assert rel(j1, i1) < 1e-12 and rel(j2, i2) < 1e-12


def test_finite_differences_rev_backward_local():
    """Acceptance 2: central differences (f64, step 1e-6) within rel 1e-6 on a tiny block."""
    mc = O.ModelConfig(1, 4, 1, 8, 3, 4, 3)
    rng = np.random.default_rng(7)
    p = rng.standard_normal(O.param_count(mc)) * 0.5
    _, blocks, _ = O.blocks_of(mc, p)
    b = blocks[0]
    i1, i2 = rng.standard_normal((2, 1, 3, 4))
    w1, w2 = rng.standard_normal((2, 1, 3, 4))
    o1, o2 = O.rev_forward(b, i1, i2)
    _, (d_i1, d_i2), (fg, gg) = O.rev_backward_local(b, o1, o2, w1, w2)

    def L(a1, a2):
        q1, q2 = O.rev_forward(b, a1, a2)
        return float((q1 * w1).sum() + (q2 * w2).sum())

    eps = 1e-6
    for arr, grad in ((i1, d_i1), (i2, d_i2)):
        num = np.zeros_like(arr)
        for idx in np.ndindex(arr.shape):
            old = arr[idx]
            arr[idx] = old + eps
            lp = L(i1, i2)
            arr[idx] = old - eps
            lm = L(i1, i2)
            arr[idx] = old
            num[idx] = (lp - lm) / (2 * eps)
        assert rel(grad, num) < 1e-6
    # a parameter: w_qkv
    W = b.f.w_qkv
    num = np.zeros_like(W)
    for idx in np.ndindex(W.shape):
        old = W[idx]
        W[idx] = old + eps
        lp = L(i1, i2)
        W[idx] = old - eps
        lm = L(i1, i2)
        W[idx] = old
        num[idx] = (lp - lm) / (2 * eps)
    assert rel(fg["d_w_qkv"], num) < 1e-6


def test_pareprop_numpy_identical_and_slot_order():
    mc = O.ModelConfig(3, 16, 2, 32, 8, 16, 5)
    p = O.init_params(mc, 2)
    x, lab = O.synthetic_batch(mc, 2, seed=3)
    a = O.step(mc, p, x, lab, "reprop")
    b = O.step(mc, p, x, lab, "pareprop")
    assert a.loss == b.loss and np.array_equal(a.grads, b.grads)
    assert b.slots[0] == ("R", 3) and b.slots[-1] == ("G", 1)
    gi = [s for s in b.slots if s[0] == "G"]
    assert gi == [("G", 3), ("G", 2), ("G", 1)]


def test_makespan_oracle():
    """Acceptance 6a: equal slot times -> PaReprop/Reprop backward makespan = (L+1)/(2L)."""
    for L in (1, 2, 3, 12, 48, 1000):
        r = O.makespan(L, 1.0, 1.0, pipelined=True) / O.makespan(L, 1.0, 1.0, pipelined=False)
        assert abs(r - (L + 1) / (2 * L)) < 1e-15
    # forward:backward = 1:2 -> hides 25% in the limit (§3.3)
    L = 10 ** 6
    assert abs(O.makespan(L, 1, 2, True) / O.makespan(L, 1, 2, False) - 2 / 3) < 1e-5


def test_sgd_descent_oracle():
    """Acceptance 9 on the oracle: 20 SGD steps on a fixed 8-sample batch."""
    mc = O.ModelConfig(2, 16, 2, 32, 8, 16, 5)
    p = O.init_params(mc, 1)
    x, lab = O.synthetic_batch(mc, 8, seed=2)
    losses = []
    for _ in range(20):
        r = O.step(mc, p, x, lab)
        losses.append(r.loss)
        p = O.sgd_update(p, r.grads, 1.0)
    assert losses[-1] < 0.8 * losses[0]


# ---------------------------------------------------------------- data parallel (gloo)
# (widths / hidden multiples of 64, head_dim a multiple of 8: the engine's constraints)
DP_ISO = dict(depth=2, width=64, heads=2, hidden=128, seq_len=8, in_dim=16, num_classes=5)
DP_HIER = dict(depth=4, width=64, heads=2, hidden=128, seq_len=32, in_dim=16, num_classes=5,
               window=4, depths=(1, 2, 1), widths=(64, 128, 192), stage_heads=(2, 4, 6),
               reduction=4, fusion="mlp")


def _engine_cfg(kw):
    from paper_2306_09342_b200.engine import ModelConfig
    kw = dict(kw)
    return ModelConfig(**kw)


def _dp_worker(rank, world, port, kw, q):
    try:
        _dp_work(rank, world, port, kw, q)
    except Exception as ex:  # report instead of leaving the parent waiting on the queue
        q.put((rank, repr(ex), None, None))


def _dp_work(rank, world, port, kw, q):
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    import torch
    import torch.distributed as dist
    from oracle import revprop_oracle as O2
    from paper_2306_09342_b200.engine import bucket_plan
    mc = O2.ModelConfig(**kw)
    p = O2.init_params(mc, 3)
    x, lab = O2.synthetic_batch(mc, 4, seed=8)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    shard = slice(rank * x.shape[0] // world, (rank + 1) * x.shape[0] // world)
    r = O2.step(mc, p, x[shard], lab[shard])
    g = torch.from_numpy(r.grads.copy())
    # the engine's own bucket plan (rp_model_bucket_plan, the function its step enqueues
    # from): one all-reduce (sum) per bucket in the engine's issue order ...
    plan = bucket_plan(_engine_cfg(kw))
    for off, n, _ in plan:
        sl = g[off:off + n]
        dist.all_reduce(sl)
        g[off:off + n] = sl
    # ... then that bucket's SGD step with 1/world folded in (engine.cpp bucket_update)
    lr = 0.5
    p_new = p - (lr * (1.0 / world)) * g.numpy()
    q.put((rank, g.numpy() / world, p_new, plan))
    dist.destroy_process_group()


@pytest.mark.parametrize("kw", [DP_ISO, DP_HIER], ids=["isotropic", "hierarchical"])
def test_data_parallel_buckets_gloo(kw):
    """The N>1 path on world_size 2 (gloo, two processes) with the engine's bucket plan: the
    buckets tile the parameter vector exactly once, the per-bucket all-reduced mean of the
    per-shard gradients equals the full-batch gradient, and both ranks end with identical
    parameters equal to full-batch SGD."""
    import multiprocessing as mp
    import socket
    mc = O.ModelConfig(**kw)
    p = O.init_params(mc, 3)
    x, lab = O.synthetic_batch(mc, 4, seed=8)
    full = O.step(mc, p, x, lab).grads
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dp_worker, args=(r, 2, port, kw, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    out = {}
    for _ in range(2):
        rk, g, pn, plan = q.get(timeout=180)
        assert plan is not None, g
        out[rk] = (g, pn, plan)
    for pr in ps:
        pr.join(timeout=60)
    plan = out[0][2]
    cover = np.zeros(p.size, np.int64)
    for off, n, _ in plan:
        cover[off:off + n] += 1
    assert np.all(cover == 1)
    assert [k for _, _, k in plan][0] == "head" and plan[-1][2] == "embed"
    assert rel(out[0][0], full) < 1e-12 and np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert rel(out[0][1], p - 0.5 * full) < 1e-12


# ---------------------------------------------------------------- hierarchical (Rev-Swin) path
GOLD_H = np.load(os.path.join(HERE, "golden", "reference_golden_hier.npz"))
HIER_AVG = O.ModelConfig(depth=4, width=16, heads=2, hidden=32, seq_len=16, in_dim=16,
                         num_classes=5, window=4, depths=(2, 2), widths=(16, 32),
                         stage_heads=(2, 4), reduction=2)
HIER_MLP = O.ModelConfig(depth=4, width=16, heads=2, hidden=48, seq_len=32, in_dim=16,
                         num_classes=5, window=4, depths=(1, 2, 1), widths=(16, 24, 32),
                         stage_heads=(2, 3, 4), reduction=4, fusion="mlp")


@pytest.mark.parametrize("name,r", [("bavg", 2), ("bmlp", 4)])
def test_boundary_golden(name, r):
    """fuse -> patch_merge and the VJPs vs the reference's layers.cpp:261-303."""
    G = lambda k: GOLD_H[f"{name}_{k}"]
    fw = G("fusion_w") if f"{name}_fusion_w" in GOLD_H.files else None
    f, concat = O.fuse(G("i1"), G("i2"), fw)
    y, grouped = O.patch_merge(f, G("merge_w"), r)
    assert rel(y, G("y")) < 1e-13
    d_f, d_mw = O.patch_merge_vjp(grouped, G("merge_w"), r, G("d_y"))
    d1, d2, d_fw = O.fuse_vjp(concat, fw, d_f)
    assert rel(d1, G("d_i1")) < 1e-13 and rel(d2, G("d_i2")) < 1e-13
    assert rel(d_mw, G("d_merge_w")) < 1e-13
    if fw is not None:
        assert rel(d_fw, G("d_fusion_w")) < 1e-13


def test_boundary_spec_known_answers():
    """SPEC.md:155-172 examples."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 6, 4))
    sel = np.concatenate([np.eye(4), np.zeros((4, 4))])  # merge_w = [I; 0]
    y, _ = O.patch_merge(x, sel, 2)
    assert np.array_equal(y, x[:, 0::2])  # even-indexed tokens
    assert y.shape == (2, 3, 4)
    assert np.array_equal(O.fuse(x, x)[0], x)  # idempotent average
    assert np.all(O.fuse(x, -x)[0] == 0)  # cancellation
    eye2 = np.concatenate([np.eye(4), np.eye(4)])  # stacked identity -> i1 + i2
    z = rng.standard_normal(x.shape)
    assert np.allclose(O.fuse(x, z, eye2)[0], x + z, atol=1e-15)
    with pytest.raises(AssertionError):
        O.patch_merge(x[:, :5], sel, 2)


@pytest.mark.parametrize("name,mc", [("havg", HIER_AVG), ("hmlp", HIER_MLP)])
def test_hier_step_golden(name, mc):
    G = lambda k: GOLD_H[f"{name}_{k}"]
    params = G("params")
    assert np.array_equal(params, O.init_params(mc, 5))
    # shape chain: tokens after stage s = N / r^s, widths chain
    st = O.stages(mc)
    assert [g.tokens for g in st] == [mc.seq_len // mc.reduction ** s for s in range(len(st))]
    r = O.step(mc, params, G("x"), G("labels"))
    assert abs(r.loss - float(G("loss"))) < 1e-12
    assert rel(r.grads, G("grads")) < 1e-10
    p = O.step(mc, params, G("x"), G("labels"), engine="pareprop")
    assert p.loss == r.loss and np.array_equal(p.grads, r.grads)
    # slot order per stage: blocks last -> first within a stage, stages last -> first
    gs = [b for lane, b in r.slots if lane == "G"]
    assert gs == list(range(mc.depth, 0, -1))


@needs_ref
def test_hier_oracle_matches_compiled_reference():
    from oracle import ref as R
    for mc in (HIER_AVG, HIER_MLP):
        params = O.init_params(mc, 21)
        x, lab = O.synthetic_batch(mc, 3, seed=8)
        loss, grads = R.hier_step(mc, params, x, lab)
        r = O.step(mc, params, x, lab)
        assert abs(r.loss - loss) < 1e-12
        assert rel(r.grads, grads) < 1e-10
