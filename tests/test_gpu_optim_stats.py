"""Optimizer exactness and StepStats on the B200.

* SGD: with lr != 0 the update is p - lr * g in fp32, bit for bit.
* AdamW: five steps match torch.optim.AdamW (fp32, CPU) fed the engine's own
  gradients, within 1e-6 of the parameters' scale.
* StepStats and the live ledger (ledger.hpp:18-104): peak equals the
  ledger formula of each engine, blocks_processed equals the depth, lane busy time is at
  most the wall time, the arena's real activation allocation lies between the Reprop and
  PaReprop ledger peaks and is flat in depth, and the engine's allocations agree with the
  device's own free-memory count (cudaMemGetInfo).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import revprop_oracle as O  # noqa: E402

TI = dict(width=192, heads=3, hidden=768, seq_len=197, in_dim=768, num_classes=100)


def _engine(depth=2, batch=8, **kw):
    from paper_2306_09342_b200.engine import Engine, ModelConfig, bf16_bits
    cfg = ModelConfig(depth=depth, batch=batch, **TI, **kw)
    eng = Engine(cfg)
    mc = O.ModelConfig(cfg.depth, cfg.width, cfg.heads, cfg.hidden, cfg.seq_len, cfg.in_dim,
                       cfg.num_classes)
    x, lab = O.synthetic_batch(mc, batch, seed=21)
    eng.set_batch(bf16_bits(x), lab)
    return eng, cfg


@pytest.mark.parametrize("mode", [1, 2], ids=["reprop", "pareprop"])
@pytest.mark.parametrize("lr", [0.1, 0.37])
def test_sgd_update_bit_exact(mode, lr):
    eng, _ = _engine()
    eng.set_lr(lr)
    p0 = eng.params()
    eng.step(mode, graph=True)
    g = eng.grads()
    p1 = eng.params()
    want = p0 - np.float32(lr) * g          # fp32: one rounding for the product, one for -
    np.testing.assert_array_equal(p1, want)
    # the next step uses the updated parameters (the bf16 shadow was rewritten too)
    eng.step(mode, graph=True)
    g2 = eng.grads()
    np.testing.assert_array_equal(eng.params(), p1 - np.float32(lr) * g2)
    eng.close()


def test_adamw_matches_torch():
    eng, cfg = _engine(optimizer=1, beta1=0.9, beta2=0.999, adam_eps=1e-8, weight_decay=0.05)
    lr = 1e-3
    eng.set_lr(lr)
    p = torch.tensor(eng.params(), dtype=torch.float32, requires_grad=True)
    opt = torch.optim.AdamW([p], lr=lr, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.05,
                            foreach=False)
    scale = float(p.detach().abs().max())
    for step in range(5):
        eng.step(1, graph=False)
        g = eng.grads()
        p.grad = torch.tensor(g)
        opt.step()
        got = eng.params()
        err = float(np.max(np.abs(got - p.detach().numpy())))
        assert err <= 1e-6 * scale, (step, err, scale)
    eng.close()


@pytest.mark.parametrize("depth", [2, 6])
def test_step_stats_and_ledger(depth):
    from paper_2306_09342_b200.engine import PAREPROP, REPROP, VANILLA, activation_bytes
    eng, cfg = _engine(depth=depth)
    eng.enable_vanilla()
    eng.set_instrument(True)
    peaks = {}
    for mode in (VANILLA, REPROP, PAREPROP):
        eng.step(mode, graph=False)
        st = eng.step_stats()
        peaks[mode] = st.peak_activation_bytes
        assert st.mode == mode
        assert st.peak_activation_bytes == activation_bytes(cfg, mode)[0], mode
        assert st.blocks_processed == depth
        assert st.ledger_events > 2 * depth
        assert 0 < st.wall_ns
        assert all(0 < b <= st.wall_ns for b in st.lane_busy_ns), (st.lane_busy_ns, st.wall_ns)
        assert abs(st.loss - eng.loss()) == 0.0
    eng.set_instrument(False)
    eng.step(PAREPROP, graph=True)
    st = eng.step_stats()
    assert st.lane_busy_ns == (-1, -1) and st.peak_activation_bytes == peaks[PAREPROP]
    # the rotating-buffer arena (shared by both engines) sits between the two ledger peaks:
    # it stores the block inputs of lanes R and G in 5 buffers where the ledger counts 6
    blk = activation_bytes(cfg, REPROP)[1]
    act_wo_vanilla = st.arena_activation_bytes - 2 * depth * cfg.batch * cfg.seq_len * cfg.width * 4
    assert peaks[REPROP] <= act_wo_vanilla <= peaks[PAREPROP]
    assert peaks[PAREPROP] - peaks[REPROP] == blk
    # peak(reprop) < peak(vanilla) for depth >= 4 (equal at depth 2: the stash
    # of two block inputs is the stored boundary plus one block footprint minus its caches)
    assert peaks[VANILLA] > peaks[REPROP] if depth >= 4 else peaks[VANILLA] >= peaks[REPROP]
    eng.close()


def test_arena_flat_in_depth_and_matches_device():
    """The activation arena does not grow with depth (the paper's memory claim) and the
    engine's allocations are what the device sees as used (cudaMemGetInfo)."""
    from paper_2306_09342_b200.engine import Engine, ModelConfig
    acts = []
    for depth in (2, 8):
        torch.cuda.synchronize()
        free0, _ = torch.cuda.mem_get_info()
        eng = Engine(ModelConfig(depth=depth, width=768, heads=12, hidden=3072, seq_len=197,
                                 in_dim=768, num_classes=1000, batch=64))
        free1, _ = torch.cuda.mem_get_info()
        eng.step(1, graph=False)
        st = eng.step_stats()
        acts.append(st.arena_activation_bytes)
        used = free0 - free1
        assert st.arena_total_bytes <= used <= st.arena_total_bytes + (256 << 20), (
            used, st.arena_total_bytes)
        eng.close()
    assert acts[0] == acts[1]
