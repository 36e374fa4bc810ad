"""Generate tests/golden/*.npz from the reference compiled in place (oracle/_ref).

    python tests/golden/make_golden.py

Every array here is produced by the reference's own code (ref:proj/core/src/ops.cpp,
layers.cpp, rng.hpp) or by the SPEC restatement in oracle/ref_shim.cpp that calls it.
The fixtures are small (tiny shapes, f64 and f32) so the CPU suite checks the numpy oracle
against them in seconds, including on machines without /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from oracle import revprop_oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

TINY = O.ModelConfig(depth=3, width=16, heads=2, hidden=32, seq_len=8, in_dim=16, num_classes=5)
TINY_WIN = O.ModelConfig(depth=2, width=16, heads=2, hidden=64, seq_len=8, in_dim=16,
                         num_classes=5, window=4)
# hierarchical (Rev-Swin-style): two stages / average fusion, three stages / mlp fusion, r=4
HIER_AVG = O.ModelConfig(depth=4, width=16, heads=2, hidden=32, seq_len=16, in_dim=16,
                         num_classes=5, window=4, depths=(2, 2), widths=(16, 32),
                         stage_heads=(2, 4), reduction=2)
HIER_MLP = O.ModelConfig(depth=4, width=16, heads=2, hidden=48, seq_len=32, in_dim=16,
                         num_classes=5, window=4, depths=(1, 2, 1), widths=(16, 24, 32),
                         stage_heads=(2, 3, 4), reduction=4, fusion="mlp")


def main_hier():
    """reference_golden_hier.npz: the reference's boundary layers (layers.cpp:261-303) on
    random arrays, and hierarchical steps through ref_hier_step."""
    rng = np.random.default_rng(20261017)
    g = {}
    for name, fusion, r in [("bavg", None, 2), ("bmlp", True, 4)]:
        B, N, d, dn = 2, 8, 6, 10
        i1, i2 = rng.standard_normal((B, N, d)), rng.standard_normal((B, N, d))
        mw = rng.standard_normal((r * d, dn))
        fw = rng.standard_normal((2 * d, d)) if fusion else None
        dy = rng.standard_normal((B, N // r, dn))
        y, d1, d2, dmw, dfw = R.boundary(i1, i2, mw, fw, r, dy)
        g.update({f"{name}_{k}": v for k, v in dict(
            i1=i1, i2=i2, merge_w=mw, d_y=dy, y=y, d_i1=d1, d_i2=d2, d_merge_w=dmw).items()})
        if fusion:
            g[f"{name}_fusion_w"], g[f"{name}_d_fusion_w"] = fw, dfw
    for name, mc in [("havg", HIER_AVG), ("hmlp", HIER_MLP)]:
        params = O.init_params(mc, 5)
        assert params.size == R.hier_param_count(mc)
        x, lab = O.synthetic_batch(mc, 2, seed=13)
        loss, grads = R.hier_step(mc, params, x, lab)
        g.update({f"{name}_params": params, f"{name}_x": x, f"{name}_labels": lab,
                  f"{name}_loss": np.float64(loss), f"{name}_grads": grads})
    np.savez_compressed(os.path.join(OUT, "reference_golden_hier.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_golden_hier.npz"), len(g), "arrays")


def main():
    assert R.build(), "needs /root/reference (or a prebuilt oracle/_ref)"
    g = {}
    # rng.hpp known vectors
    for seed, stream in [(0, 0), (7, 123), (2 ** 63 + 5, (1 << 56) | (3 << 32) | 17)]:
        u, z, t = R.rng(seed, stream, 16)
        key = f"rng_{seed}_{stream}"
        g[key + "_u64"], g[key + "_normal"], g[key + "_trunc"] = u, z, t
    rng = np.random.default_rng(20260101)
    # layer_norm (ops.cpp:264-345)
    x = rng.standard_normal((5, 12)) * 3 + 1
    gm, bt, dy = rng.standard_normal(12), rng.standard_normal(12), rng.standard_normal((5, 12))
    y, inv, dx, dg, db = R.layer_norm(x, gm, bt, 1e-5, dy)
    g.update(ln_x=x, ln_g=gm, ln_b=bt, ln_dy=dy, ln_y=y, ln_inv=inv, ln_dx=dx, ln_dg=dg, ln_db=db)
    for name, mc in [("full", TINY), ("win", TINY_WIN)]:
        params = O.init_params(mc, 3)
        pb = R.block_slice(mc, params, 1)
        pf, pgp = R.split_block(mc, pb)
        B = 2
        xx = rng.standard_normal((B, mc.seq_len, mc.width))
        dyy = rng.standard_normal(xx.shape)
        ya, dxa, dpa = R.attention(mc, pf, xx, dyy)
        ym, dxm, dpm = R.mlp(mc, pgp, xx, dyy)
        i1, i2 = rng.standard_normal(xx.shape), rng.standard_normal(xx.shape)
        o1, o2 = R.rev_forward(mc, pb, i1, i2)
        d1, d2 = rng.standard_normal(xx.shape), rng.standard_normal(xx.shape)
        (ri1, ri2), (di1, di2), dpb = R.rev_backward_local(mc, pb, o1, o2, d1, d2)
        xin, lab = O.synthetic_batch(mc, 3, seed=9)
        loss, grads, peak, _ = R.step(mc, params, xin, lab, "reprop")
        p32 = params.astype(np.float32)
        loss32, grads32, _, _ = R.step(mc, p32, xin.astype(np.float32), lab, "reprop")
        g.update({f"{name}_{k}": v for k, v in dict(
            params=params, x=xx, dy=dyy, attn_y=ya, attn_dx=dxa, attn_dp=dpa, mlp_y=ym,
            mlp_dx=dxm, mlp_dp=dpm, i1=i1, i2=i2, o1=o1, o2=o2, d1=d1, d2=d2, ri1=ri1, ri2=ri2,
            di1=di1, di2=di2, dpb=dpb, step_x=xin, step_labels=lab, step_loss=np.float64(loss),
            step_grads=grads, step_loss32=np.float64(loss32), step_grads32=grads32).items()})
    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_golden.npz"), len(g), "arrays")


if __name__ == "__main__":
    if "--hier-only" not in sys.argv:
        main()
    main_hier()
