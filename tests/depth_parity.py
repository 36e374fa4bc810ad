"""Parity at the depths the reversible path exists for (SURVEY.md §7 hard part 4:
bf16 invertibility compounds over depth). TEST INFRASTRUCTURE: used by
tests/test_gpu_depth.py and, run as a script on the B200, writes the per-depth error table
(profiles/round2_depth_parity.{json,md}) quoted in DESIGN.md §5:

    python tests/depth_parity.py [case ...] --out profiles/round2_depth_parity

For each case one eager Reprop step of the GPU engine runs with the recompute trace on
(rp_engine_set_trace): every block's input pair as the forward saw it -- exactly what the
Vanilla engine stores (in Vanilla mode X_j IS the stash) -- and as lane R reconstructed it
from the block's output in the backward. Reported, per block:
  rec   max|X_rec - X_fwd| / max|X_fwd|   reconstruction error of the inverse chain
  fwd   max|X_fwd - X_oracle| / max|X_oracle|   forward vs the f64 oracle
and per parameter tensor the gradient's max-relative error against the f64 oracle
(oracle/revprop_oracle.py, pinned to the compiled reference), run on the same bf16-rounded
weights and inputs. Parameters come from the engine's own init (the counter RNG the oracle
restates) so the 1.6 B-parameter G48 case does not need a host-side init.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import revprop_oracle as O  # noqa: E402

# name -> (geometry, per-GPU batch)
CASES = {
    # BASELINE.json configs[0]: RevViT-Ti, depth 12, batch 8
    "ti-d12-b8": (dict(depth=12, width=192, heads=3, hidden=768), 8),
    # configs[1] geometry (the benchmarked RevViT-B) at depth 12
    "b-d12-b2": (dict(depth=12, width=768, heads=12, hidden=3072), 2),
    # configs[2] geometry (RevViT-L) at depth 24
    "l-d24-b1": (dict(depth=24, width=1024, heads=16, hidden=4096), 1),
    # configs[4]: RevViT-G-style, depth 48, d 1664, 16 heads of 104
    "g48-d48-b1": (dict(depth=48, width=1664, heads=16, hidden=6656), 1),
    # the same with the exact coupling turned off (plain fp32 residual adds): what the
    # reconstruction costs without it -- reported, held to the looser PLAIN_* bounds
    "b-d12-b2-plain": (dict(depth=12, width=768, heads=12, hidden=3072,
                            exact_coupling_bits=-1), 2),
    "g48-d48-b1-plain": (dict(depth=48, width=1664, heads=16, hidden=6656,
                              exact_coupling_bits=-1), 1),
}
COMMON = dict(seq_len=197, in_dim=768, num_classes=1000)

# stated tolerances (bf16 GEMM operands / fp32 accumulate and residual stream vs f64)
TOL_REC = 0.0      # exact coupling: every recomputed block input equals the stored one bit for bit
TOL_FWD = 2e-2     # forward activations vs the oracle
TOL_GRAD_MATRIX = 2e-2  # per weight-matrix gradient, max-relative
TOL_GRAD = 5e-2    # per parameter tensor incl. the LayerNorm / bias vectors, max-relative
TOL_L2 = 1e-2      # whole gradient vector, relative L2
TOL_LOSS = 1e-3    # relative
# plain fp32 coupling (exact_coupling_bits = -1): the fp32 round-trip error of each inverse
# is re-rounded by the next block's bf16 GEMM operands and compounds over depth
PLAIN_REC_L2 = 3e-2
PLAIN_GRAD_L2 = 2e-2


def l2rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def maxrel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _bf16_round_inplace_f64(p32, mc):
    """The oracle's parameter vector: bf16-rounded matrices (the GPU's GEMM operands),
    fp32 vectors, as f64."""
    from paper_2306_09342_b200.engine import bf16_round
    pref = np.empty(p32.size, np.float64)
    off = 0
    for _, shape in O.tensor_shapes(mc):
        n = int(np.prod(shape))
        seg = p32[off:off + n]
        pref[off:off + n] = bf16_round(seg) if len(shape) == 2 else seg
        off += n
    return pref


def run_case(name, verbose=False):
    import torch
    from paper_2306_09342_b200.engine import (REPROP, VANILLA, Engine, ModelConfig, bf16_bits,
                                              bf16_round)
    geo, batch = CASES[name]
    cfg = ModelConfig(**geo, **COMMON, batch=batch)
    mc = O.ModelConfig(cfg.depth, cfg.width, cfg.heads, cfg.hidden, cfg.seq_len, cfg.in_dim,
                       cfg.num_classes)
    t0 = time.time()
    eng = Engine(cfg)  # parameters from the engine's counter-RNG init (seed 0)
    p32 = eng.params()
    pref = _bf16_round_inplace_f64(p32, mc)
    x, lab = O.synthetic_batch(mc, batch, seed=11)
    eng.set_batch(bf16_bits(x), lab)
    eng.set_lr(0.0)
    nf = eng.trace_floats()
    tf = torch.zeros(nf, device="cuda")
    tr = torch.zeros(nf, device="cuda")
    eng.set_trace(tf.data_ptr(), tr.data_ptr())
    eng.step(REPROP, graph=False)
    loss = eng.loss()
    stats = eng.step_stats()
    g = eng.grads()
    fwd = tf.cpu().numpy()
    rec = tr.cpu().numpy()
    eng.set_trace(0, 0)
    # the same step with every block input stored instead of recomputed (Vanilla): the
    # gradient error that is NOT due to the reconstruction
    eng.enable_vanilla()
    eng.step(VANILLA, graph=False)
    g_van = eng.grads()
    eng.close()
    del tf, tr
    t_gpu = time.time() - t0

    t0 = time.time()
    xr = bf16_round(x).astype(np.float64)
    r = O.step(mc, pref, xr, lab)
    embed_w, blocks, _ = O.blocks_of(mc, pref)
    e = xr @ embed_w
    o = (e, e)
    T, d = batch * mc.seq_len, mc.width
    rows = []
    for b, blk in enumerate(blocks):
        off = b * 2 * T * d
        f1, f2 = fwd[off:off + T * d], fwd[off + T * d:off + 2 * T * d]
        r1, r2 = rec[off:off + T * d], rec[off + T * d:off + 2 * T * d]
        rows.append(dict(block=b,
                         rec=max(maxrel(r1, f1), maxrel(r2, f2)),
                         rec_l2=max(l2rel(r1, f1), l2rel(r2, f2)),
                         fwd=max(maxrel(f1, o[0].reshape(-1)), maxrel(f2, o[1].reshape(-1)))))
        o = O.rev_forward(blk, *o)
    worst_t, worst_v, worst_m, off = [], [], [], 0
    for tname, shape in O.tensor_shapes(mc):
        n = int(np.prod(shape))
        e = maxrel(g[off:off + n], r.grads[off:off + n])
        (worst_m if len(shape) == 2 else worst_v).append((e, tname))
        worst_t.append((e, tname))
        off += n
    l2 = l2rel(g, r.grads)
    t_oracle = time.time() - t0
    res = dict(case=name, depth=cfg.depth, width=cfg.width, heads=cfg.heads, batch=batch,
               loss=loss, loss_oracle=float(r.loss),
               loss_rel=abs(loss - r.loss) / abs(r.loss),
               rec_max=max(x["rec"] for x in rows), fwd_max=max(x["fwd"] for x in rows),
               grad_worst=max(worst_t)[0], grad_worst_tensor=max(worst_t)[1], grad_l2=l2,
               grad_worst_matrix=max(worst_m)[0], grad_worst_vector=max(worst_v)[0],
               rec_l2_max=max(x["rec_l2"] for x in rows),
               vanilla_grad_l2=l2rel(g_van, r.grads),
               vanilla_grad_worst=max(maxrel(g_van[o_:o_ + n_], r.grads[o_:o_ + n_])
                                      for o_, n_ in _slices(mc)),
               reprop_vs_vanilla_l2=l2rel(g, g_van),
               blocks=rows, stats=dict(peak_activation_bytes=stats.peak_activation_bytes,
                                       blocks_processed=stats.blocks_processed),
               seconds_gpu=round(t_gpu, 1), seconds_oracle=round(t_oracle, 1))
    if verbose:
        print(json.dumps({k: v for k, v in res.items() if k != "blocks"}))
    return res


def _slices(mc):
    off = 0
    for _, shape in O.tensor_shapes(mc):
        n = int(np.prod(shape))
        yield off, n
        off += n


def to_markdown(results):
    lines = ["| case | depth | d | batch | loss rel | rec max / L2 (worst block) | fwd max | "
             "grad worst matrix / vector (tensor) | grad L2 | Vanilla grad L2 / worst | "
             "Reprop vs Vanilla L2 |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in results:
        lines.append(f"| {r['case']} | {r['depth']} | {r['width']} | {r['batch']} | "
                     f"{r['loss_rel']:.1e} | {r['rec_max']:.1e} / {r['rec_l2_max']:.1e} | "
                     f"{r['fwd_max']:.1e} | {r['grad_worst_matrix']:.1e} / "
                     f"{r['grad_worst_vector']:.1e} ({r['grad_worst_tensor']}) | "
                     f"{r['grad_l2']:.1e} | {r['vanilla_grad_l2']:.1e} / "
                     f"{r['vanilla_grad_worst']:.1e} | {r['reprop_vs_vanilla_l2']:.1e} |")
    lines.append("")
    lines.append("Per-block reconstruction error, max|X_rec - X_fwd| / max|X_fwd| (relative L2 in "
                 "brackets), block 0 first:")
    lines.append("")
    for r in results:
        lines.append(f"- {r['case']}: " + " ".join(f"{x['rec']:.1e} [{x['rec_l2']:.0e}]"
                                                   for x in r["blocks"]))
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=list(CASES))
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = [run_case(c, verbose=True) for c in a.cases]
    if a.out:
        with open(a.out + ".json", "w") as f:
            json.dump(res, f, indent=1)
        with open(a.out + ".md", "w") as f:
            f.write(to_markdown(res))
