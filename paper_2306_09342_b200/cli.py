"""bench-cli on the B200 engine.

    python -m paper_2306_09342_b200.cli bench  configs/revvit_b.cfg [--out bench.csv]
    python -m paper_2306_09342_b200.cli verify configs/verify_tiny.cfg
    python -m paper_2306_09342_b200.cli probe  configs/revvit_b.cfg --budget-bytes 80e9

Config files are flat UTF-8 `key = value` text with dotted keys; command-line
flags override file keys. CSV columns, header always written:
    engine,batch,depth,width,seq_len,throughput_mean,throughput_std,peak_bytes,wall_ns_per_step
Throughput is samples/s per repeat (device-timed, CUDA events around `steps` graph-replayed
training steps after `warmup` steps); mean and sample std over `repeats`; peak_bytes is the
engine's activation ledger (rp_activation_bytes). `verify` checks the GPU engine against
the CPU oracle and exits non-zero on any failure.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import statistics
import sys

import numpy as np

ENGINES = {"vanilla": 0, "reprop": 1, "pareprop": 2}
DEFAULTS = {
    "model.depth": "12", "model.width": "768", "model.heads": "12", "model.mlp_ratio": "4",
    "model.seq_len": "197", "model.in_dim": "768", "model.num_classes": "1000",
    "model.window": "0", "bench.batch_sizes": "256", "bench.engines": "reprop,pareprop",
    "bench.steps": "10", "bench.warmup": "2", "bench.repeats": "3", "bench.out": "bench.csv",
    "optim.kind": "sgd", "optim.lr": "0.001", "seed": "0",
    # hierarchical: model.kind = hierarchical plus comma lists per stage
    "model.kind": "isotropic", "model.depths": "", "model.widths": "", "model.stage_heads": "",
    "model.reduction": "2", "model.fusion": "average",
}


def read_config(path: str | None) -> dict:
    cfg = dict(DEFAULTS)
    if path:
        with open(path, encoding="utf-8") as f:
            for ln, line in enumerate(f, 1):
                line = line.split("#", 1)[0].strip()
                if not line:
                    continue
                if "=" not in line:
                    raise SystemExit(f"{path}:{ln}: expected `key = value`")
                k, v = (t.strip() for t in line.split("=", 1))
                cfg[k] = v
    return cfg


def model_config(cfg: dict, batch: int):
    from .engine import ModelConfig
    w = int(cfg["model.width"])
    hier = {}
    if cfg["model.kind"] == "hierarchical":
        ints = lambda k: tuple(int(v) for v in cfg[k].split(",") if v.strip())
        hier = dict(depths=ints("model.depths"), widths=ints("model.widths"),
                    stage_heads=ints("model.stage_heads"), reduction=int(cfg["model.reduction"]),
                    fusion=cfg["model.fusion"])
    elif cfg["model.kind"] != "isotropic":
        raise SystemExit("model.kind must be isotropic or hierarchical")
    return ModelConfig(depth=int(cfg["model.depth"]), width=w, heads=int(cfg["model.heads"]),
                       hidden=int(cfg["model.mlp_ratio"]) * w, seq_len=int(cfg["model.seq_len"]),
                       in_dim=int(cfg["model.in_dim"]), num_classes=int(cfg["model.num_classes"]),
                       window=int(cfg["model.window"]), batch=batch, seed=int(cfg["seed"]),
                       optimizer=1 if cfg["optim.kind"] == "adamw" else 0, **hier)


def cmd_bench(cfg: dict) -> int:
    import torch

    from .engine import Engine, activation_bytes
    engines = [e.strip() for e in cfg["bench.engines"].split(",") if e.strip()]
    steps, warm, reps = int(cfg["bench.steps"]), int(cfg["bench.warmup"]), int(cfg["bench.repeats"])
    out = cfg["bench.out"]
    rows = []
    for B in [int(b) for b in cfg["bench.batch_sizes"].split(",")]:
        mc = model_config(cfg, B)
        try:
            eng = Engine(mc)
        except Exception as ex:  # infeasible batch is recorded, not fatal
            print(f"batch {B}: infeasible ({ex})", file=sys.stderr)
            continue
        eng.set_lr(float(cfg["optim.lr"]))
        if "vanilla" in engines:
            eng.enable_vanilla()
        stream = torch.cuda.ExternalStream(eng.stream_ptr)
        for name in engines:
            mode = ENGINES[name]
            for _ in range(warm):
                eng.step(mode)
            eng.sync()
            thr, wall = [], []
            for _ in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(steps):
                    eng.step(mode)
                b.record(stream)
                b.synchronize()
                ms = a.elapsed_time(b)
                thr.append(B * steps / (ms / 1e3))
                wall.append(ms * 1e6 / steps)
            peak, _ = activation_bytes(mc, mode)
            row = dict(engine=name, batch=B, depth=mc.depth, width=mc.width, seq_len=mc.seq_len,
                       throughput_mean=statistics.mean(thr),
                       throughput_std=statistics.stdev(thr) if len(thr) > 1 else 0.0,
                       peak_bytes=peak, wall_ns_per_step=int(statistics.mean(wall)))
            rows.append(row)
            print(json.dumps(row), flush=True)
        eng.close()
    cols = ["engine", "batch", "depth", "width", "seq_len", "throughput_mean", "throughput_std",
            "peak_bytes", "wall_ns_per_step"]
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=cols)
        w.writeheader()
        w.writerows(rows)
    print(f"{'engine':>9} {'batch':>6} {'img/s':>10} {'+-':>8} {'peak MB':>9}")
    for r in rows:
        print(f"{r['engine']:>9} {r['batch']:>6} {r['throughput_mean']:>10.1f} "
              f"{r['throughput_std']:>8.1f} {r['peak_bytes'] / 1e6:>9.1f}")
    return 0


def cmd_verify(cfg: dict, inject_fault: bool = False) -> int:
    """Engine vs oracle on a small model: step grads (stated tolerance), PaReprop == Reprop
    bit-exact, Vanilla ~ Reprop, lr = 0 leaves the model unchanged. inject_fault corrupts
    every block's VJP first: the report must then flag the gradient checks
    and the exit status be nonzero."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import revprop_oracle as O

    from .engine import PAREPROP, REPROP, VANILLA, Engine, bf16_bits, bf16_round
    B = int(cfg["bench.batch_sizes"].split(",")[0])
    mc = model_config(cfg, B)
    om = O.ModelConfig(mc.depth, mc.width, mc.heads, mc.hidden, mc.seq_len, mc.in_dim,
                       mc.num_classes, mc.window or None, depths=mc.depths, widths=mc.widths,
                       stage_heads=mc.stage_heads, reduction=mc.reduction, fusion=mc.fusion)
    eng = Engine(mc)
    p32 = O.init_params(om, int(cfg["seed"]), np.float32)
    eng.set_params(p32)
    x, lab = O.synthetic_batch(om, B, seed=int(cfg["seed"]) + 1)
    eng.set_batch(bf16_bits(x), lab)
    eng.set_lr(0.0)
    eng.enable_vanilla()
    if inject_fault:
        eng.inject_fault(1)
    report = []

    def check(name, ok, value):
        report.append((name, bool(ok), value))

    eng.step(REPROP, graph=False)
    g_r, l_r = eng.grads(), eng.loss()
    eng.step(PAREPROP, graph=True)
    check("pareprop == reprop (bit-exact grads)", np.array_equal(eng.grads(), g_r), 0.0)
    eng.step(VANILLA, graph=False)
    g_v = eng.grads()
    rel_v = float(np.linalg.norm(g_v - g_r) / np.linalg.norm(g_r))
    check("vanilla ~ reprop (rel L2 <= 1e-3)", rel_v <= 1e-3, rel_v)
    check("lr = 0 leaves parameters unchanged", np.array_equal(eng.params(), p32), 0.0)
    pref = p32.astype(np.float64)
    off = 0
    for _, shape in O.tensor_shapes(om):
        n = int(np.prod(shape))
        if len(shape) == 2:
            pref[off:off + n] = bf16_round(p32[off:off + n])
        off += n
    r = O.step(om, pref, bf16_round(x).astype(np.float64), lab)
    rl = abs(l_r - r.loss) / abs(r.loss)
    check("loss vs oracle (rel <= 1e-3)", rl <= 1e-3, rl)
    rg = float(np.linalg.norm(g_r - r.grads) / np.linalg.norm(r.grads))
    check("grads vs oracle (rel L2 <= 2e-2)", rg <= 2e-2, rg)
    worst = 0.0
    off = 0
    for name, shape in O.tensor_shapes(om):
        n = int(np.prod(shape))
        a, b = g_r[off:off + n], r.grads[off:off + n]
        worst = max(worst, float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)))
        off += n
    check("per-tensor grads vs oracle (max rel <= 5e-2)", worst <= 5e-2, worst)
    # round trip (f32 bound 1e-4): rev_forward, then the inverse inside
    # rev_backward_local, on a block that is not its stage's first; F and G are recomputed
    # by the same kernels, so what remains is fp32 add / subtract rounding (and the bf16
    # LayerNorm output of the recovered i1 rounding the other way in a few elements)
    blk = next((g.first + 1 for g in O.stages(om) if g.depth >= 2), None)
    if blk is not None and not inject_fault:
        import torch
        g = next(g for g in O.stages(om) if g.first <= blk < g.first + g.depth)
        rows = B * g.tokens
        gen = torch.Generator(device="cuda").manual_seed(7)
        i1 = torch.randn(rows, g.d, device="cuda", generator=gen)
        i2 = torch.randn(rows, g.d, device="cuda", generator=gen)
        o1, o2, r1, r2, d1, d2 = (torch.empty_like(i1) for _ in range(6))
        z = torch.zeros_like(i1)
        eng.rev_forward(blk, i1, i2, o1, o2)
        eng.rev_backward_local(blk, o1, o2, z, z, r1, r2, d1, d2)
        rt = max(float((r1 - i1).abs().max() / i1.abs().max()),
                 float((r2 - i2).abs().max() / i2.abs().max()))
        check("round trip X -> rev_forward -> inverse (rel <= 1e-4)", rt <= 1e-4, rt)
    eng.close()
    for name, ok, v in report:
        print(f"[{'PASS' if ok else 'FAIL'}] {name}: {v:.3e}")
    return 0 if all(ok for _, ok, _ in report) else 1


def cmd_probe(cfg: dict, budget: float) -> int:
    from .engine import activation_bytes, probe_max_batch
    mc = model_config(cfg, 1)
    for name in [e.strip() for e in cfg["bench.engines"].split(",") if e.strip()]:
        b = probe_max_batch(mc, ENGINES[name], int(budget))
        from dataclasses import replace
        peak, _ = activation_bytes(replace(mc, batch=b), ENGINES[name])
        lo, hi = max(1, b // 3), max(1, b // 2)
        print(f"{name}: max batch {b} (peak {peak / 1e9:.2f} GB of {budget / 1e9:.2f} GB); "
              f"recommended PaReprop operating band {lo}-{hi} (33-50%, PAPER.md:144)")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="revprop-b200")
    ap.add_argument("command", choices=["bench", "verify", "probe"])
    ap.add_argument("config", nargs="?")
    ap.add_argument("--seed", type=int)
    ap.add_argument("--out")
    ap.add_argument("--engines")
    ap.add_argument("--batch-sizes")
    ap.add_argument("--budget-bytes", type=float, default=80e9)
    ap.add_argument("--dtype", default="bf16", choices=["bf16"])
    ap.add_argument("--inject-fault", action="store_true",
                    help="verify: corrupt the VJP first (the report must flag it)")
    a = ap.parse_args(argv)
    cfg = read_config(a.config)
    if a.seed is not None:
        cfg["seed"] = str(a.seed)
    if a.out:
        cfg["bench.out"] = a.out
    if a.engines:
        cfg["bench.engines"] = a.engines
    if a.batch_sizes:
        cfg["bench.batch_sizes"] = a.batch_sizes
    if a.command == "bench":
        return cmd_bench(cfg)
    if a.command == "verify":
        return cmd_verify(cfg, a.inject_fault)
    return cmd_probe(cfg, a.budget_bytes)


if __name__ == "__main__":
    sys.exit(main())
