"""How much can running the recompute lane beside the gradient lane gain at all?

    python tools/pareprop_bound.py [batches=32,64,128,256] [out=profiles/round2_pareprop_bound]

Per-GPU batch B, RevViT-B, CUDA graphs, device-timed (CUDA events on the engine stream,
K steps after warm-up): Reprop, PaReprop, and three diagnostic schedules whose results are
garbage but whose time bounds the overlap -- PaReprop with the lanes free-running (no
rendezvous at all: lane R never waits for lane G and vice versa, so any concurrency the GPU
can give them it gives), lane R only, lane G only, neither (forward + head + update).
gain bound = Reprop / free-running - 1.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200.engine import PAREPROP, PRESETS, REPROP, Engine, ModelConfig  # noqa: E402


def main():
    batches = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,64,128,256").split(",")]
    out = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    for B in batches:
        p = dict(PRESETS["revvit-b"], batch=B)
        eng = Engine(ModelConfig(**p))
        eng.set_lr(0.0)
        stream = torch.cuda.ExternalStream(eng.stream_ptr)
        K = max(5, 2560 // B)

        def timed(mode, diag):
            eng.set_diag(diag)
            for _ in range(3):
                eng.step(mode)
            eng.sync()
            best = 1e30
            for _ in range(3):
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record(stream)
                for _ in range(K):
                    eng.step(mode)
                e.record(stream)
                e.synchronize()
                best = min(best, s.elapsed_time(e) / K)
            return best
        r = {"batch": B,
             "reprop_ms": timed(REPROP, 0), "pareprop_ms": timed(PAREPROP, 0),
             "free_lanes_ms": timed(PAREPROP, 1), "lane_r_only_ms": timed(PAREPROP, 2),
             "lane_g_only_ms": timed(PAREPROP, 4), "no_backward_ms": timed(PAREPROP, 6)}
        eng.set_diag(0)
        eng.close()
        r["pareprop_gain_pct"] = 100 * (r["reprop_ms"] / r["pareprop_ms"] - 1)
        r["gain_bound_pct"] = 100 * (r["reprop_ms"] / r["free_lanes_ms"] - 1)
        bw = r["reprop_ms"] - r["no_backward_ms"]
        r["backward_ms"] = bw
        r["lane_r_ms"] = r["lane_r_only_ms"] - r["no_backward_ms"]
        r["lane_g_ms"] = r["lane_g_only_ms"] - r["no_backward_ms"]
        rows.append(r)
        print(json.dumps(r), flush=True)
    if out:
        with open(out + ".json", "w") as f:
            json.dump(rows, f, indent=1)
        with open(out + ".md", "w") as f:
            f.write("# PaReprop overlap bound (RevViT-B, CUDA graphs, device-timed; tools/pareprop_bound.py)\n\n")
            f.write("| per-GPU batch | Reprop ms | PaReprop ms | gain | free-running lanes ms | gain bound | "
                    "backward ms (lane R + lane G) | lane R ms | lane G ms |\n|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['batch']} | {r['reprop_ms']:.2f} | {r['pareprop_ms']:.2f} | "
                        f"{r['pareprop_gain_pct']:+.1f}% | {r['free_lanes_ms']:.2f} | "
                        f"{r['gain_bound_pct']:+.1f}% | {r['backward_ms']:.2f} | {r['lane_r_ms']:.2f} | "
                        f"{r['lane_g_ms']:.2f} |\n")


if __name__ == "__main__":
    main()
