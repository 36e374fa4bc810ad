#!/usr/bin/env python
"""Training-throughput benchmark: RevViT-B PaReprop (vs Reprop) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1, one rank per GPU)

Prints ONE JSON line (rank 0). Metric (BASELINE.json): train img/s of PaReprop, with the
same-GPU Reprop number and the PaReprop gain beside it. A step is one full training
iteration of RevViT-B/16 (depth 12, dim 768, 12 heads, 197 tokens, batch 256 per GPU):
embed, 12 reversible blocks forward, head + cross-entropy, backward with activation
recomputation, bucketed gradient allreduce (N > 1) and the SGD update of every parameter.

`value` is device-timed (CUDA events on the engine stream around K graph-replayed steps,
max over ranks) with the batch resident in HBM; `e2e` is the same metric through the
public API with the batch copied from pinned host memory and the loss read back every
step. The per-step working set (~4.5 GB of activations and caches) is far larger than
the 126 MB L2, so no explicit flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PRESET = "revvit-b"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return dict(bf16=d["bf16_tflops"], bf16_sustained=d["bf16_tflops_sustained"],
                    hbm=d["hbm_gbs"], source="measured")
    except Exception:
        return dict(bf16=1590.0, bf16_sustained=1400.0, hbm=6650.0, source="fallback")


def model_flops_per_img(c):
    """model FLOPs/img = 3 (L F_blk + embed + head); HFU adds one more
    block forward for the inverse recompute."""
    N, d, h = c["seq_len"], c["width"], c["hidden"]
    f_blk = 8 * N * d * d + 4 * N * d * h + 4 * N * N * d
    embed = 2 * N * c["in_dim"] * d
    head = 2 * d * c["num_classes"]
    model = 3 * (c["depth"] * f_blk + embed + head)
    executed = model + c["depth"] * f_blk
    return model, executed


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unavailable"]}
        busy = [x for x in sm if x > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- CPU reference
def _ref_cfg(preset, depth=None):
    from oracle import revprop_oracle as O
    from paper_2306_09342_b200.engine import PRESETS
    p = dict(PRESETS[preset])
    return O.ModelConfig(depth or p["depth"], p["width"], p["heads"], p["hidden"], p["seq_len"],
                         768, p.get("num_classes", 1000))


def _ref_runner(mc, images, threads, engine):
    """One training step of the reference's own CPU code (oracle/_ref: ref ops.cpp +
    layers.cpp compiled in place, SPEC engines in ref_shim.cpp) on `images` images, the batch
    split over `threads` shards run concurrently (ref_step_dp); PaReprop runs each shard's
    recompute lane on its own extra thread. Parameters and inputs are seeded
    random (timing is data-independent). Falls back to the numpy port of the
    same algorithm (kind "port", one thread) when oracle/_ref is absent."""
    from oracle import revprop_oracle as O
    rng = np.random.default_rng(0)
    params = (0.02 * rng.standard_normal(O.param_count(mc))).astype(np.float32)
    x = rng.standard_normal((images, mc.seq_len, mc.in_dim)).astype(np.float32)
    lab = rng.integers(0, mc.num_classes, images)
    try:
        from oracle import ref as R
        R.lib()
        return "reference", lambda: R.step_dp(mc, params, x, lab, threads, engine)
    except Exception:
        p64, x64 = params.astype(np.float64), x.astype(np.float64)
        return "port", lambda: O.step(mc, p64, x64, lab, engine)


def cpu_reference_sample(threads: int, steps: int = 1, warmup: int = 0):
    """The reference's CPU path on the benchmarked workload: full depth-12 RevViT-B PaReprop
    training steps (embed, 12 reversible blocks forward, head + CE, the two-lane backward with
    recompute, all parameter grads), each on threads // 2 images -- one image per shard, each
    shard a 2-thread PaReprop pipeline, so every host thread is busy. Warm-up steps run the
    same code on a depth-1 model (the CPU code needs no warm-up beyond loading; this keeps a
    K-step run bounded)."""
    images = max(1, threads // 2)
    mc = _ref_cfg("revvit-b")
    kind, run = _ref_runner(mc, images, images, "pareprop")
    if kind == "port":
        images, threads = 1, 1
    if warmup:
        _, run_w = _ref_runner(_ref_cfg("revvit-b", depth=1), images, images, "pareprop")
        for _ in range(warmup):
            run_w()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    used = 2 * images if kind == "reference" else 1
    return dict(value=images / t, unit="img/s", cores=used, kind=kind,
                sample=(f"full RevViT-B training step (depth 12, PaReprop, fp32) of the "
                        f"{'reference CPU code' if kind == 'reference' else 'numpy port'} on "
                        f"{images} image(s), one 2-lane pipeline per image on {used} host "
                        f"thread(s), {t:.1f} s/step")), ts


def cpu_reference_ti():
    """BASELINE.json configs[0] in the same run: RevViT-Ti (depth 12, d 192) fp32 batch 8 on
    the reference CPU code, Reprop on 1 thread vs PaReprop on 2, one step each."""
    mc = _ref_cfg("revvit-ti")
    out = {"config": "RevViT-Ti fp32 batch 8 (BASELINE configs[0]), reference CPU code"}
    for engine in ("reprop", "pareprop"):
        kind, run = _ref_runner(mc, 8, 1, engine)
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        out[engine] = {"s_per_step": dt, "img_per_s": 8 / dt,
                       "threads": 1 if engine == "reprop" else 2, "kind": kind}
    out["pareprop_gain_pct"] = 100 * (out["reprop"]["s_per_step"] /
                                      out["pareprop"]["s_per_step"] - 1)
    return out


WORKLOAD = ("RevViT-B/16 train step (depth 12, dim 768, 12 heads, 197 tokens, 1000 classes), "
            "PaReprop, SGD")


def workload_config(world, per_gpu, engine="pareprop"):
    """The `config` object both arms print (same workload, batch and geometry)."""
    return {"workload": WORKLOAD, "global_batch": per_gpu * world, "per_gpu_batch": per_gpu,
            "seq_len": 197, "parallelism": f"dp{world}", "engine": engine,
            "l2": "per-step working set ~4.5 GB >> 126 MB L2 (no flush needed)"}


def host_threads():
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    return max(1, min(n, 32))


def main_reference(a, rank):
    if rank != 0:
        return 0
    thr = host_threads()
    base, ts = cpu_reference_sample(thr, steps=a.steps, warmup=a.warmup)
    # the same config object as the GPU arm (same workload, batch, engine); what the CPU
    # actually ran per step is in cpu_baseline.sample
    cfg = workload_config(a.gpus, a.batch or 256)
    line = {
        "impl": "reference", "metric": "train img/s (RevViT-B PaReprop step)",
        "value": base["value"], "unit": "img/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1000.0 * float(np.mean(ts)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": base["value"], "unit": "img/s", "cores": base["cores"],
                         "kind": base["kind"], "sample": base["sample"]},
        "e2e": {"value": base["value"], "unit": "img/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- GPU arm
def main_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2306_09342_b200.engine import (PAREPROP, PRESETS, REPROP, Engine, ModelConfig,
                                              nccl_unique_id)

    torch.cuda.set_device(local_rank)
    p = dict(PRESETS[PRESET])
    if a.batch:
        p["batch"] = a.batch
    # data parallel: every replica starts from the same weights (seed 1234) and draws its
    # own synthetic shard of the batch (seed 1234 + rank)
    cfg = ModelConfig(device=local_rank, seed=1234, r_ctas=a.r_ctas, g_ctas=a.g_ctas, **p)
    eng = Engine(cfg)
    eng.synthetic_batch(1234 + rank)
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.comm_init(obj[0], world, rank)
    eng.set_lr(1e-3)
    stream = torch.cuda.ExternalStream(eng.stream_ptr)
    B = cfg.batch

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(mode, K, sampler=None):
        barrier()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(K):
            eng.step(mode)
        e.record(stream)
        e.synchronize()
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(s.elapsed_time(e))

    # warm-up (first call captures the CUDA graph of each mode)
    for mode in (REPROP, PAREPROP):
        for _ in range(a.warmup):
            eng.step(mode)
    eng.sync()
    ms_r = timed(REPROP, a.steps)
    with ClockSampler(local_rank) as cs:
        ms_p = timed(PAREPROP, a.steps)
    clocks = cs.summary()
    img_p = world * B * a.steps / (ms_p / 1e3)
    img_r = world * B * a.steps / (ms_r / 1e3)
    loss = eng.loss()

    # ---- end to end through the public API: pinned host batch in, loss out, every step
    T = B * cfg.seq_len
    h_in = torch.empty(T * cfg.in_dim, dtype=torch.int16, pin_memory=True)
    h_lab = torch.empty(B, dtype=torch.int32, pin_memory=True)
    rng = np.random.default_rng(rank)
    h_in.numpy()[:] = (rng.standard_normal(T * cfg.in_dim).astype(np.float32).view(np.uint32)
                       >> 16).astype(np.uint16).view(np.int16)
    h_lab.numpy()[:] = rng.integers(0, cfg.num_classes, B)
    h2d = T * cfg.in_dim * 2 + B * 4
    d2h = 4
    h_loss = torch.empty(1, dtype=torch.float32, pin_memory=True)
    # pipelined input: step i's batch is copied (H2D, pinned) while step i-1 computes; every
    # step's loss is read back (D2H) asynchronously; both copies are inside the timed region
    eng.prefetch_batch(h_in.data_ptr(), h_lab.data_ptr())
    for _ in range(2):
        eng.step(PAREPROP)
        eng.prefetch_batch(h_in.data_ptr(), h_lab.data_ptr())
        eng.read_loss_async(h_loss.data_ptr())
    eng.wait_loss()
    eng.sync()
    barrier()
    t0 = time.perf_counter()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(a.steps):
        eng.step(PAREPROP)                                   # consumes the prefetched batch
        eng.prefetch_batch(h_in.data_ptr(), h_lab.data_ptr())  # next step's H2D, overlapped
        eng.read_loss_async(h_loss.data_ptr())               # this step's loss, D2H
    e.record(stream)
    e.synchronize()
    eng.wait_loss()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(max(s.elapsed_time(e), 1e3 * (time.perf_counter() - t0)))
    img_e2e = world * B * a.steps / (e2e_ms / 1e3)

    # ---- live roofline of the dominant kernel (the tcgen05 GEMM), one eager step
    pk = peaks()
    gms, gflops, glaunch = eng.gemm_profile(REPROP)  # kernels serialised: clean durations
    ach = gflops / (gms / 1e3) / 1e12
    # DRAM bytes per GEMM launch: the ncu capture of this build's step committed under
    # profiles/ (tools/gemm_traffic.py; re-captured whenever the kernels change)
    traffic, traffic_src = None, "profiles/round2_gemm_traffic.json"
    try:
        with open(os.path.join(ROOT, traffic_src)) as f:
            traffic = json.load(f)["avg_dram_bytes_per_launch"]
    except Exception:
        traffic_src = "unavailable"
    mf, hf = model_flops_per_img(dict(p, in_dim=cfg.in_dim, num_classes=cfg.num_classes))
    per_gpu = img_p / world
    launches = eng.graph_kernels(PAREPROP)

    # The overlap bound at this batch: PaReprop with its two lanes free-running (no
    # rendezvous; results garbage, timing only, rp_engine_set_diag) -- no schedule of the
    # two lanes can beat it (profiles/round2_pareprop_bound.md sweeps the batch)
    bound = None
    if world == 1 and not a.no_small_batch:
        eng.set_diag(1)
        for _ in range(3):
            eng.step(PAREPROP)
        ms_free = timed(PAREPROP, a.steps)
        eng.set_diag(0)
        bound = {"free_running_lanes_ms_per_step": ms_free / a.steps,
                 "gain_bound_pct": 100.0 * (ms_r / ms_free - 1.0)}
    # PaReprop vs Reprop at small per-GPU batches, where a single stream leaves SMs idle
    # (same kernels, same device-timed protocol)
    small = []
    if world == 1 and not a.no_small_batch:
        eng.close()
        eng = None
        for bs in (8, 32):
            es = Engine(ModelConfig(device=local_rank, seed=1234 + rank, **dict(p, batch=bs)))
            es.set_lr(1e-3)
            for mode in (REPROP, PAREPROP):
                for _ in range(max(a.warmup, 3)):
                    es.step(mode)
            es.sync()
            streams = torch.cuda.ExternalStream(es.stream_ptr)

            def timed_small(mode, K):
                torch.cuda.synchronize()
                s0 = torch.cuda.Event(enable_timing=True)
                e0 = torch.cuda.Event(enable_timing=True)
                s0.record(streams)
                for _ in range(K):
                    es.step(mode)
                e0.record(streams)
                e0.synchronize()
                return s0.elapsed_time(e0)
            k_small = max(a.steps, 20)
            r_ms = min(timed_small(REPROP, k_small) for _ in range(2))
            p_ms = min(timed_small(PAREPROP, k_small) for _ in range(2))
            small.append({"per_gpu_batch": bs, "reprop_img_s": bs * k_small / (r_ms / 1e3),
                          "pareprop_img_s": bs * k_small / (p_ms / 1e3),
                          "gain_pct": 100.0 * (r_ms / p_ms - 1.0)})
            es.close()

    # RevViT-L (BASELINE's metric names RevViT-B/L; configs[2] is L data parallel at
    # 1/2/4/8 GPUs): the same device-timed protocol on the L preset, per-GPU batch 256, at
    # every world size (its own NCCL communicator for N > 1)
    revvit_l = None
    if not a.no_revvit_l:
        if eng is not None:
            eng.close()
            eng = None
        pl_ = dict(PRESETS["revvit-l"])
        el = Engine(ModelConfig(device=local_rank, seed=1234, **pl_))
        el.synthetic_batch(1234 + rank)
        if world > 1:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            el.comm_init(obj[0], world, rank)
        el.set_lr(1e-3)
        sl_ = torch.cuda.ExternalStream(el.stream_ptr)
        for mode in (REPROP, PAREPROP):
            for _ in range(3):
                el.step(mode)
        el.sync()

        def timed_l(mode, K):
            barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            e0 = torch.cuda.Event(enable_timing=True)
            s0.record(sl_)
            for _ in range(K):
                el.step(mode)
            e0.record(sl_)
            e0.synchronize()
            barrier()
            return max_over_ranks(s0.elapsed_time(e0))
        kl = 5
        lr_ms, lp_ms = timed_l(REPROP, kl), timed_l(PAREPROP, kl)
        bl = pl_["batch"]
        mfl, _ = model_flops_per_img(dict(pl_, in_dim=el.cfg.in_dim, num_classes=el.cfg.num_classes))
        img_lp = world * bl * kl / (lp_ms / 1e3)
        revvit_l = {"config": f"RevViT-L (depth 24, dim 1024, 16 heads, 197 tokens), per-GPU batch {bl}, "
                              f"dp{world}, device-timed over {kl} steps",
                    "reprop_img_s": world * bl * kl / (lr_ms / 1e3), "pareprop_img_s": img_lp,
                    "pareprop_gain_pct": 100.0 * (lr_ms / lp_ms - 1.0),
                    "mfu": mfl * img_lp / world / (peaks()["bf16"] * 1e12)}
        el.close()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            cpu, _ = cpu_reference_sample(host_threads(), steps=1, warmup=0)
            cpu["configs0_ti"] = cpu_reference_ti()
        except Exception as ex:  # never let the baseline kill the GPU line
            cpu = {"value": None, "unit": "img/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {ex}"}
    if rank == 0:
        line = {
            "metric": "train img/s (RevViT-B PaReprop step)",
            "value": img_p, "unit": "img/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_p / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": workload_config(world, B),
            "reprop": {"value": img_r, "ms_per_step": ms_r / a.steps},
            "pareprop_gain_pct": 100.0 * (img_p / img_r - 1.0),
            "pareprop_gain_small_batch": small,
            "pareprop_overlap_bound": bound,
            "revvit_l": revvit_l,
            "mfu": mf * per_gpu / (pk["bf16"] * 1e12),
            "hfu": hf * per_gpu / (pk["bf16"] * 1e12),
            "loss": loss,
            "e2e": {"value": img_e2e, "unit": "img/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "tensor", "kernel": "gemm_sm100_kernel (all tcgen05 GEMMs of "
                                                      "one step)",
                         "achieved": ach, "peak": pk["bf16_sustained"], "unit": "TFLOP/s",
                         "frac": ach / pk["bf16_sustained"],
                         "peak_note": f"{pk['source']} sustained bf16 (kernel timed inside a step)",
                         "launches_per_step": glaunch, "traffic": traffic,
                         "traffic_note": "avg dram__bytes_read+write per GEMM launch of one "
                                         "step, ncu, " + traffic_src},
            "gpu_launches": launches * a.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if eng is not None:
        eng.close()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--r-ctas", type=int, default=0)
    ap.add_argument("--g-ctas", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-small-batch", action="store_true")
    ap.add_argument("--no-revvit-l", action="store_true")
    a = ap.parse_args(argv)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: start the N ranks ourselves (one per GPU,
        # torchrun on 127.0.0.1) and return their status; rank 0 prints the line
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)]
        cmd += list(sys.argv[1:] if argv is None else argv)
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return main_reference(a, rank)
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but the launcher started {world} rank(s)")
    if world > 1:
        # deterministic bucket all-reduces (the engine pins the same when unset); must be set
        # before the first NCCL communicator of the process
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return main_ours(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
