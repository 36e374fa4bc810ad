"""Python front end of the C++ training engine (include/revprop_b200.h, csrc/engine.cpp).

Mirrors the reference's engines module: `step_reprop`, `step_pareprop`,
`sgd_update`, on the isotropic reversible model of SPEC.md:270-335. All arithmetic runs in
the sm_100a library; this module only moves host arrays and calls the C ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, lib

REPROP, PAREPROP = 1, 2


class ModelConfigC(C.Structure):
    _fields_ = [("depth", C.c_int64), ("width", C.c_int64), ("heads", C.c_int64),
                ("hidden", C.c_int64), ("seq_len", C.c_int64), ("in_dim", C.c_int64),
                ("num_classes", C.c_int64), ("batch", C.c_int64), ("window", C.c_int64),
                ("seed", C.c_uint64), ("device", C.c_int), ("r_ctas", C.c_int),
                ("g_ctas", C.c_int), ("lane_priority", C.c_int), ("optimizer", C.c_int),
                ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
                ("weight_decay", C.c_float), ("stages", C.c_int64),
                ("stage_depth", C.c_int64 * 8), ("stage_width", C.c_int64 * 8),
                ("stage_heads", C.c_int64 * 8), ("reduction", C.c_int64), ("fusion", C.c_int),
                ("comm_ctas", C.c_int), ("exact_coupling_bits", C.c_int)]


@dataclass
class ModelConfig:
    """SPEC.md:275-278 (isotropic) plus the per-GPU batch."""
    depth: int = 12
    width: int = 768
    heads: int = 12
    hidden: int = 3072
    seq_len: int = 197
    in_dim: int = 768
    num_classes: int = 1000
    batch: int = 256
    window: int = 0
    seed: int = 0
    device: int = 0
    r_ctas: int = 0
    g_ctas: int = 0
    lane_priority: int = 1
    optimizer: int = 0          # 0 SGD, 1 AdamW
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    weight_decay: float = 0.0
    # hierarchical (Rev-Swin-style): blocks / width / heads per stage,
    # tokens merged per boundary group, fusion kind ("average" | "mlp", layers.hpp:142)
    depths: tuple | None = None
    widths: tuple | None = None
    stage_heads: tuple | None = None
    reduction: int = 2
    fusion: str = "average"
    comm_ctas: int = 0          # NCCL CTAs per all-reduce (0 = 4), SMs reserved for them
    exact_coupling_bits: int = 0  # residual grid 2^-bits for bit-exact inverses (0 = 17, -1 off)

    def __post_init__(self):
        if self.depths:
            self.depth = int(sum(self.depths))
            self.width, self.heads = int(self.widths[0]), int(self.stage_heads[0])


PRESETS = {
    # BASELINE.json configs
    "revvit-ti": dict(depth=12, width=192, heads=3, hidden=768, seq_len=197, batch=8),
    "revvit-b": dict(depth=12, width=768, heads=12, hidden=3072, seq_len=197, batch=256),
    "revvit-l": dict(depth=24, width=1024, heads=16, hidden=4096, seq_len=197, batch=256),
    "rev-roberta-base": dict(depth=12, width=768, heads=12, hidden=3072, seq_len=512,
                             batch=64, num_classes=2),
    # BASELINE config 5: RevViT-G-style (depth 48, dim 1664, 16 heads of 104, MLP ratio 4)
    "revvit-g48": dict(depth=48, width=1664, heads=16, hidden=6656, seq_len=197, batch=64),
    # hierarchical Rev-Swin-B (Swin-B stages: C = 128, depths 2-2-18-2,
    # heads 4-8-16-32, 7x7 windows over 56x56 tokens of 4x4x3 patches, 2x2 merges as r = 4
    # adjacent tokens, ref ops.cpp:393-399), average fusion
    "rev-swin-b": dict(depth=24, width=128, heads=4, hidden=512, seq_len=3136, in_dim=48,
                       window=49, depths=(2, 2, 18, 2), widths=(128, 256, 512, 1024),
                       stage_heads=(4, 8, 16, 32), reduction=4, batch=128),
}


def _fn(name, restype, argtypes):
    f = getattr(lib(), name)
    f.restype, f.argtypes = restype, argtypes
    return f


_P, _I64, _I = C.c_void_p, C.c_int64, C.c_int
_API = {
    "rp_engine_create": (_I, [C.POINTER(ModelConfigC), C.POINTER(_P)]),
    "rp_activation_bytes": (_I, [C.POINTER(ModelConfigC), _I, C.POINTER(_I64), C.POINTER(_I64)]),
    "rp_engine_destroy": (None, [_P]),
    "rp_engine_param_count": (_I64, [_P]),
    "rp_engine_tensor_table": (_I, [_P, _P, _P, _I64]),
    "rp_engine_init_params": (_I, [_P, C.c_uint64]),
    "rp_engine_synthetic_batch": (_I, [_P, C.c_uint64]),
    "rp_engine_set_params": (_I, [_P, _P]),
    "rp_engine_get_params": (_I, [_P, _P]),
    "rp_engine_get_grads": (_I, [_P, _P]),
    "rp_engine_set_batch": (_I, [_P, _P, _P]),
    "rp_engine_prefetch_batch": (_I, [_P, _P, _P]),
    "rp_engine_read_loss_async": (_I, [_P, _P]),
    "rp_engine_wait_loss": (_I, [_P]),
    "rp_engine_set_batch_device": (_I, [_P, _P, _P]),
    "rp_engine_set_lr": (_I, [_P, C.c_float]),
    "rp_engine_set_partition": (_I, [_P, _I, _I]),
    "rp_engine_invalidate_graphs": (_I, [_P]),
    "rp_engine_inject_fault": (_I, [_P, _I]),
    "rp_engine_enable_vanilla": (_I, [_P]),
    "rp_engine_step": (_I, [_P, _I, _I]),
    "rp_engine_sync": (_I, [_P]),
    "rp_engine_read_loss": (_I, [_P, C.POINTER(C.c_float)]),
    "rp_engine_stream": (_P, [_P]),
    "rp_engine_graph_kernels": (_I64, [_P, _I]),
    "rp_engine_gemm_profile": (_I, [_P, _I, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(_I64)]),
    "rp_engine_set_instrument": (_I, [_P, _I]),
    "rp_engine_slot_log": (_I, [_P, _P]),
    "rp_nccl_unique_id": (_I, [_P]),
    "rp_engine_comm_init": (_I, [_P, _P, _I, _I]),
    "rp_engine_rev_forward": (_I, [_P, _I64, _P, _P, _P, _P]),
    "rp_engine_rev_backward_local": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "rp_engine_rev_inverse": (_I, [_P, _I64, _P, _P, _P, _P]),
    "rp_engine_attention_forward": (_I, [_P, _I64, _P, _P]),
    "rp_engine_mlp_forward": (_I, [_P, _I64, _P, _P]),
    "rp_engine_attention_vjp": (_I, [_P, _I64, _P, _P, _P]),
    "rp_engine_mlp_vjp": (_I, [_P, _I64, _P, _P, _P]),
    "rp_engine_boundary_forward": (_I, [_P, _I64, _P, _P, _P]),
    "rp_engine_boundary_vjp": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P]),
    "rp_engine_step_stats": (_I, [_P, _P]),
    "rp_engine_set_caller_stream": (_I, [_P, _P]),
    "rp_engine_trace_floats": (_I64, [_P]),
    "rp_engine_set_trace": (_I, [_P, _P, _P]),
    "rp_model_bucket_plan": (_I, [C.POINTER(ModelConfigC), _P, _P, _P, _I64]),
    "rp_engine_set_diag": (_I, [_P, _I]),
}


class StepStatsC(C.Structure):
    _fields_ = [("loss", C.c_float), ("mode", C.c_int), ("wall_ns", C.c_int64),
                ("peak_activation_bytes", C.c_int64), ("lane_busy_ns", C.c_int64 * 2),
                ("blocks_processed", C.c_int64), ("ledger_events", C.c_int64),
                ("arena_activation_bytes", C.c_int64), ("arena_param_bytes", C.c_int64),
                ("arena_total_bytes", C.c_int64)]


@dataclass
class StepStats:
    """SPEC.md:350-353 (plus the ledger event count and the arena's real allocations)."""
    loss: float
    mode: int
    wall_ns: int
    peak_activation_bytes: int
    lane_busy_ns: tuple
    blocks_processed: int
    ledger_events: int
    arena_activation_bytes: int
    arena_param_bytes: int
    arena_total_bytes: int
_bound = {}


def api(name):
    if name not in _bound:
        r, a = _API[name]
        _bound[name] = _fn(name, r, a)
    return _bound[name]


def exported_symbols():
    return list(_API)


def _np_ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + 0x7FFF
    return ((u + r) >> 16).astype(np.uint16)


def bf16_round(x: np.ndarray) -> np.ndarray:
    return (bf16_bits(x).astype(np.uint32) << 16).view(np.float32)


class Engine:
    """One GPU's training engine. `step(mode)` runs forward + backward + (allreduce) + SGD."""

    def __init__(self, cfg: ModelConfig):
        self.cfg = cfg
        c = _cfg_c(cfg)
        h = C.c_void_p()
        check(api("rp_engine_create")(C.byref(c), C.byref(h)), "engine_create")
        self._h = h
        self.n_params = api("rp_engine_param_count")(h)

    def close(self):
        if getattr(self, "_h", None):
            api("rp_engine_destroy")(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def tensor_table(self):
        cap = 1 + 10 * self.cfg.depth + 2 * len(self.cfg.depths or ()) + 1
        off = np.zeros(cap, np.int64)
        num = np.zeros(cap, np.int64)
        n = api("rp_engine_tensor_table")(self._h, _np_ptr(off), _np_ptr(num), cap)
        if n < 0:
            check(n)
        return off[:n], num[:n]

    def set_params(self, flat: np.ndarray):
        a = np.ascontiguousarray(flat, dtype=np.float32)
        assert a.size == self.n_params
        check(api("rp_engine_set_params")(self._h, _np_ptr(a)), "set_params")

    def params(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float32)
        check(api("rp_engine_get_params")(self._h, _np_ptr(out)), "get_params")
        return out

    def grads(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float32)
        check(api("rp_engine_get_grads")(self._h, _np_ptr(out)), "get_grads")
        return out

    def set_batch(self, inputs_bf16: np.ndarray, labels: np.ndarray):
        x = np.ascontiguousarray(inputs_bf16, dtype=np.uint16)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        check(api("rp_engine_set_batch")(self._h, _np_ptr(x), _np_ptr(y)), "set_batch")
        self.sync()  # host buffers may be freed by the caller afterwards

    def set_batch_ptr(self, inputs_ptr: int, labels_ptr: int):
        """Async H2D from caller-owned (pinned) host memory."""
        check(api("rp_engine_set_batch")(self._h, C.c_void_p(inputs_ptr), C.c_void_p(labels_ptr)),
              "set_batch")

    def prefetch_batch(self, inputs_ptr: int, labels_ptr: int):
        """Start the host -> device copy of the next step's batch (pinned host pointers);
        it overlaps the current step and is consumed by the next step()."""
        check(api("rp_engine_prefetch_batch")(self._h, C.c_void_p(inputs_ptr),
                                                C.c_void_p(labels_ptr)), "prefetch_batch")

    def read_loss_async(self, loss_ptr: int):
        """Device -> host copy of the last enqueued step's loss into pinned memory."""
        check(api("rp_engine_read_loss_async")(self._h, C.c_void_p(loss_ptr)), "read_loss_async")

    def wait_loss(self):
        check(api("rp_engine_wait_loss")(self._h), "wait_loss")

    def set_batch_device(self, inputs_ptr: int, labels_ptr: int):
        check(api("rp_engine_set_batch_device")(self._h, C.c_void_p(inputs_ptr),
                                                C.c_void_p(labels_ptr)), "set_batch_device")

    def synthetic_batch(self, seed: int):
        check(api("rp_engine_synthetic_batch")(self._h, seed), "synthetic_batch")

    def set_lr(self, lr: float):
        check(api("rp_engine_set_lr")(self._h, lr), "set_lr")

    def set_partition(self, r_ctas: int, g_ctas: int):
        check(api("rp_engine_set_partition")(self._h, r_ctas, g_ctas), "set_partition")

    def enable_vanilla(self):
        """Allocate the store-everything stash so step(VANILLA) works."""
        check(api("rp_engine_enable_vanilla")(self._h), "enable_vanilla")

    def inject_fault(self, kind: int = 1):
        """Verify's fault-injection hook: 1 corrupts the F-path VJP, 0 heals."""
        check(api("rp_engine_inject_fault")(self._h, kind), "inject_fault")

    def invalidate_graphs(self):
        check(api("rp_engine_invalidate_graphs")(self._h), "invalidate_graphs")

    def step(self, mode=REPROP, graph=True):
        check(api("rp_engine_step")(self._h, mode, int(graph)), "step")

    def step_stats(self) -> "StepStats":
        """StepStats of the last step (waits for it)."""
        st = StepStatsC()
        check(api("rp_engine_step_stats")(self._h, C.byref(st)), "step_stats")
        return StepStats(st.loss, st.mode, st.wall_ns, st.peak_activation_bytes,
                         tuple(st.lane_busy_ns), st.blocks_processed, st.ledger_events,
                         st.arena_activation_bytes, st.arena_param_bytes, st.arena_total_bytes)

    def set_caller_stream(self, stream_ptr: int):
        """Stream whose prior work the block / layer entry points wait for (default: the
        legacy default stream)."""
        check(api("rp_engine_set_caller_stream")(self._h, C.c_void_p(stream_ptr)),
              "set_caller_stream")

    def trace_floats(self) -> int:
        return int(api("rp_engine_trace_floats")(self._h))

    def set_trace(self, fwd_ptr: int, rec_ptr: int):
        """Recompute trace buffers (device pointers, trace_floats() floats each; 0 = off)."""
        check(api("rp_engine_set_trace")(self._h, C.c_void_p(fwd_ptr or None),
                                         C.c_void_p(rec_ptr or None)), "set_trace")

    def set_diag(self, flags: int):
        """Timing experiments only (results are garbage while set): 1 free-running PaReprop
        lanes, 2 skip lane G, 4 skip lane R; 0 = the real schedule."""
        check(api("rp_engine_set_diag")(self._h, flags), "set_diag")

    def sync(self):
        check(api("rp_engine_sync")(self._h), "sync")

    def loss(self) -> float:
        v = C.c_float()
        check(api("rp_engine_read_loss")(self._h, C.byref(v)), "read_loss")
        return v.value

    @property
    def stream_ptr(self) -> int:
        return api("rp_engine_stream")(self._h)

    def graph_kernels(self, mode) -> int:
        return int(api("rp_engine_graph_kernels")(self._h, mode))

    def gemm_profile(self, mode):
        """(ms, flops, launches) of every tcgen05 GEMM in one eager step."""
        ms, fl, n = C.c_double(), C.c_double(), C.c_int64()
        check(api("rp_engine_gemm_profile")(self._h, mode, C.byref(ms), C.byref(fl), C.byref(n)),
              "gemm_profile")
        return ms.value, fl.value, n.value

    def set_instrument(self, on: bool):
        check(api("rp_engine_set_instrument")(self._h, int(on)), "instrument")

    def slot_log(self) -> np.ndarray:
        out = np.zeros((2, self.cfg.depth, 2), np.float32)
        check(api("rp_engine_slot_log")(self._h, _np_ptr(out)), "slot_log")
        return out

    def comm_init(self, uid: bytes, world: int, rank: int):
        """Join the data-parallel group (rp_engine_comm_init). The NCCL algorithm / protocol
        are pinned for a deterministic reduction order unless already set."""
        import os
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(api("rp_engine_comm_init")(self._h, buf, world, rank), "comm_init")

    # revcore on caller-owned device pointers (torch tensors)
    def rev_forward(self, b, i1, i2, o1, o2):
        check(api("rp_engine_rev_forward")(self._h, b, i1.data_ptr(), i2.data_ptr(),
                                           o1.data_ptr(), o2.data_ptr()), "rev_forward")

    # layers API (ref layers.hpp:82-138) on block b's parameters, device tensors
    def attention_forward(self, b, x, y):
        check(api("rp_engine_attention_forward")(self._h, b, x.data_ptr(), y.data_ptr()),
              "attention_forward")

    def mlp_forward(self, b, x, y):
        check(api("rp_engine_mlp_forward")(self._h, b, x.data_ptr(), y.data_ptr()), "mlp_forward")

    def attention_vjp(self, b, x, d_y, d_x):
        check(api("rp_engine_attention_vjp")(self._h, b, x.data_ptr(), d_y.data_ptr(),
                                             d_x.data_ptr()), "attention_vjp")

    def mlp_vjp(self, b, x, d_y, d_x):
        check(api("rp_engine_mlp_vjp")(self._h, b, x.data_ptr(), d_y.data_ptr(), d_x.data_ptr()),
              "mlp_vjp")

    def rev_inverse(self, b, o1, o2, i1, i2):
        """SPEC.md:222-230 on device tensors (block b not first in its stage)."""
        check(api("rp_engine_rev_inverse")(self._h, b, o1.data_ptr(), o2.data_ptr(),
                                           i1.data_ptr(), i2.data_ptr()), "rev_inverse")

    def boundary_forward(self, stage, o1, o2, y):
        """patch_merge(fuse(o1, o2)) after `stage` (layers.cpp:261-287)."""
        check(api("rp_engine_boundary_forward")(self._h, stage, o1.data_ptr(), o2.data_ptr(),
                                                y.data_ptr()), "boundary_forward")

    def boundary_vjp(self, stage, o1, o2, d_i1, d_i2, d_o1, d_o2):
        """fuse_vjp(patch_merge_vjp(d_i1 + d_i2)) (layers.cpp:269-303); param grads in grads()."""
        check(api("rp_engine_boundary_vjp")(self._h, stage, o1.data_ptr(), o2.data_ptr(),
                                            d_i1.data_ptr(), d_i2.data_ptr(), d_o1.data_ptr(),
                                            d_o2.data_ptr()), "boundary_vjp")

    def rev_backward_local(self, b, o1, o2, d_o1, d_o2, i1, i2, d_i1, d_i2):
        check(api("rp_engine_rev_backward_local")(
            self._h, b, o1.data_ptr(), o2.data_ptr(), d_o1.data_ptr(), d_o2.data_ptr(),
            i1.data_ptr(), i2.data_ptr(), d_i1.data_ptr(), d_i2.data_ptr()), "rev_backward_local")


def _cfg_c(cfg: "ModelConfig") -> ModelConfigC:
    c = ModelConfigC(cfg.depth, cfg.width, cfg.heads, cfg.hidden, cfg.seq_len, cfg.in_dim,
                     cfg.num_classes, cfg.batch, cfg.window, cfg.seed, cfg.device, cfg.r_ctas,
                     cfg.g_ctas, cfg.lane_priority, cfg.optimizer, cfg.beta1, cfg.beta2,
                     cfg.adam_eps, cfg.weight_decay)
    c.comm_ctas = cfg.comm_ctas
    c.exact_coupling_bits = cfg.exact_coupling_bits
    if cfg.depths:
        if not (len(cfg.depths) == len(cfg.widths) == len(cfg.stage_heads) <= 8):
            raise _capi.ConfigError("depths / widths / stage_heads: same length, at most 8")
        c.stages = len(cfg.depths)
        for s, (L, d, H) in enumerate(zip(cfg.depths, cfg.widths, cfg.stage_heads)):
            c.stage_depth[s], c.stage_width[s], c.stage_heads[s] = L, d, H
        c.reduction = cfg.reduction
        if cfg.fusion not in ("average", "mlp"):
            raise _capi.ConfigError("fusion must be 'average' or 'mlp'")
        c.fusion = 1 if cfg.fusion == "mlp" else 0
    return c


VANILLA = 0


def activation_bytes(cfg: "ModelConfig", mode: int):
    """(peak activation bytes, block footprint) the ledger predicts for an engine mode."""
    peak, blk = C.c_int64(), C.c_int64()
    c = _cfg_c(cfg)
    check(api("rp_activation_bytes")(C.byref(c), mode, C.byref(peak), C.byref(blk)),
          "activation_bytes")
    return peak.value, blk.value


def probe_max_batch(cfg: "ModelConfig", mode: int, budget_bytes: int) -> int:
    """doubling search over batch against the ledger-predicted peak;
    returns the largest feasible power of two (BudgetError if batch 1 does not fit)."""
    from dataclasses import replace
    b = 1
    if activation_bytes(replace(cfg, batch=1), mode)[0] > budget_bytes:
        raise _capi.BudgetError("batch 1 exceeds the byte budget")
    while activation_bytes(replace(cfg, batch=2 * b), mode)[0] <= budget_bytes:
        b *= 2
    return b


def bucket_plan(cfg: "ModelConfig"):
    """The engine's data-parallel gradient buckets in all-reduce order:
    [(offset, size, kind)] with kind 'embed' | 'block' | 'boundary' | 'head'."""
    cap = cfg.depth + 16
    off = np.zeros(cap, np.int64)
    n = np.zeros(cap, np.int64)
    k = np.zeros(cap, np.int32)
    c = _cfg_c(cfg)
    cnt = api("rp_model_bucket_plan")(C.byref(c), _np_ptr(off), _np_ptr(n), _np_ptr(k), cap)
    if cnt < 0:
        check(-cnt, "bucket_plan")
    names = ("embed", "block", "boundary", "head")
    return [(int(off[i]), int(n[i]), names[k[i]]) for i in range(cnt)]


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(api("rp_nccl_unique_id")(buf), "nccl_unique_id")
    return bytes(buf)


def step_reprop(engine: Engine, graph=True):
    """SPEC.md:369-377."""
    engine.step(REPROP, graph)


def step_pareprop(engine: Engine, graph=True):
    """SPEC.md:378-386."""
    engine.step(PAREPROP, graph)
