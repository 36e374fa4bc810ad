"""ctypes binding of the C ABI declared in include/revprop_b200.h.

Status codes are mapped back onto the reference's exception hierarchy
(ref:proj/core/include/revprop/errors.hpp:9-48). There is deliberately no fallback:
if the shared library is missing, importing this module's `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("RP_LIB") or
                 Path(__file__).resolve().parent / "_lib" / "librevprop_b200.so")  # RP_LIB: A/B builds


class Error(RuntimeError):
    """Base class (errors.hpp:9-12)."""


class ShapeError(Error):
    """errors.hpp:15-18."""


class ContractError(Error):
    """errors.hpp:21-24."""


class ConfigError(Error):
    """errors.hpp:27-30."""


class BudgetError(Error):
    """errors.hpp:33-36."""


class SchedulerError(Error):
    """errors.hpp:39-42."""


class AccountingError(Error):
    """errors.hpp:45-48."""


class DeviceError(Error):
    """CUDA / driver failure (RP_ERR_CUDA)."""


_CODE_TO_EXC = {1: ShapeError, 2: ContractError, 3: ConfigError, 4: BudgetError,
                5: SchedulerError, 6: AccountingError, 7: DeviceError}

(RP_EPI_BF16, RP_EPI_F32, RP_EPI_BIAS_GELU, RP_EPI_RESID, RP_EPI_GELU_BWD,
 RP_EPI_BIAS_GELU_SLOPE, RP_EPI_MUL, RP_EPI_ROWDOT) = range(8)


class GemmDesc(C.Structure):
    _fields_ = [
        ("A", C.c_void_p), ("lda", C.c_int64), ("a_mn", C.c_int),
        ("B", C.c_void_p), ("ldb", C.c_int64), ("b_mn", C.c_int),
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("epi", C.c_int),
        ("out", C.c_void_p), ("ldo", C.c_int64),
        ("out2", C.c_void_p), ("ldo2", C.c_int64),
        ("aux", C.c_void_p), ("ldaux", C.c_int64),
        ("bias", C.c_void_p), ("sign", C.c_float),
        ("splits", C.c_int), ("workspace", C.c_void_p),
        ("max_ctas", C.c_int), ("bn", C.c_int),
        ("colsum_part", C.c_void_p),
        ("rowdot", C.c_void_p), ("rd_seq", C.c_int64),
        ("quantum", C.c_float),
    ]


_lib = None

# name -> (restype, argtypes)
_P, _I64, _I, _D = C.c_void_p, C.c_int64, C.c_int, C.c_double
_SIGS = {
    "rp_last_error": (C.c_char_p, []),
    "rp_version": (_I, [C.c_char_p, _I]),
    "rp_set_pdl": (_I, [_I]),
    "rp_gemm": (_I, [C.POINTER(GemmDesc), _P]),
    "rp_gemm_plan_create": (_I, [C.POINTER(GemmDesc), C.POINTER(_P)]),
    "rp_gemm_plan_launch": (_I, [_P, _P]),
    "rp_gemm_plan_set_max_ctas": (_I, [_P, _I]),
    "rp_gemm_plan_destroy": (None, [_P]),
    "rp_layer_norm_fwd": (_I, [_P, _P, _P, _I64, _I64, _D, _P, _P, _P, _P]),
    "rp_layer_norm_bwd": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _I, _P]),
    "rp_layer_norm_bwd_ex": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _I,
                                  _P]),
    "rp_set_ln_bwd_impl": (_I, [_I]),
    "rp_layer_norm_bwd_workspace_floats": (_I64, [_I64, _I64]),
    "rp_colsum": (_I, [_P, _I, _I64, _I64, _P, _P, _I, _P]),
    "rp_colsum_workspace_floats": (_I64, [_I64, _I64]),
    "rp_colsum_parts": (_I, [_P, _I64, _I64, _P, _I, _P]),
    "rp_attention_fwd": (_I, [_P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "rp_attention_bwd": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "rp_attention_bwd_ex": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _I, _P]),
    "rp_attention_bwd_workspace_floats": (_I64, [_I64, _I64, _I64]),
    "rp_set_attention_impl": (_I, [_I]),
    "rp_set_attention_fwd_variant": (_I, [_I]),
    "rp_set_attention_window_variant": (_I, [_I]),
    "rp_set_mma_issue": (_I, [_I]),
    "rp_set_gemm_trace": (_I, [_P]),
    "rp_set_attention_trace": (_I, [_P]),
}


def lib_path() -> Path:
    return _LIB_PATH


def lib():
    """Load the sm_100a library (no fallback: raises if it was not built)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: build it with `python -m paper_2306_09342_b200.build`")
        # torch first: its bundled libnccl.so.2 (newer than the system one) must be the one
        # the dynamic loader binds for both torch and this library's ncclAllReduce -- loaded
        # the other way round, torch's CUDA library fails on symbols the older NCCL lacks
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        L = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = lib().rp_last_error().decode(errors="replace")
    raise _CODE_TO_EXC.get(rc, Error)(f"{what}: {msg}" if what else msg)
