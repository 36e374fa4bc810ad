"""CPU checks of the C-ABI boundary: the library loads, exports every entry point that
include/revprop_b200.h declares, and rejects bad shapes/configs with the status codes that
map onto the reference's exception classes (errors.hpp:9-48) -- all before touching a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "revprop_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def capi():
    from paper_2306_09342_b200 import _capi
    if not _capi.lib_path().exists():
        from paper_2306_09342_b200 import build
        build.build()
    _capi.lib()
    return _capi


def test_header_declares_the_boundary():
    names = declared()
    for must in ("rp_gemm", "rp_layer_norm_fwd", "rp_layer_norm_bwd", "rp_attention_fwd",
                 "rp_attention_bwd", "rp_engine_create", "rp_engine_step",
                 "rp_engine_rev_forward", "rp_engine_rev_backward_local", "rp_colsum",
                 "rp_engine_comm_init", "rp_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(capi):
    lib = capi.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_bindings_cover_only_declared_symbols():
    from paper_2306_09342_b200 import _capi, engine
    names = set(declared())
    assert set(_capi.exported_symbols()) <= names
    assert set(engine.exported_symbols()) <= names


def test_gemm_shape_and_contract_errors(capi):
    d = capi.GemmDesc()
    d.A = d.B = 0x1000
    d.lda = d.ldb = d.ldo = 64
    d.M, d.N, d.K = 128, 10, 64  # N not a multiple of 16
    d.epi = capi.RP_EPI_BF16
    d.out = 0x1000
    with pytest.raises(capi.ShapeError):
        capi.check(capi.lib().rp_gemm(C.byref(d), None))
    d.N = 64
    d.M = 0
    with pytest.raises(capi.ShapeError):
        capi.check(capi.lib().rp_gemm(C.byref(d), None))
    d.M, d.K = 128, 1024
    d.splits = 4  # split-K is only defined for the fp32 wgrad epilogue
    with pytest.raises(capi.ContractError):
        capi.check(capi.lib().rp_gemm(C.byref(d), None))


def test_layer_norm_and_attention_argument_errors(capi):
    L = capi.lib()
    with pytest.raises(capi.ShapeError, match="cols"):
        capi.check(L.rp_layer_norm_fwd(None, None, None, 4, 6, 1e-5, None, None, None, None))
    with pytest.raises(capi.ShapeError, match="eps"):
        capi.check(L.rp_layer_norm_fwd(None, None, None, 4, 8, 0.0, None, None, None, None))
    with pytest.raises(capi.ShapeError, match="head_dim"):
        capi.check(L.rp_attention_fwd(None, 2, 8, 2, 32, None, None, None))


def test_engine_config_errors(capi):
    from paper_2306_09342_b200.engine import Engine, ModelConfig
    with pytest.raises(capi.ConfigError):
        Engine(ModelConfig(depth=0))
    with pytest.raises(capi.ConfigError, match="head_dim"):
        Engine(ModelConfig(width=768, heads=8))
