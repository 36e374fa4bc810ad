"""The reference's own layer code (compiled in place) against the B200 path reached through
the reference-typed adapter of INTEGRATION.md §2 (examples/reference_adapter_test.cpp, built in
the container by build() / tests/test_capi.py where the reference's headers exist)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2306_09342_b200", "_lib", "reference_adapter_test")


@pytest.mark.skipif(not os.path.exists(EXE), reason="adapter test binary not built")
def test_reference_adapter_on_b200():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER OK" in r.stdout
