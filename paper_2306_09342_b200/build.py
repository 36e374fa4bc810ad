"""Build the sm_100a shared library in-tree.

    python -m paper_2306_09342_b200.build            # incremental
    python -m paper_2306_09342_b200.build --clean

Every .cu/.cpp under csrc/ is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (objects under build/),
then linked into ``paper_2306_09342_b200/_lib/librevprop_b200.so``. The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "librevprop_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + str(ROOT / "include"),
          "-I" + str(CSRC)]
NVFLAGS = ARCH + COMMON + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
LINK_LIBS = ["-lnccl", "-lpthread"]


def _sources() -> list[Path]:
    return sorted(p for p in CSRC.iterdir() if p.suffix in (".cu", ".cpp"))


def _headers() -> list[Path]:
    hs = [p for p in CSRC.iterdir() if p.suffix in (".h", ".cuh", ".hpp")]
    hs += list((ROOT / "include").glob("*.h"))
    return hs


def _obj_for(src: Path) -> Path:
    return OBJ / (src.name + ".o")


def _stale(src: Path, obj: Path, newest_header: float) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or newest_header > t


def _compile(src: Path, verbose: bool) -> tuple[Path, str]:
    obj = _obj_for(src)
    cmd = [NVCC] + NVFLAGS + ["-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [NVCC] + ARCH + COMMON + ["-x", "cu", "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    log = r.stdout + r.stderr
    if verbose:
        print(log)
    return obj, log


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    newest_header = max((h.stat().st_mtime for h in _headers()), default=0.0)
    todo = [s for s in srcs if _stale(s, _obj_for(s), newest_header)]
    logs = {}
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
            for obj, log in ex.map(lambda s: _compile(s, verbose), todo):
                logs[obj.name] = log
        (ROOT / "build" / "ptxas.log").write_text(
            "\n".join(f"== {k}\n{v}" for k, v in sorted(logs.items())))
    objs = [_obj_for(s) for s in srcs]
    if todo or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + LINK_LIBS
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


REFERENCE_INCLUDE = Path("/root/reference/proj/core/include")
ADAPTER_TEST = LIB_DIR / "reference_adapter_test"
ORACLE_REF = ROOT / "oracle" / "_ref"


def build_adapter_test(verbose: bool = False) -> Path | None:
    """Compile examples/reference_adapter_test.cpp: the reference-typed adapter
    (examples/reference_adapter.hpp over include/revprop_b200.hpp) against the reference's own
    headers, linked with the reference's layer code compiled in place (oracle/_ref/{ops,layers}.o)
    and librevprop_b200.so. Only where /root/reference exists (this container); the binary
    travels to the GPU box in-tree (git-ignored), where tests/test_gpu_adapter.py runs it."""
    objs = [ORACLE_REF / "ops.o", ORACLE_REF / "layers.o"]
    if not REFERENCE_INCLUDE.exists() or not all(o.exists() for o in objs):
        return None
    srcs = [ROOT / "examples" / "reference_adapter_test.cpp", ROOT / "examples" / "reference_adapter.hpp",
            ROOT / "include" / "revprop_b200.hpp", ROOT / "include" / "revprop_b200.h", LIB]
    if ADAPTER_TEST.exists() and all(ADAPTER_TEST.stat().st_mtime >= s.stat().st_mtime for s in srcs):
        return ADAPTER_TEST
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-include", "algorithm",
           "-I" + str(REFERENCE_INCLUDE), "-I" + str(ROOT / "include"),
           "-I/usr/local/cuda/include", str(srcs[0])] + [str(o) for o in objs] + [
           "-L" + str(LIB_DIR), "-lrevprop_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,$ORIGIN", "-pthread", "-o", str(ADAPTER_TEST)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"adapter test build failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stdout + r.stderr)
    return ADAPTER_TEST


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    if a.clean:
        shutil.rmtree(ROOT / "build", ignore_errors=True)
        if LIB.exists():
            LIB.unlink()
    lib = build(verbose=a.verbose)
    print(lib)
    return 0


if __name__ == "__main__":
    sys.exit(main())
