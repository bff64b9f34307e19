"""Build liblcma.so in-tree with nvcc for sm_100a (no GPU needed to compile)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblcma.so")
SOURCES = ["lcma_api.cu", "schemes.cpp", "decision.cpp"]
HEADERS = ["ptx.cuh", "umma_gemm.cuh", "combine.cuh", "schemes.h", "decision.h", "diag.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "lcma.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = LIB) -> str:
    if out == LIB and not force and not _stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-cudart", "static", "-I", os.path.join(HERE, "..", "include"),
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", tmp] + os.environ.get("LCMA_NVCC_FLAGS", "").split() + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


DIAG_LIB = os.path.join(HERE, "liblcma_diag.so")


def build_diag(force: bool = False) -> str:
    """The -DLCMA_DIAG build (tuning / diagnostic environment knobs, see
    csrc/diag.h): used by tests/_diag_homes.py and tools/, never by the
    product path."""
    if not force and os.path.exists(DIAG_LIB) and os.path.exists(LIB) and \
            os.path.getmtime(DIAG_LIB) >= os.path.getmtime(LIB) and not _stale():
        return DIAG_LIB
    old = os.environ.get("LCMA_NVCC_FLAGS", "")
    os.environ["LCMA_NVCC_FLAGS"] = (old + " -DLCMA_DIAG").strip()
    try:
        return build(force=True, out=DIAG_LIB)
    finally:
        os.environ["LCMA_NVCC_FLAGS"] = old


if __name__ == "__main__":
    # --out PATH: build a variant (e.g. with LCMA_NVCC_FLAGS) beside the
    # in-tree library, loaded with LCMA_LIB=PATH for tuning experiments
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else LIB
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out))
