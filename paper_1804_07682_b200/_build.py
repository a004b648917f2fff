"""Build libgna_b200.so in-tree with nvcc for sm_100a (no torch, no JIT cache)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgna_b200.so")
HEADER = os.path.join(ROOT, "include", "gna_b200.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "-cudart", "static",  # torch ships a cu128 runtime; keep ours private
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h")) + [HEADER])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: dict | None = None) -> str:
    """Compile csrc/gna_b200.cu; `out`/`defines` build tuning variants (tools/variants.py)."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    tmp = target + ".tmp.%d" % os.getpid()
    dflags = ["-D%s=%s" % kv for kv in (defines or {}).items()]
    cmd = [nvcc(), *NVCC_FLAGS, *dflags, *(["-Xptxas", "-v"] if verbose else []), "-o", tmp,
           os.path.join(CSRC, "gna_b200.cu")]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


PROBE_SRC = os.path.join(ROOT, "tools", "probe_fp64.cu")
PROBE_BIN = os.path.join(ROOT, "build", "probe_fp64")


def build_probe() -> str:
    """FP64-pipe microbenchmark executable (measurement tooling, not the product)."""
    os.makedirs(os.path.dirname(PROBE_BIN), exist_ok=True)
    if not os.path.exists(PROBE_BIN) or os.path.getmtime(PROBE_BIN) < os.path.getmtime(PROBE_SRC):
        subprocess.check_call([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-o", PROBE_BIN, PROBE_SRC])
    return PROBE_BIN


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
