"""Build libhp.so (sm_100a) in-tree with nvcc.

    python -m paper_2005_07068_b200.build [--force]

The library is the C ABI of include/hp.h; the Python binding (hp.py) only loads it.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("kernels.cu", "pso.cu", "api.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in ("common.cuh", "fk.cuh", "pso.cuh",
                                                      "tile.cuh", "eval.cuh", "fit.cuh", "batch.cuh")] + [
    os.path.join(os.path.dirname(HERE), "include", "hp.h")]
LIB = os.path.join(HERE, "libhp.so")
# debug build for the single-GPU loopback test of the sharded paths (include/hp.h
# hp_shard_loopback); never loaded by the product binding unless a test asks for it
LOOPBACK_LIB = os.path.join(HERE, "libhp_loopback.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile SRC into `out`; `defines` (e.g. ["HP_NW=4"]) select tuning variants."""
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
        [f"-D{d}" for d in defines] + ["-o", tmp] + SRC
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


def build_loopback(force: bool = False) -> str:
    return build(force=force, out=LOOPBACK_LIB, defines=["HP_LOOPBACK_TEST=1"])


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv,
                out=outs[0] if outs else LIB, defines=defs))
