"""Build libcacheprune.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRCS = ["cp_index.cu", "cp_match.cu", "cp_gather.cu", "cp_score.cu", "cp_annotate.cu", "cp_policy.cu"]
OUT = os.path.join(HERE, "libcacheprune.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "--extended-lambda"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(HERE, "csrc", s) for s in SRCS] + [os.path.join(HERE, "csrc", "cp_internal.cuh"),
                                                             os.path.join(HERE, "..", "include", "cacheprune.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        cmd = [NVCC] + FLAGS + ["-o", OUT] + [os.path.join(HERE, "csrc", s) for s in SRCS]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    build(force=True, verbose=True)
