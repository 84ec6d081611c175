"""Build libcacheprune.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

Provenance: the SHA-256 of every source the library is compiled from (csrc/*.cu, csrc/*.cuh,
include/cacheprune.h) and the flags is compiled into it (`cp_build_info()`); the library is rebuilt
whenever that hash differs from the current sources' (not on file times, which a copy to another box
does not preserve), and `_lib.lib()` refuses a library built from other sources."""
from __future__ import annotations

import hashlib
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRCS = ["cp_index.cu", "cp_match.cu", "cp_gather.cu", "cp_score.cu", "cp_annotate.cu", "cp_policy.cu"]
DEPS = SRCS + ["cp_internal.cuh"]
HEADER = os.path.join(HERE, "..", "include", "cacheprune.h")
OUT = os.path.join(HERE, "libcacheprune.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "--extended-lambda"]


def source_hash() -> str:
    """SHA-256 over the flags and the bytes of every source file, in a fixed order."""
    h = hashlib.sha256(" ".join(FLAGS).encode())
    for p in [os.path.join(HERE, "csrc", s) for s in DEPS] + [HEADER]:
        with open(p, "rb") as f:
            h.update(os.path.basename(p).encode() + b"\0" + f.read())
    return h.hexdigest()


def built_hash(path: str = OUT) -> str:
    """The source hash compiled into a built library ('' if absent or unreadable).  Reads the
    embedded string without loading the library (no CUDA context needed)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        return ""
    i = data.find(b"cp-src-sha256=")
    return data[i + 14:i + 78].decode() if i >= 0 else ""


def build(force: bool = False, verbose: bool = False) -> str:
    want = source_hash()
    if force or built_hash() != want:
        cmd = [NVCC] + FLAGS + [f"-DCP_SRC_SHA256=\"{want}\"", "-o", OUT] + [os.path.join(HERE, "csrc", s) for s in SRCS]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        if built_hash() != want:
            raise RuntimeError("libcacheprune.so does not carry the source hash it was built with")
    return OUT


if __name__ == "__main__":
    build(force=True, verbose=True)
