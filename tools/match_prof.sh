#!/bin/bash
# Diagnostic build of the library with the matcher phase profiler (-DCP_MATCH_PROF), then config 2's
# 256-request match timed phase by phase (GPU box only).  Not the hashed build: CP_DIAGNOSTIC_BUILD=1.
set -e
cd "$(dirname "$0")/.."
H=paper_2605_23640_b200
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr --extended-lambda -DCP_MATCH_PROF -o $H/libcacheprune.so $H/csrc/cp_index.cu $H/csrc/cp_match.cu \
  $H/csrc/cp_gather.cu $H/csrc/cp_score.cu $H/csrc/cp_annotate.cu $H/csrc/cp_policy.cu
CP_DIAGNOSTIC_BUILD=1 python - <<'PY'
import ctypes as C, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2605_23640_b200 as cp
from paper_2605_23640_b200 import _lib as L
sys.argv = ["bench.py", "--by", "layer"]; args = bench.parse()
S = bench.setup_ours(args, 0, 1, torch.device("cuda", 0))
f = L.lib().cp_match_prof_read; f.argtypes = [C.c_void_p]; f.restype = C.c_int
base = (C.c_ulonglong * 8)(); f(base)
n = 20
for k in range(n):
    S.idx.match_spans(S.rdb, 1000 + k, hits=S.hits, no_touch=True)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 8)(); f(buf)
names = ["tokens + prefix hashes", "windows -> filter -> full-hash check", "verification", "session + greedy + hits + plan", "last-CTA ticket"]
tot = sum(buf[i] - base[i] for i in range(5))
for i, nm in enumerate(names):
    d = (buf[i] - base[i]) / n / S.rb.num_reqs
    print(f"{i} {nm:40s} {d:10.0f} cycles per CTA  {100 * (buf[i] - base[i]) / tot:5.1f}%")
PY
