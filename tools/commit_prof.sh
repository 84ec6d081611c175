#!/bin/bash
# Diagnostic build of the library with the commit phase profiler, then a churn run (GPU box only).
set -e
cd "$(dirname "$0")/.."
H=paper_2605_23640_b200
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr --extended-lambda -DCP_COMMIT_PROF -o $H/libcacheprune.so $H/csrc/cp_index.cu $H/csrc/cp_match.cu \
  $H/csrc/cp_gather.cu $H/csrc/cp_score.cu $H/csrc/cp_annotate.cu $H/csrc/cp_policy.cu
CP_DIAGNOSTIC_BUILD=1 python tools/commit_prof.py "$@"   # a diagnostic build: not the hashed flags
