#!/bin/bash
# Launch list of the bench's timed steps (NVTX range "timed"): per-kernel durations, serialized and
# cold-cache under ncu -- compare SHARES of the step, not absolute times.
# usage (on the GPU box): tools/ncu_step.sh OUT.csv [bench.py args...]
out=$1; shift
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$out" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra "$@" > /dev/null
python tools/launch_table.py "$out"
