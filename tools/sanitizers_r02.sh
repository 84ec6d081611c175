export PYTORCH_NO_CUDA_MEMORY_CACHING=1
S=/usr/local/cuda/bin/compute-sanitizer
o=gpurun_out/sanitizers_r02.txt
echo "--- round 2: racecheck on the parallel commit apply + pins + sessions (tests/test_gpu_fuzz_index.py commit paths, test_gpu_pins.py, test_gpu_sessions.py seeds 0-3)" >> $o
timeout 900 $S --tool racecheck --print-limit 20 python -m pytest -q -x tests/test_gpu_fuzz_index.py -k "commit_paths and (300 or 301 or 302 or 303 or 304 or 305)" 2>&1 | tail -3 >> $o
timeout 900 $S --tool racecheck --print-limit 20 python -m pytest -q -x tests/test_gpu_pins.py -k "vs_oracle and (0 or 1 or 2)" 2>&1 | tail -3 >> $o
timeout 900 $S --tool racecheck --print-limit 20 python -m pytest -q -x tests/test_gpu_sessions.py -k "vs_oracle and (0 or 1 or 2 or 3)" 2>&1 | tail -3 >> $o
echo "--- memcheck: guards, views, pins, sessions, score fuzz (N3 grp), annotator long, privacy block 0" >> $o
timeout 1200 $S --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_guards.py tests/test_gpu_views.py tests/test_gpu_pins.py tests/test_gpu_fuzz_score.py -k "not 7 or guards" 2>&1 | tail -3 >> $o
timeout 1200 $S --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_sessions.py -k "vs_oracle and (0 or 1 or 5)" 2>&1 | tail -3 >> $o
echo "--- synccheck + initcheck: commit paths fuzz (4 seeds)" >> $o
timeout 900 $S --tool synccheck python -m pytest -q -x tests/test_gpu_fuzz_index.py -k "commit_paths and (300 or 301 or 302 or 303)" 2>&1 | tail -3 >> $o
timeout 900 $S --tool initcheck python -m pytest -q -x tests/test_gpu_fuzz_index.py -k "commit_paths and (300 or 301)" 2>&1 | tail -3 >> $o
tail -40 $o
