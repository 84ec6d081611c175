"""Phase profile of k_ins_commit under config-5 churn.  Needs a library built with -DCP_COMMIT_PROF
(diagnostic build, see tools/commit_prof.sh); prints accumulated clock64 cycles per phase:
0 relation CSR, 1 parallel prefix decisions, 2 LRU candidate list (radix select + sort),
3 sequential apply / deferred page traffic, 4 write-back; 5-9 sub-phases of the parallel apply; counters 13-15."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import churn_bench  # noqa: E402
from paper_2605_23640_b200 import _lib as L  # noqa: E402

if __name__ == "__main__":
    churn_bench.main()
    buf = (C.c_ulonglong * 16)()
    f = L.lib().cp_commit_prof_read
    f.argtypes = [C.c_void_p]
    f.restype = C.c_int
    assert f(buf) == 0
    names = {0: "relation CSR", 1: "parallel prefix", 2: "LRU candidates", 3: "sequential apply", 4: "write-back",
             5: " par: init", 6: " par: decisions", 7: " par: store scans", 8: " par: victims+checks", 9: " par: apply",
             10: " lru: min/max pass", 11: " lru: radix passes", 12: " lru: collect"}
    tot = sum(buf[i] for i in range(13))
    for i in range(16):
        if buf[i]:
            print(f"{i:2d} {names.get(i, 'counter'):18s} {buf[i]:>14d}" + (f"  {100 * buf[i] / tot:5.1f}%" if i < 13 else ""))
