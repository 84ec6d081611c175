"""One rank of config 5 (BASELINE configs[4]) on this GPU: bench.extra_config5 with the rank's
rectangles of an N-GPU layout.  usage: churn_rank.py RANK WORLD {head,balanced,layer} N3_UNITS OWNER(0/1)
Prints one line '@@{json}'.  Under ncu, `--nvtx --nvtx-include "timed/"` selects the timed batches."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_23640_b200 as cp  # noqa: E402
from paper_2605_23640_b200.shard import make_layout  # noqa: E402

rank, world, by, n3u, owner = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], float(sys.argv[4]), bool(int(sys.argv[5]))
rects = make_layout(rank, world, 32, 8, by, n3u)
print("@@" + json.dumps(bench.extra_config5(torch, cp, torch.device("cuda", 0), rects=rects, owner=owner)))
