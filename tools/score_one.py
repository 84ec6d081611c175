"""One config-2 N3 call (cp_score_deviation on the 512 reader spans) per variant listed on the command
line (cp_set_score_variant), for ncu captures of the row kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from paper_2605_23640_b200 import _lib as L  # noqa: E402
from synth.gen import attention_torch, make_workload  # noqa: E402

wl = make_workload(2)
_, rb = wl.rounds[0]
attn = {r: attention_torch(int(rb.lens[r]), rb.segments[r], 0.01, seed=r, device="cuda")
        for r in sorted(set(int(x) for x in rb.span_req))}
args = ([attn[int(r)] for r in rb.span_req], [int(rb.lens[int(r)]) for r in rb.span_req], [1] * len(rb.span_req),
        [int(b) for b in rb.span_begin], [int(b) + int(m) - 1 for b, m in zip(rb.span_begin, rb.span_len)])
for v in [int(x) for x in sys.argv[1:]] or [0]:
    L.check(L.lib().cp_set_score_variant(v))
    for _ in range(2):
        cp.score_deviation(*args, 1, 4)
    torch.cuda.synchronize()
