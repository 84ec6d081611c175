"""One annotator request of n tokens (default 10K, one coarse segment per ~1K tokens), run `reps`
times (or "batch": the 256 config-2 prompts); for ncu launch lists: ncu --metrics gpu__time_duration.sum python tools/annotate_one.py 10000 3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import attention_torch  # noqa: E402


def batch(reps):
    """The 256 config-2 writer prompts in one call (the many-request / flat form)."""
    from synth.gen import make_workload
    wb, _ = make_workload(2).rounds[0]
    mats = [attention_torch(int(wb.lens[r]), wb.segments[r], 0.01, seed=r) for r in range(wb.num_reqs)]
    masks = [torch.from_numpy(wb.req_mask(r).copy()).cuda() for r in range(wb.num_reqs)]
    for _ in range(reps):
        res = cp.annotate_spans(mats, masks, [1] * len(mats), min_len=128, workspace_bytes=8 << 30)
    torch.cuda.synchronize()
    print("batch", len(res), res[0][:2])


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "batch":
        return batch(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rng = np.random.default_rng(0)
    mask = np.zeros(n, np.uint8)
    mask[rng.choice(n, size=max(1, n // 1000), replace=False)] = 1
    bounds = [0] + [int(i) for i in np.nonzero(mask)[0]] + [n]
    segs = [(a + (a > 0), b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a + (a > 0)]
    A = attention_torch(n, segs, 0.01, seed=n)
    M = torch.from_numpy(mask).cuda()
    for _ in range(reps):
        res = cp.annotate_spans([A], [M], [1], min_len=128)
    torch.cuda.synchronize()
    print(n, res[0][:3])


if __name__ == "__main__":
    main()
