"""One annotator request of n tokens (default 10K, one coarse segment per ~1K tokens), run `reps`
times; for ncu launch lists: ncu --metrics gpu__time_duration.sum python tools/annotate_one.py 10000 3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import attention_torch  # noqa: E402


def main():
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
