"""A/B the gather kernel variants on the config-2 bench workload (prints GB/s per variant)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_23640_b200 as cp  # noqa: E402


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--by", default="layer")
    ap.add_argument("--shard-world", type=int, default=0)
    ap.add_argument("--shard-rank", type=int, default=0)
    A = ap.parse_args()
    A.scale = 1.0
    S = bench.setup_ours(A, 0, 1, torch.device("cuda", 0))
    S.idx.match_spans(S.rdb, 1000, hits=S.hits)
    torch.cuda.synchronize()
    cov = int(S.hits.req_covered.sum()); rec = int(S.hits.req_recompute.sum())
    row = S.shard.num_layers * S.shard.num_heads * S.g.head_dim * 2
    nbytes = (cov - rec) * 2 * row * 2 + rec * 2 * row
    out = {}
    variants = [0, 5, 3, 6, 8, 9, 4]
    for v in variants + variants[:-1]:
        cp._lib.lib().cp_set_gather_variant(v)
        for _ in range(3):
            S.idx.gather_rerotate(S.rdb, S.hits, S.dst)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n):
            S.idx.gather_rerotate(S.rdb, S.hits, S.dst)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        out.setdefault(f"variant{v}", []).append({"ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1)})
        print(v, out[f"variant{v}"][-1], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
