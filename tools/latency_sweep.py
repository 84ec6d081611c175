"""M6: single-request match latency vs request length against a 1,000-segment index.

The paper's only number on this path is its CPU retriever: 8.3 ms per 10,000-token request
(7.2 ms matching + 1.1 ms hashing, Xeon Silver 4510, averaged over 200 runs L1163).
This times cp_match_spans (hashing + prefix filter + verification + assembly, one request per call)
on the B200 and the CPU oracle on the same request, lengths 2.5K-10K (L1160)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle.oracle as O  # noqa: E402
import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import Batch, pack_batches, _fill, _passage  # noqa: E402


def main():
    rng = np.random.default_rng(6)
    nseg = 1000
    segs = [_passage(6, i, 128, 512) for i in range(nseg)]           # 1,000 stored segments
    writers = []
    for i, t in enumerate(segs):
        writers.append(Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=np.zeros(len(t), np.uint8),
                             writer_ids=np.array([i], np.int64), span_req=np.zeros(1, np.int32),
                             span_begin=np.zeros(1, np.int32), span_len=np.array([len(t)], np.int32)))
    wb = pack_batches(writers)
    cap = int(wb.span_len.sum()) + 1024
    cfg = cp.IndexConfig(num_layers=1, num_kv_heads=1, head_dim=16, dtype="bf16", pool_capacity_tokens=cap,
                         max_entries=cap // 128 + nseg + 64, max_span_len=512, max_req_tokens=50000,
                         max_batch_reqs=nseg, max_batch_tokens=max(wb.total_tokens, 50000), max_spans_per_insert=nseg)
    dev = torch.device("cuda", 0)
    idx = cp.KVIndex(cfg, dev)
    db = cp.DeviceBatch.from_numpy(wb.tokens, wb.offsets, wb.mask, dev)
    bt = torch.arange(wb.total_tokens // 16 + nseg + 1, dtype=torch.int32).view(1, -1)[:, : 0]
    nb = [(int(n) + 15) // 16 for n in wb.lens]
    bt = torch.zeros((nseg, max(nb)), dtype=torch.int32)
    o = 0
    for r, k in enumerate(nb):
        bt[r, :k] = torch.arange(o, o + k); o += k
    kv = cp.PagedKV.allocate(1, o, 1, 16, torch.bfloat16, bt, dev)
    sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev) for a in (wb.span_req, wb.span_begin, wb.span_len)]
    idx.insert(db, kv, *sp, None, None, 1)
    assert idx.last_error() == 0
    oidx = O.OracleIndex(128, 42, cap, idx.num_pages)
    oidx.insert(wb, None, None, 1)
    out = {"paper_cpu_ms_at_10k": 8.3, "paper_hw": "2x Xeon Silver 4510 (CPU retriever), P:L1220", "rows": []}
    for n in [2500, 5000, 7500, 10000, 20000, 50000]:        # > 10240: the scratch-array matcher
        # request: segments planted between fresh filler, ~70% covered
        parts, used = [], 0
        while used < n:
            if rng.random() < 0.3:
                f = _fill(rng, int(rng.integers(20, 200))); parts.append(f); used += len(f)
            else:
                t = segs[int(rng.integers(0, nseg))]; parts.append(t); used += len(t)
        req = np.concatenate(parts)[:n].astype(np.int32)
        rb = Batch(tokens=req, offsets=np.array([0, n], np.int64), mask=np.zeros(n, np.uint8),
                   writer_ids=np.array([0], np.int64))
        rdb = cp.DeviceBatch.from_numpy(rb.tokens, rb.offsets, None, dev)
        hits = cp.Hits(n // 128 + 2, 1, n, dev)
        for _ in range(5):
            idx.match_spans(rdb, 2, no_touch=True, use_mask=False, hits=hits)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        e0.record()
        for _ in range(reps):
            idx.match_spans(rdb, 2, no_touch=True, use_mask=False, hits=hits)
        e1.record()
        torch.cuda.synchronize()
        gpu_ms = e0.elapsed_time(e1) / reps
        h = hits.to_host()
        t0 = time.perf_counter()
        res = oidx.match(rb, t=2, no_touch=True, use_mask=False)
        cpu_ms = (time.perf_counter() - t0) * 1e3
        same = (res.num_hits == h["num_hits"] and np.array_equal(res.hit_dst, h["hit_dst"])
                and np.array_equal(res.hit_entry, h["hit_entry"]))
        out["rows"].append({"n": n, "gpu_match_ms": round(gpu_ms, 4), "oracle_cpu_ms": round(cpu_ms, 2),
                            "hits": int(res.num_hits), "covered": int(res.req_covered[0]),
                            "candidates": int(res.req_candidates[0]), "parity": bool(same)})
        print(out["rows"][-1], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "latency_sweep.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
