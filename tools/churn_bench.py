"""Config 5 (BASELINE configs[4]): high-churn serving mix on one GPU = one KV-head shard of the
8-GPU head-sharded layout (Llama-3-8B: 32 layers x 1 of 8 KV heads x 128, bf16).

40 batches x 256 requests of ~1.6K tokens: [system 128] + 9 x ([PII 3-5] [passage 128-192]) from a
100K-passage Zipf(1.1) corpus.  Per batch (every request is a reader, then a writer):
  cp_match_spans -> cp_gather_rerotate -> cp_score_deviation (rho = 1/4) -> cp_index_insert
under a 1.5M-token LRU budget (the Zipf draws touch ~16K distinct passages = 2.6M tokens, so the
budget forces steady LRU eviction: 'high churn').  Reports per-phase device times, the
insert outcome mix and index-level invariants (budget, live counts, no device error).
Writes gpurun_out/churn.json."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import Geometry, attention_torch, churn_workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=40)
    ap.add_argument("--per-batch", type=int, default=256)
    ap.add_argument("--corpus", type=int, default=100000)
    ap.add_argument("--capacity", type=int, default=1_500_000)
    ap.add_argument("--heads", type=int, default=1)
    args = ap.parse_args()
    g = Geometry(32, 8, 128, "bf16", 500000.0)
    t0 = time.time()
    wl = churn_workload(batches=args.batches, per_batch=args.per_batch, corpus=args.corpus,
                        capacity_tokens=args.capacity, geometry=g)
    gen_s = time.time() - t0
    dev = torch.device("cuda", 0)
    w = g.window_len
    spans_max = max(len(b.span_len) for b, _ in wl.rounds)
    toks_max = max(b.total_tokens for b, _ in wl.rounds)
    cfg = cp.IndexConfig(num_layers=32, num_kv_heads=args.heads, head_dim=128, dtype="bf16", rope_theta=5e5,
                         pool_capacity_tokens=args.capacity, max_entries=args.capacity // w + spans_max + 64,
                         max_span_len=256, max_req_tokens=int(max(b.lens.max() for b, _ in wl.rounds)),
                         max_batch_reqs=args.per_batch, max_batch_tokens=toks_max, max_spans_per_insert=spans_max)
    idx = cp.KVIndex(cfg, dev)
    H, d = args.heads, 128
    row = 32 * H * d * 2
    rows = []
    t = 0
    for bi, (wb, rb) in enumerate(wl.rounds):
        db = cp.DeviceBatch.from_numpy(rb.tokens, rb.offsets, rb.mask, dev)
        nb = [(int(n) + 15) // 16 for n in rb.lens]
        bt = torch.zeros((rb.num_reqs, max(nb)), dtype=torch.int32)
        o = 0
        for r, k in enumerate(nb):
            bt[r, :k] = torch.arange(o, o + k); o += k
        kv = cp.PagedKV.allocate(32, o, H, d, torch.bfloat16, bt, dev, zero=False)
        for tsr in kv.k + kv.v:
            tsr.normal_()
        attn = {r: attention_torch(int(rb.lens[r]), rb.segments[r], 0.01, seed=bi * 1000 + r, device=dev)
                for r in sorted(set(int(x) for x in rb.span_req))}
        sargs = ([attn[int(r)] for r in rb.span_req], [int(rb.lens[int(r)]) for r in rb.span_req],
                 [1] * len(rb.span_req), [int(x) for x in rb.span_begin],
                 [int(x) + int(m) - 1 for x, m in zip(rb.span_begin, rb.span_len)])
        sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev) for a in (rb.span_req, rb.span_begin, rb.span_len)]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        torch.cuda.synchronize()
        t += 1
        ev[0].record()
        hits = idx.match_spans(db, t)
        ev[1].record()
        idx.gather_rerotate(db, hits, kv)
        ev[2].record()
        sc, bits, so, bo = cp.score_deviation(*sargs, 1, 4)
        ev[3].record()
        boff = torch.tensor(bo[:-1], dtype=torch.int64, device=dev)
        ids, oc = idx.insert(db, kv, *sp, bits, boff, t)
        ev[4].record()
        torch.cuda.synchronize()
        err = idx.last_error()
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        ocn = oc.cpu().numpy()
        h = hits.to_host()
        cov, rec = int(h["req_covered"].sum()), int(h["req_recompute"].sum())
        gbytes = (cov - rec) * 2 * row * 2 + rec * 2 * row
        rows.append({"batch": bi, "err": err, "match_ms": ms[0], "gather_ms": ms[1], "score_ms": ms[2],
                     "insert_ms": ms[3], "hits": h["num_hits"], "covered": cov, "tokens": rb.total_tokens,
                     "gather_GBps": gbytes / ms[1] / 1e6 if ms[1] > 0 else 0.0,
                     "stored": int(np.sum((ocn == 0) | (ocn == 1))), "superseded": int(np.sum(ocn == 1)),
                     "duplicate": int(np.sum(ocn == 2)), "dropped": int(np.sum(ocn == 3))})
        print(json.dumps(rows[-1]), flush=True)
        del kv, attn
        if err:
            break
    snap = idx.snapshot(with_tokens=False)
    summary = {
        "workload": "config 5 high-churn, one KV-head shard (1 of 8) of Llama-3-8B KV",
        "batches": len(rows), "requests": sum(r["tokens"] > 0 for r in rows) * args.per_batch,
        "capacity_tokens": args.capacity, "final_live_entries": snap["num_live"], "final_live_tokens": snap["live_tokens"],
        "next_id": snap["next_id"], "budget_ok": snap["live_tokens"] <= args.capacity, "device_error": snap["error"],
        "mean_ms": {k: float(np.mean([r[k] for r in rows[1:]])) for k in ("match_ms", "gather_ms", "score_ms", "insert_ms")},
        "match_rate": float(sum(r["covered"] for r in rows) / sum(r["tokens"] for r in rows)),
        "outcomes": {k: int(sum(r[k] for r in rows)) for k in ("stored", "superseded", "duplicate", "dropped")},
        "removed_by_lru_or_supersede": int(sum(r["stored"] for r in rows) - snap["num_live"]),
        "mean_gather_GBps": float(np.mean([r["gather_GBps"] for r in rows[1:]])),
        "generator_s": gen_s,
        "commits_parallel_serial_why": list(idx.commit_stats()),
        "commit_path": os.environ.get("CP_COMMIT_SERIAL", "0") != "0" and "sequential (CP_COMMIT_SERIAL=1)" or "default",
        "rows": rows,
    }
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "churn.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))


if __name__ == "__main__":
    main()
