"""NEXT-3: the method (CrossUserSelective) vs the FixedChunk(128) and PrefixOnly baseline policies
on the BASELINE workloads (Fig. 4, §5.7).

For each config and policy, one index on the GPU is filled from the writer batches (the method:
the workload's coarse-segment spans; FixedChunk / PrefixOnly: cp_policy_spans), then the readers are
matched with the policy's cp_match_spans flag.  Reports match rate (covered / request tokens),
reused (non-recompute) tokens and the device time of cp_policy_spans and cp_match_spans.
Match rates do not depend on the KV payload, so the pools here hold a 1-layer x 1-head geometry.
Writes gpurun_out/policy_compare.json."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import make_workload  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def run(cfg_id, scale, dev):
    wl = make_workload(cfg_id, scale=scale)
    g = wl.geometry
    w = g.window_len
    out = {"workload": wl.name, "config": cfg_id, "rounds": len(wl.rounds)}
    writers = [wb for wb, _ in wl.rounds if wb is not None]
    readers = [rb for _, rb in wl.rounds]
    lens = [int(b.lens.max()) for b in writers + readers]
    for policy in (None, "fixed_chunk", "prefix_only"):
        name = policy or "selective"
        spans_cap = max(b.total_tokens // w + b.num_reqs for b in writers)
        icfg = cp.IndexConfig(num_layers=1, num_kv_heads=1, head_dim=64, dtype="bf16", rope_theta=g.rope_theta,
                              window_len=w, pool_capacity_tokens=wl.pool_capacity_tokens,
                              max_entries=min(131072, wl.pool_capacity_tokens // w + spans_cap + 64),
                              max_span_len=wl.max_span_len, max_req_tokens=min(10240, max(lens)),
                              max_batch_reqs=max(b.num_reqs for b in writers + readers),
                              max_batch_tokens=max(b.total_tokens for b in writers + readers),
                              max_spans_per_insert=spans_cap)
        idx = cp.KVIndex(icfg, dev)
        t = 0
        cov = rec = tot = nh = 0
        spans_ms, match_ms, nspans = [], [], 0
        for wb, rb in wl.rounds:
            if wb is not None:
                db = cp.DeviceBatch.from_numpy(wb.tokens, wb.offsets, wb.mask, dev)
                if policy is None:
                    sp = tuple(torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev)
                               for a in (wb.span_req, wb.span_begin, wb.span_len))
                else:
                    spans_ms.append(timed(lambda: cp.policy_spans(db, policy, w, wl.max_span_len)))
                    sp = cp.policy_spans(db, policy, w, wl.max_span_len)
                nspans += int(sp[0].numel())
                nb = [(int(n) + 15) // 16 for n in wb.lens]
                bt = torch.zeros((wb.num_reqs, max(nb)), dtype=torch.int32)
                o = 0
                for r, k in enumerate(nb):
                    bt[r, :k] = torch.arange(o, o + k); o += k
                kv = cp.PagedKV.allocate(1, o, 1, 64, torch.bfloat16, bt, dev, zero=True)
                t += 1
                # recompute marks: none (match rates only)
                idx.insert(db, kv, *sp, None, None, t)
                del kv
            rdb = cp.DeviceBatch.from_numpy(rb.tokens, rb.offsets, rb.mask, dev)
            t += 1
            hits = idx.match_spans(rdb, t, policy=policy)
            match_ms.append(timed(lambda: idx.match_spans(rdb, t, no_touch=True, hits=hits, policy=policy)))
            cov += int(hits.req_covered.sum()); rec += int(hits.req_recompute.sum())
            nh += int(hits.num_hits.item()); tot += rb.total_tokens
        if idx.last_error():
            raise RuntimeError(f"{name}: device error")
        out[name] = {"match_rate": round(cov / max(tot, 1), 4), "covered_tokens": cov, "request_tokens": tot,
                     "hits": nh, "stored_spans_offered": nspans,
                     "match_ms_median_per_round": round(float(np.mean(match_ms)), 4),
                     "policy_spans_ms": round(float(np.mean(spans_ms)), 4) if spans_ms else None}
        del idx
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,5")
    ap.add_argument("--scale5", type=float, default=0.1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    res = []
    for c in [int(x) for x in args.configs.split(",")]:
        r = run(c, args.scale5 if c == 5 else 1.0, dev)
        print(json.dumps(r), flush=True)
        res.append(r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "policy_compare.json"), "w") as f:
        json.dump({"note": "match rates of the method vs the NEXT-3 baseline policies (tools/policy_compare.py)",
                   "results": res}, f, indent=1)


if __name__ == "__main__":
    main()
