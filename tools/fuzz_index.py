"""Long randomized GPU-vs-oracle search over the index / matcher / gather (the generators of
tests/test_gpu_fuzz_index.py), many more seeds than the test suite runs, and the NEXT-3 policies.
Usage: python tools/fuzz_index.py [first_seed] [count].  Prints failing seeds with their first notes
and writes gpurun_out/fuzz_index.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from tests.harness import Case, ParityReport  # noqa: E402
from tests.test_gpu_fuzz_index import _workload  # noqa: E402


def one(seed):
    heavy = seed % 2 == 0
    policy = [None, None, None, "fixed_chunk", "prefix_only"][seed % 5]
    w = [8, 8, 32, 128][(seed // 7) % 4]                  # window lengths up to the paper's 128
    wl = _workload(seed, "bf16" if (seed // 2) % 2 else "fp32", heavy=heavy, w=w)
    rho = (0, 4) if seed % 3 == 1 else (1, 4)          # no recompute marks: pages can link (NEXT-2)
    sessions = policy is None and seed % 8 == 6                # R#33 session turns (method policy only)
    pins = seed % 8 in (3, 6)                                  # R#32 random pins / releases
    case = Case(wl, seed=seed, sample_reqs=None, use_reader_mask=seed % 7 != 0, policy=policy, rho=rho,
                max_sessions=4 if sessions else 0, batch_slack=64 if sessions else 0)
    rep = ParityReport()
    held = []
    prev = None
    import dataclasses
    rng = np.random.default_rng(seed + 7)
    for wb, rb in wl.rounds:
        if seed % 6 == 5 and rng.random() < 0.5 and len(wb.span_len):
            # inject one invalid span (covers a masked token, or is shorter than w, or runs past the
            # request) at a random position: both sides must reject the whole call without side effects
            kind = int(rng.integers(3))
            r = int(rng.integers(wb.num_reqs))
            n = int(wb.lens[r])
            masked = np.nonzero(wb.req_mask(r))[0]
            if kind == 0 and len(masked):
                b0 = max(0, int(masked[0]) - 4); bad = (r, b0, min(n - b0, 12))
            elif kind == 1:
                bad = (r, 0, min(n, 5))
            else:
                bad = (r, max(0, n - 4), 12)
            pos = int(rng.integers(len(wb.span_len)))          # replace a span: the call keeps its span count
            def put(arr, v):
                arr = np.array(arr, np.int32)
                arr[pos] = v
                return arr
            wb = dataclasses.replace(wb, span_req=put(wb.span_req, bad[0]), span_begin=put(wb.span_begin, bad[1]),
                                     span_len=put(wb.span_len, bad[2]))
        if pins:
            import torch
            ents = case.dev.snapshot(with_tokens=False)["entries"]
            if ents and rng.random() < 0.7:
                e = ents[int(rng.integers(0, len(ents)))]
                pg = [int(x) for x in rng.choice(e["pages"], size=min(2, len(e["pages"])), replace=False)]
                case.dev.pin_links(torch.tensor(pg, dtype=torch.int32, device="cuda"), 1)
                assert case.dev.last_error() == 0 and case.orc.pin_pages(pg, 1) == 0
                held.append(pg)
            if held and rng.random() < 0.3:
                pg = held.pop(int(rng.integers(0, len(held))))
                case.dev.pin_links(torch.tensor(pg, dtype=torch.int32, device="cuda"), -1)
                assert case.dev.last_error() == 0 and case.orc.pin_pages(pg, -1) == 0
        case.insert(wb, rep, concurrent_readers=prev if seed % 4 == 1 else None)   # split insert beside match/gather
        if not rep.ok:
            break
        sess = None
        if sessions:
            keep = [r for r in range(wb.num_reqs) if int(wb.lens[r]) <= wl.max_span_len]
            sw = wb.subset(keep)
            case.insert_session(sw, rng.integers(1, 5, sw.num_reqs).astype(np.int32), rep)
            if not rep.ok:
                break
            sess = rng.integers(0, 5, rb.num_reqs).astype(np.int32)
        case.match_and_gather(rb, rep, sessions=sess)
        if not rep.ok:
            break
        if seed % 3 == 1:
            case.compare_links(wb, rep)                    # writers re-reading: delta-0 aligned hits link
            case.compare_links(rb, rep)
            if not rep.ok:
                break
        prev = rb
        if seed % 3 == 0:
            case.match_and_gather(wb, rep, no_touch=True)
            if not rep.ok:
                break
    return rep


def main():
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 500
    fails, stats, t0 = [], {}, time.time()
    for seed in range(first, first + count):
        try:
            rep = one(seed)
            ok, notes = rep.ok, rep.notes[:4]
            for k, v in rep.stats.items():
                if isinstance(v, (int, float)) and k in ("stored", "duplicate", "hits", "moved_hits", "covered",
                                                          "linked_blocks", "session_stored"):
                    stats[k] = stats.get(k, 0) + v
        except Exception as e:  # noqa: BLE001 -- report and continue
            ok, notes = False, [repr(e)[:300]]
        if not ok:
            fails.append({"seed": seed, "notes": notes})
            print("FAIL", seed, notes, flush=True)
    out = {"first_seed": first, "count": count, "failures": fails, "stats": stats, "seconds": round(time.time() - t0, 1)}
    print(json.dumps(out)[:2000])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fuzz_index.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
