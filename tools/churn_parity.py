"""Config 5 end to end with oracle parity at every batch: the full high-churn mix (40 batches x 256
requests, 100K-passage Zipf corpus, 1.5M-token budget on one KV-head shard), each batch
match -> gather -> insert on the device and in the oracle, comparing insert outcomes / ids, the whole
live index, hits, plans, stats and sampled KV rows.  Writes gpurun_out/churn_parity.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth.gen import Geometry, churn_workload  # noqa: E402
from tests.harness import Case, ParityReport  # noqa: E402


def main():
    batches = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    g = Geometry(32, 8, 128, "bf16", 500000.0)
    wl = churn_workload(batches=batches, per_batch=256, corpus=100000, capacity_tokens=1_500_000, geometry=g)
    case = Case(wl, head_range=(0, 1), sample_reqs=1, sample_layers=[0, 31])
    rep = ParityReport()
    t0 = time.time()
    done = 0
    for wb, rb in wl.rounds:
        case.match_and_gather(rb, rep)
        if not rep.ok:
            break
        case.insert(wb, rep)
        if not rep.ok:
            break
        done += 1
    out = {"what": __doc__.split("\n\n")[0].replace("\n", " "), "batches": batches, "batches_ok": done,
           "ok": rep.ok, "notes": rep.notes[:8], "stats": rep.stats, "live_entries": len(case.orc.live_entries()),
           "ids_issued": case.orc.num_ids, "seconds": round(time.time() - t0, 1)}
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "churn_parity.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
