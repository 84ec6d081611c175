"""Print parity statistics per workload (GPU vs oracle); writes gpurun_out/parity_report.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth.gen import make_workload  # noqa: E402
from tests.harness import Case, ParityReport, run_round_parity  # noqa: E402


def main():
    out = {}
    t0 = time.time()
    out["config1_toy"] = run_round_parity(Case(make_workload(1)))
    out["config1_toy"]["secs"] = time.time() - t0
    for name, cfg, scale, kw in [("config2_reduced", 2, 0.125, dict(sample_reqs=4, sample_layers=[0, 31])),
                                 ("config2_full", 2, 1.0, dict(sample_reqs=2, sample_layers=[0, 31])),
                                 ("config3_reduced", 3, 0.08, dict(sample_reqs=3, sample_layers=[0, 31]))]:
        t0 = time.time()
        case = Case(make_workload(cfg, scale=scale), **kw)
        rep = ParityReport()
        wb, rb = case.wl.rounds[0]
        case.insert(wb, rep, sparse_kv=(cfg == 3))
        case.score_parity(wb, rep, max_spans=16)
        case.match_and_gather(rb, rep)
        out[name] = dict(ok=rep.ok, notes=rep.notes[:5], secs=time.time() - t0, **rep.stats)
        del case
    if "--all" in sys.argv:
        # every request's K/V rows compared (not a sample) at full BASELINE sizes, on a few layers
        for name, cfg, kw in [("config2_full_all_requests", 2, dict(sample_layers=[0, 13, 31])),
                              ("config3_full_all_requests", 3, dict(sample_layers=[0, 31])),
                              ("config4_layer_shard_all_requests", 4, dict(layer_range=(70, 80), sample_layers=[0, 9]))]:
            t0 = time.time()
            case = Case(make_workload(cfg), sample_reqs=None, **kw)
            rep = ParityReport()
            wb, rb = case.wl.rounds[0]
            case.insert(wb, rep, sparse_kv=(cfg != 2))
            case.match_and_gather(rb, rep)
            out[name] = dict(ok=rep.ok, notes=rep.notes[:5], secs=time.time() - t0, requests_checked=rb.num_reqs,
                             **rep.stats)
            print(name, out[name]["ok"], round(out[name]["secs"], 1), flush=True)
            del case
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.json"), "w") as f:
        json.dump(out, f, indent=1, default=float)
    print(json.dumps(out, indent=1, default=float))


if __name__ == "__main__":
    main()
