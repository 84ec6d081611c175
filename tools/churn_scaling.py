"""Projected scaling of config 5 (BASELINE configs[4], high-churn serving mix) on 2, 4 and 8 GPUs, from
one GPU.

A rank holds a set of (layer, KV head) units of Llama-3-8B KV: `head` = 8 / N KV heads of every layer;
`balanced` = contiguous units in (layer, head) order with the N3 owner (the last rank, which holds the
final layer's attention) given bench.N3_UNITS[5] fewer units.  The index metadata, the match and the
insert's control plane are replicated.  A rank is run alone on this GPU (`bench.extra_config5` with the
rank's rectangles: the same seeded churn workload, LRU budget full, then timed batches in the bench's
schedule); the projected N-GPU step is the max over ranks.  Ranks run: head -- rank 0 (the owner; the
others are the same step without N3, reported); balanced -- the owner and the first rank with the most
units (the others hold as many or fewer units).  N = 1 does not fit one B200 (the 8-head pool
alone is 1.5M x 32 x 8 x 128 x 2 B x 2 = 197 GB), so efficiency is relative to N = 2:
E(N) = 2 T(2) / (N T(N)).  Writes gpurun_out/churn_scaling_<layout>.json."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_23640_b200.shard import balanced_units, make_layout  # noqa: E402

def run(rank, world, by, n3u, owner):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "churn_rank.py"), str(rank), str(world), by,
                          str(n3u), str(int(owner))], cwd=ROOT, capture_output=True, text=True, timeout=1200)
    lines = [l for l in out.stdout.splitlines() if l.startswith("@@")]
    if out.returncode or not lines:
        raise RuntimeError(f"{by} rank {rank}/{world}: rc={out.returncode}\n{out.stderr[-3000:]}")
    return json.loads(lines[-1][2:])


def main():
    by = sys.argv[1] if len(sys.argv) > 1 else "balanced"
    sys.path.insert(0, ROOT)
    import bench
    n3u = bench.N3_UNITS[5] if by == "balanced" else 0.0
    res = {"layout": by, "n3_units": n3u, "note": __doc__.split("\n\n")[1].replace("\n", " "), "rows": []}
    for n in (2, 4, 8):
        if by == "head":
            ranks = {0: True}
        else:
            u = balanced_units(n, 32, 8, n3u)
            most = max(b - a for a, b in u[:-1])
            first = min(r for r in range(n - 1) if u[r][1] - u[r][0] == most)
            ranks = {first: False, n - 1: True}
        per = {r: run(r, n, by, n3u, own) for r, own in ranks.items()}
        steps = {r: d["per_batch_median"]["step_ms"] for r, d in per.items()}
        row = {"n": n, "step_ms_max_over_ranks": max(steps.values()),
               "per_rank": {str(r): {"rects": d["rects"], "units": d["units"], "runs_n3": d["runs_n3"],
                                     "per_batch_median": d["per_batch_median"],
                                     "per_batch_step_ms": d["per_batch_step_ms"],
                                     "stored_per_batch": d["stored_per_batch"],
                                     "evicted_per_batch": d["evicted_per_batch"],
                                     "copy_in_bytes_per_batch": d["copy_in_bytes_per_batch"],
                                     "commit_GBps_lower_bound": d["commit_GBps_lower_bound"],
                                     **({"warning": d["warning"]} if "warning" in d else {})}
                            for r, d in per.items()}}
        if by == "head":
            m = per[0]["per_batch_median"]
            row["other_ranks_step_ms_est"] = round(m["step_ms"] - m["score_ms"], 4)
        res["rows"].append(row)
        print(json.dumps({"n": n, "steps": steps}), flush=True)
    t2 = res["rows"][0]["step_ms_max_over_ranks"]
    for row in res["rows"]:
        row["efficiency_vs_n2"] = round(2 * t2 / (row["n"] * row["step_ms_max_over_ranks"]), 4)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"churn_scaling_{by}.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps([(r["n"], r["step_ms_max_over_ranks"], r["efficiency_vs_n2"]) for r in res["rows"]]))


if __name__ == "__main__":
    main()
