"""Projected strong scaling of the layer- (or head-) sharded bench step from one GPU.

This box gives one GPU, so each rank of an N-GPU layout is run alone on it (`bench.py --shard-world N
--shard-rank r`: that rank's shard of the pool / destination caches, the replicated match + insert,
and N3 only on the rank that owns the final layer).  The N-GPU step time is projected as the max over
the ranks that differ (rank 0 and the N3 owner -- the other ranks equal rank 0 -- or, for the
balanced layout, every rank), i.e. no NVLink cost
is modelled beyond what the step already contains: the only collective of the step is the
index-update broadcast of the packed recompute bits (~50 KB, microseconds).  Writes
gpurun_out/scaling_sim.json."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args):
    out = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--no-e2e", "--no-extra"] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


def main():
    by = sys.argv[1] if len(sys.argv) > 1 else "layer"
    extra = sys.argv[2:]                      # e.g. --config 3, --n3-units 5; --base 2: efficiency vs N = 2
    base = 1
    if "--base" in extra:
        i = extra.index("--base")
        base = int(extra[i + 1])
        extra = extra[:i] + extra[i + 2:]
    res = {"by": by, "args": extra, "base_n": base, "note": __doc__.split("\n\n")[1].replace("\n", " "), "rows": []}
    if base == 1:
        one = run(["--by", by] + extra)
        t1 = one["ms_per_step"]
        res["rows"].append({"n": 1, "ms_per_step": t1, "value_GBps": one["value"], "efficiency": 1.0})
    for n in [n for n in (2, 4, 8) if n >= base]:
        owner = n - 1 if by in ("layer", "balanced") else 0
        # balanced: every rank's rectangles differ, so every rank is run
        ranks = list(range(n)) if by == "balanced" else sorted({0, owner})
        per = {r: run(["--by", by, "--shard-world", str(n), "--shard-rank", str(r)] + extra) for r in ranks}
        tmax = max(d["ms_per_step"] for d in per.values())
        if n == base and base > 1:           # e.g. config 4: one GPU cannot hold the whole pool
            t1, one = base * tmax, {"value": next(iter(per.values()))["value"]}   # whole job at N = base: base ranks
        res["rows"].append({
            "n": n, "ms_per_step_max_over_ranks": tmax,
            "per_rank": {str(r): {"ms_per_step": d["ms_per_step"], "breakdown_ms": d["breakdown_ms"],
                                  "shard_rects": d["config"].get("shard_rects")} for r, d in per.items()},
            "projected_value_GBps": round(one["value"] * t1 / tmax, 1),
            "efficiency_T1_over_N_TN": round(t1 / (n * tmax), 4)})
        print(json.dumps(res["rows"][-1]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = by + ("_" + "_".join(a.strip("-") for a in extra) if extra else "") + (f"_base{base}" if base > 1 else "")
    with open(os.path.join(ROOT, "gpurun_out", f"scaling_sim_{tag}.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
