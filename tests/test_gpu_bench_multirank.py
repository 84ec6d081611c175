"""The bench's N > 1 path end to end: two ranks (torchrun, gloo, both on cuda:0 -- this box has one
GPU) run the layer-sharded step with the N3 owner's bit broadcast, barriers, max-over-ranks timing and
the e2e leg; rank 0 prints one JSON line.  Catches collective-count mismatches between ranks."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("overlap", [3, 2, 0])
def test_two_rank_bench_runs_and_reports(overlap):
    env = dict(os.environ, BENCH_DEVICE0="1", BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29611 + overlap), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--scale", "0.1", "--no-cpu-baseline", "--overlap", str(overlap)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "balanced-sharded x2" and d["gpu_launches"] > 0   # config 2 default


def test_single_rank_bench_line_has_the_contract_keys():
    cmd = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--scale", "0.1", "--cpu-seconds", "1"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2 and r["peak"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in d["config"] and "sm_mhz" in d["clocks"]


def test_world_size_one_nccl_group_runs_the_multirank_path():
    """--dist-ws1: a world-size-1 NCCL process group, so bench.py's N > 1 branch -- the device-tensor
    NCCL broadcast of the recompute bits (shard.broadcast_update), the barriers and the max-over-ranks
    all_reduce -- executes on this one-GPU box (the driver's SCALE run is then not its first execution)."""
    env = {k: v for k, v in os.environ.items() if k not in ("BENCH_DIST_BACKEND", "RANK", "WORLD_SIZE")}
    env["MASTER_PORT"] = "29641"
    cmd = [sys.executable, "bench.py", "--dist-ws1", "--steps", "3", "--warmup", "3", "--scale", "0.1",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["config"].get("dist_backend") == "nccl"


@pytest.mark.parametrize("rank", [0, 3, 7])
def test_balanced_layout_rank_runs(rank):
    """One simulated rank of the 8-GPU balanced layer layout (base index + pool views) runs the step."""
    cmd = [sys.executable, "bench.py", "--by", "balanced", "--shard-world", "8", "--shard-rank", str(rank),
           "--steps", "3", "--warmup", "3", "--scale", "0.1", "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    from paper_2605_23640_b200.shard import balanced_units
    u0, u1 = balanced_units(8, 32, 8, d["config"]["n3_units"])[rank]
    assert d["config"]["shard_units"] == u1 - u0 and d["value"] > 0


def test_two_rank_balanced_bench_runs():
    env = dict(os.environ, BENCH_DEVICE0="1", BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29651", "bench.py", "--gpus", "2", "--by", "balanced",
           "--steps", "3", "--warmup", "3", "--scale", "0.1", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "balanced-sharded x2"


def test_cuda_graph_step_matches_the_eager_step():
    """The timed steps are replays of one captured step (device clock, cp_index_set_clock): the same
    hits, coverage and byte counts as eager steps, no device error; the line says which it used."""
    outs = {}
    for flag in ([], ["--no-graph"]):
        cmd = [sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--scale", "0.1", "--no-cpu-baseline",
               "--no-extra"] + flag
        out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-3000:]
        outs[bool(flag)] = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    g, e = outs[False], outs[True]
    assert g["config"]["cuda_graph"] is True and e["config"]["cuda_graph"] is False
    for k in ("covered_tokens", "reused_tokens", "recompute_tokens", "hits"):
        assert g[k] == e[k], k
    assert g["roofline"]["algorithmic_bytes_per_launch"] == e["roofline"]["algorithmic_bytes_per_launch"]
    assert g["gpu_launches"] == e["gpu_launches"]
