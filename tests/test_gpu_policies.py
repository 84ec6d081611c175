"""GPU parity for the NEXT-3 baseline policies (R#28-29): cp_policy_spans and
cp_match_spans with CP_MATCH_FIXED_CHUNK / CP_MATCH_PREFIX_ONLY vs the oracle, bit exact on spans,
entry tables, hits, plan codes and gathered V (K within the gather's tolerance), plus the
granularity-gap direction measured through the C-ABI."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.gen import Batch, Geometry, Workload, make_workload, pack_batches  # noqa: E402
from tests.harness import Case, run_round_parity  # noqa: E402

VOCAB = 128256


def _assert(res):
    assert res["ok"], res["notes"]


@pytest.mark.parametrize("policy", ["fixed_chunk", "prefix_only"])
def test_policies_toy_all_rounds(policy):
    res = run_round_parity(Case(make_workload(1), policy=policy), score=False)
    _assert(res)
    assert res["policy_spans"] > 0


@pytest.mark.parametrize("policy", ["fixed_chunk", "prefix_only"])
def test_policies_msmarco_config2_reduced(policy):
    case = Case(make_workload(2, scale=0.125), sample_reqs=4, sample_layers=[0, 31], policy=policy)
    res = run_round_parity(case, score=False)
    _assert(res)
    assert res["covered"] > 0
    if policy == "prefix_only":
        assert res["hits"] > 0


@pytest.mark.parametrize("policy", ["fixed_chunk", "prefix_only"])
def test_policies_multidoc_config3_reduced(policy):
    case = Case(make_workload(3, scale=0.08), sample_reqs=3, sample_layers=[0, 31], policy=policy)
    res = run_round_parity(case, score=False)
    _assert(res)


def test_prefix_only_partial_prefix_gather():
    """Readers that share a long writer prefix only in part: PrefixOnly hits shorter than their
    entry (hit_len < entry length), gathered with delta 0 as bit copies."""
    g = Geometry(4, 2, 64, "bf16", 500000.0, window_len=16)
    rng = np.random.default_rng(31)
    sysp = rng.integers(1000, 90000, 100).astype(np.int32)
    writers, readers = [], []
    for i in range(6):
        t = np.concatenate([sysp, rng.integers(1000, 90000, 60 + 7 * i).astype(np.int32)])
        writers.append(Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=np.zeros(len(t), np.uint8),
                             writer_ids=np.array([i], np.int64)))
        cut = 40 + 23 * i
        r = np.concatenate([t[:cut], rng.integers(1000, 90000, 50).astype(np.int32)])
        m = np.zeros(len(r), np.uint8)
        if i == 5:
            m[70] = 1                                  # a sensitive token inside the shared prefix
        readers.append(Batch(tokens=r, offsets=np.array([0, len(r)], np.int64), mask=m,
                             writer_ids=np.array([100 + i], np.int64)))
    wl = Workload("prefix_partial", g, [(pack_batches(writers), pack_batches(readers))],
                  pool_capacity_tokens=100000, max_span_len=512)
    case = Case(wl, policy="prefix_only")
    res = run_round_parity(case, score=False)
    _assert(res)
    assert res["hits"] == 6 and res["partial_hits"] >= 5


def _straddle_round(seed, pairs=32):
    """S:L401 / S:L645: shared spans straddling a 128-token chunk boundary, shifted by 1-64 tokens
    between writer and reader; the writer's text outside the span is private (masked)."""
    rng = np.random.default_rng(seed)
    writers, readers = [], []
    for i in range(pairs):
        shift, span_len, pos = int(rng.integers(1, 65)), int(rng.integers(160, 320)), int(rng.integers(0, 128))
        n = pos + shift + span_len + 64
        span = rng.integers(0, VOCAB, span_len).astype(np.int32)
        wt = rng.integers(0, VOCAB, n).astype(np.int32)
        wt[pos:pos + span_len] = span
        wm = np.ones(n, np.uint8)
        wm[pos:pos + span_len] = 0
        rt = rng.integers(0, VOCAB, n).astype(np.int32)
        rt[pos + shift:pos + shift + span_len] = span
        writers.append(Batch(tokens=wt, offsets=np.array([0, n], np.int64), mask=wm,
                             writer_ids=np.array([i], np.int64), span_req=np.zeros(1, np.int32),
                             span_begin=np.array([pos], np.int32), span_len=np.array([span_len], np.int32)))
        readers.append(Batch(tokens=rt, offsets=np.array([0, n], np.int64), mask=np.zeros(n, np.uint8),
                             writer_ids=np.array([1000 + i], np.int64)))
    return pack_batches(writers), pack_batches(readers)


def test_granularity_gap_direction_on_device():
    g = Geometry(2, 2, 64, "bf16", 500000.0)
    wb, rb = _straddle_round(645)
    cov = {}
    for policy in (None, "fixed_chunk"):
        wl = Workload("straddle", g, [(wb, rb)], pool_capacity_tokens=1 << 20, max_span_len=1024)
        case = Case(wl, policy=policy)
        res = run_round_parity(case, score=False)
        _assert(res)
        h = case.dev  # per-request coverage from the last match, through the C-ABI
        db = case._dev_batch(rb)
        hits = h.match_spans(db, 99, no_touch=True, policy=policy)
        cov[policy] = hits.req_covered.cpu().numpy()[:rb.num_reqs]
    sel, fix = cov[None], cov["fixed_chunk"]
    assert np.all(sel > fix) and np.all(fix == 0)
