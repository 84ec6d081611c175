"""GPU parity: CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bars (north star): bit exact for hashes, entry tables, page lists, hits, plan codes, recompute
bits and gathered V; re-rotated K within max-abs 2e-2 (bf16) or 1e-5 relative (fp32).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle.oracle as O  # noqa: E402
from synth.gen import Batch, Geometry, make_workload, pack_batches  # noqa: E402
from tests.harness import Case, ParityReport, run_round_parity  # noqa: E402


def _assert(res):
    assert res["ok"], res["notes"]


def test_toy_config1_all_rounds():
    case = Case(make_workload(1))
    res = run_round_parity(case)
    _assert(res)
    assert res["moved_hits"] > 0 and res["covered"] > 0


def test_l2_persist_window_changes_no_result():
    """cp_index_l2_persist only sets a cache policy: the rounds with the metadata window on the stream give
    the oracle's results; a hit ratio outside [0, 1] is refused; 0 clears the window."""
    from paper_2605_23640_b200 import _lib as L
    case = Case(make_workload(1))
    st = torch.cuda.current_stream()
    case.dev.l2_persist(st, 1.0)
    with pytest.raises(L.CacheHitError):
        case.dev.l2_persist(st, 1.5)
    res = run_round_parity(case)
    case.dev.l2_persist(st, 0.0)
    _assert(res)
    assert res["covered"] > 0


def test_toy_gptj_and_no_reader_mask():
    wl = make_workload(1, seed=11)
    wl.geometry.rope_style = "gptj"
    case = Case(wl, use_reader_mask=False)
    _assert(run_round_parity(case))


def test_msmarco_config2_reduced():
    case = Case(make_workload(2, scale=0.125), sample_reqs=4, sample_layers=[0, 17, 31])
    res = run_round_parity(case, score=True)
    _assert(res)
    assert res["covered"] / res["tokens"] > 0.9


def test_msmarco_config2_full_size_every_request():
    """Config 2 at its full size in the bench's launch configuration: every request's K and V rows of
    the last layer (393K tokens, moved and unmoved hits, zero placeholders) against the oracle."""
    case = Case(make_workload(2), sample_reqs=None, sample_layers=[31])
    wb, rb = case.wl.rounds[0]
    rep = ParityReport()
    case.insert(wb, rep)
    case.score_parity(wb, rep, max_spans=24)
    case.match_and_gather(rb, rep, check_kv=True)
    assert rep.ok, rep.notes[:10]


def test_multidoc_config3_reduced():
    wl = make_workload(3, scale=0.08)
    case = Case(wl, sample_reqs=3, sample_layers=[0, 31])
    rep = ParityReport()
    wb, rb = wl.rounds[0]
    case.insert(wb, rep, sparse_kv=True)
    case.match_and_gather(rb, rep)
    assert rep.ok, rep.notes[:10]
    assert rep.stats["moved_hits"] > 0


def test_70b_layer_shard_config4_reduced():
    """Config 4 geometry (80 layers), one layer shard of 10 layers as one rank holds it."""
    wl = make_workload(4, scale=0.05)
    case = Case(wl, layer_range=(70, 80), sample_reqs=2, sample_layers=[0, 9])
    rep = ParityReport()
    wb, rb = wl.rounds[0]
    case.insert(wb, rep, sparse_kv=True)
    case.match_and_gather(rb, rep)
    assert rep.ok, rep.notes[:10]


def test_70b_head_shard():
    wl = make_workload(4, scale=0.03)
    case = Case(wl, layer_range=(0, 4), head_range=(3, 4), sample_reqs=2)
    rep = ParityReport()
    wb, rb = wl.rounds[0]
    case.insert(wb, rep, sparse_kv=True)
    case.match_and_gather(rb, rep)
    assert rep.ok, rep.notes[:10]


@pytest.mark.parametrize("h0,h1", [(0, 3), (2, 8), (1, 6), (4, 5)])
def test_head_ranges_of_the_balanced_layout_config3(h0, h1):
    """The balanced layout's partial-layer rectangles hold 1-7 KV heads: 3, 5 and 6 heads give 24, 40 and
    48 column tasks per token row, which do not divide the 256-thread CTA (the copy kernel then runs on
    its first 240 threads with a fixed column per thread).  Config 3 (moved hits: re-rotated K)."""
    wl = make_workload(3, scale=0.05)
    case = Case(wl, layer_range=(30, 32), head_range=(h0, h1), sample_reqs=3)
    rep = ParityReport()
    wb, rb = wl.rounds[0]
    case.insert(wb, rep, sparse_kv=True)
    case.match_and_gather(rb, rep)
    assert rep.ok, rep.notes[:10]
    assert rep.stats["moved_hits"] > 0


def test_churn_config5_reduced_with_eviction():
    """Config 5 shape with a small token budget so LRU eviction, duplicates and supersedes happen."""
    wl = make_workload(5, scale=0.02)          # 1 batch... scale rounds up below
    from synth.gen import churn_workload
    wl = churn_workload(batches=4, per_batch=24, corpus=60, capacity_tokens=9000,
                        geometry=Geometry(2, 2, 64, "bf16", 500000.0))
    case = Case(wl, sample_reqs=3)
    rep = ParityReport()
    for wb, rb in wl.rounds:
        case.match_and_gather(rb, rep)
        case.insert(wb, rep)
    assert rep.ok, rep.notes[:10]
    assert rep.stats["duplicate"] > 0


def test_supersede_and_contained():
    g = Geometry(1, 1, 16, "fp32", 10000.0, window_len=8)
    rng = np.random.default_rng(0)
    base = rng.integers(1000, 2000, 400).astype(np.int32)

    def wb(begin, end, wid):
        t = base[begin:end]
        return Batch(tokens=t.copy(), offsets=np.array([0, len(t)], np.int64), mask=np.zeros(len(t), np.uint8),
                     writer_ids=np.array([wid], np.int64), span_req=np.zeros(1, np.int32),
                     span_begin=np.zeros(1, np.int32), span_len=np.array([len(t)], np.int32))
    from synth.gen import Workload
    rounds = [(wb(50, 150, 0), wb(0, 300, 100)), (wb(0, 300, 1), wb(0, 300, 101)),
              (wb(60, 120, 2), wb(0, 300, 102)), (wb(0, 300, 3), wb(0, 300, 103))]
    wl = Workload("edge", g, rounds, pool_capacity_tokens=10000, max_span_len=512)
    case = Case(wl)
    res = run_round_parity(case, score=False)
    _assert(res)


def test_errors_have_no_side_effects():
    case = Case(make_workload(1))
    wb, rb = case.wl.rounds[0]
    rep = ParityReport()
    case.insert(wb, rep)
    before = case.dev.snapshot()
    bad = Batch(tokens=wb.tokens, offsets=wb.offsets, mask=wb.mask, writer_ids=wb.writer_ids,
                span_req=np.array([0, 0], np.int32), span_begin=np.array([0, 120], np.int32),
                span_len=np.array([128, 20], np.int32))
    case.insert(bad, rep)                      # span 1 covers PII1 -> CP_ERR_SENSITIVE_SPAN on both sides
    after = case.dev.snapshot()
    assert rep.ok, rep.notes
    assert [e["id"] for e in after["entries"]] == [e["id"] for e in before["entries"]]
    assert after["fifo_count"] == before["fifo_count"] and after["next_id"] == before["next_id"]


def test_empty_short_and_max_requests():
    g = Geometry(2, 1, 32, "bf16", 500000.0)
    rng = np.random.default_rng(5)
    long_req = rng.integers(1000, 50000, 10240).astype(np.int32)
    w = Batch(tokens=long_req[3000:5000].copy(), offsets=np.array([0, 2000], np.int64),
              mask=np.zeros(2000, np.uint8), writer_ids=np.array([0], np.int64),
              span_req=np.zeros(1, np.int32), span_begin=np.zeros(1, np.int32), span_len=np.array([2000], np.int32))
    parts = [Batch(tokens=np.zeros(0, np.int32), offsets=np.array([0, 0], np.int64), mask=np.zeros(0, np.uint8),
                   writer_ids=np.array([1], np.int64)),
             Batch(tokens=long_req[3000:3100].copy(), offsets=np.array([0, 100], np.int64),
                   mask=np.zeros(100, np.uint8), writer_ids=np.array([2], np.int64)),
             Batch(tokens=long_req, offsets=np.array([0, 10240], np.int64), mask=np.zeros(10240, np.uint8),
                   writer_ids=np.array([3], np.int64))]
    from synth.gen import Workload
    wl = Workload("edge2", g, [(w, pack_batches(parts))], pool_capacity_tokens=100000, max_span_len=2048)
    case = Case(wl)
    res = run_round_parity(case, score=False)
    _assert(res)
    assert res["hits"] == 1


def test_identical_unmasked_prompt_is_prefix_reuse():
    g = Geometry(2, 2, 64, "bf16", 500000.0)
    rng = np.random.default_rng(7)
    p = rng.integers(1000, 100000, 700).astype(np.int32)
    mk = lambda wid, spans: Batch(tokens=p.copy(), offsets=np.array([0, 700], np.int64), mask=np.zeros(700, np.uint8),
                                  writer_ids=np.array([wid], np.int64), span_req=np.zeros(len(spans), np.int32),
                                  span_begin=np.array([s[0] for s in spans], np.int32),
                                  span_len=np.array([s[1] for s in spans], np.int32))
    from synth.gen import Workload
    wl = Workload("prefix", g, [(mk(0, [(0, 700)]), mk(1, []))], pool_capacity_tokens=10000, max_span_len=1024)
    case = Case(wl, rho=(0, 4))
    rep = ParityReport()
    case.insert(wl.rounds[0][0], rep)
    case.match_and_gather(wl.rounds[0][1], rep)
    assert rep.ok, rep.notes
    assert rep.stats["hits"] == 1 and rep.stats["covered"] == 700 and rep.stats["moved_hits"] == 0


def test_hash_prefix_matches_oracle():
    import paper_2605_23640_b200 as cp
    rng = np.random.default_rng(3)
    lens = [0, 1, 5, 300, 8192, 9000]
    toks = [rng.integers(0, 128256, n).astype(np.int32) for n in lens]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    db = cp.DeviceBatch.from_numpy(np.concatenate(toks), offs, None)
    out = cp.hash_prefix(db, 42).cpu().numpy().view(np.uint64)
    B = O.hash_base(42)
    for r, t in enumerate(toks):
        exp = O.prefix_hashes(t, B)
        got = out[offs[r] + r: offs[r] + r + lens[r] + 1]
        assert np.array_equal(got, exp), r


def test_determinism_two_runs():
    outs = []
    for _ in range(2):
        case = Case(make_workload(2, scale=0.05), sample_reqs=1, sample_layers=[0])
        rep = ParityReport()
        wb, rb = case.wl.rounds[0]
        case.insert(wb, rep)
        db = case._dev_batch(rb)
        hits = case.dev.match_spans(db, 99)
        outs.append((case.dev.snapshot(), hits.to_host()))
    (s0, h0), (s1, h1) = outs
    assert [e["pages"].tolist() for e in s0["entries"]] == [e["pages"].tolist() for e in s1["entries"]]
    for k in ("hit_entry", "hit_dst", "hit_delta", "plan"):
        assert np.array_equal(h0[k], h1[k])


def test_score_edge_cases():
    import paper_2605_23640_b200 as cp
    rng = np.random.default_rng(1)
    mats, ns, ls, rs = [], [], [], []
    for n, l, r in [(1, 0, 0), (5, 0, 4), (33, 1, 32), (257, 100, 256), (1000, 3, 999), (130, 0, 129)]:
        A = np.tril(rng.uniform(0, 1, (n, n))).astype(np.float32)
        A /= A.sum(1, keepdims=True)
        mats.append(torch.from_numpy(A).cuda()); ns.append(n); ls.append(l); rs.append(r)
    A = np.eye(64, dtype=np.float32)                       # all-tie case
    mats.append(torch.from_numpy(A).cuda()); ns.append(64); ls.append(10); rs.append(39)
    for num, den in [(1, 4), (0, 4), (4, 4), (1, 10), (3, 7)]:
        sc, bits, so, bo = cp.score_deviation(mats, ns, [1] * len(ns), ls, rs, num, den)
        sc, bits = sc.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
        for q in range(len(ns)):
            m = rs[q] - ls[q] + 1
            osc, ob = O.score(mats[q].cpu().numpy(), ls[q], rs[q], num, den)
            assert np.array_equal(sc[so[q]:so[q] + m], osc)
            assert np.array_equal(bits[bo[q]:bo[q] + (m + 31) // 32], ob), (q, num, den)


def test_score_multihead_long_misaligned_rows():
    """Rows longer than one load batch (> 8 x 32 x 4 floats), odd n (rows not 16-B aligned), l* not
    a multiple of 4, several heads, non-row-stochastic attention (R#27), several spans per launch."""
    import paper_2605_23640_b200 as cp
    rng = np.random.default_rng(7)
    mats, ns, hs, ls, rs = [], [], [], [], []
    for n, h, l, r in [(2051, 2, 777, 2050), (4099, 1, 1234, 4098), (1027, 3, 1, 1026), (1536, 1, 161, 1535),
                       (4099, 1, 4097, 4098)]:
        A = np.tril(rng.uniform(0, 1.5, (h, n, n))).astype(np.float32)    # row sums != 1
        mats.append(torch.from_numpy(A).cuda()); ns.append(n); hs.append(h); ls.append(l); rs.append(r)
    for off in (1, 2, 3):                       # base pointer not 16-B aligned (a view into a larger buffer)
        n, l = 777 + off, 100 + off
        A = np.tril(rng.uniform(0, 1, (n, n))).astype(np.float32)
        flat = torch.zeros(n * n + 4, dtype=torch.float32, device="cuda")
        view = flat[off:off + n * n].view(n, n)
        view.copy_(torch.from_numpy(A))
        assert view.data_ptr() % 16 == 4 * off
        mats.append(view); ns.append(n); hs.append(1); ls.append(l); rs.append(n - 1)
    sc, bits, so, bo = cp.score_deviation(mats, ns, hs, ls, rs, 1, 4)
    sc, bits = sc.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
    for q in range(len(ns)):
        m = rs[q] - ls[q] + 1
        osc, ob = O.score(mats[q].cpu().numpy(), ls[q], rs[q], 1, 4)
        assert np.array_equal(sc[so[q]:so[q] + m], osc), q
        assert np.array_equal(bits[bo[q]:bo[q] + (m + 31) // 32], ob), q


def test_multidoc_config3_full_size_every_request():
    """Config 3 at full size (128 readers x ~4K, 512-passage pool, one GPU): all hits, plans and the
    index bit exact; every request's K and V rows of one layer (533K tokens, 88% moved hits)."""
    wl = make_workload(3)
    case = Case(wl, sample_reqs=None, sample_layers=[17])
    rep = ParityReport()
    wb, rb = wl.rounds[0]
    case.insert(wb, rep, sparse_kv=True)
    case.match_and_gather(rb, rep)
    assert rep.ok, rep.notes[:10]
    assert rep.stats["moved_hits"] > 0.8 * rep.stats["hits"]          # heavy re-rotation (system prompt: delta 0)


def test_70b_layer_shard_config4_full_size_sampled():
    """Config 4 at full size on one rank's layer shard (layers 70-79 of 80; 64 readers x 8K)."""
    wl = make_workload(4)
    case = Case(wl, layer_range=(70, 80), sample_reqs=2, sample_layers=[0, 9])
    rep = ParityReport()
    wb, rb = wl.rounds[0]
    case.insert(wb, rep, sparse_kv=True)
    case.match_and_gather(rb, rep)
    assert rep.ok, rep.notes[:10]


def _one(tokens, mask=None, spans=(), wid=0):
    t = np.asarray(tokens, np.int32)
    m = np.zeros(len(t), np.uint8) if mask is None else np.asarray(mask, np.uint8)
    return Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=m, writer_ids=np.array([wid], np.int64),
                 span_req=np.zeros(len(spans), np.int32), span_begin=np.array([s[0] for s in spans], np.int32),
                 span_len=np.array([s[1] for s in spans], np.int32))


def test_degenerate_masks_and_sizes():
    """All-sensitive writer (nothing insertable), zero-span insert, a max_span_len span, an all-masked
    reader (no hit may cover a masked token), a reader shorter than the window, a reader with no hits."""
    from synth.gen import Workload
    g = Geometry(2, 2, 64, "bf16", 500000.0)
    rng = np.random.default_rng(12)
    long_seg = rng.integers(1000, 90000, 1024).astype(np.int32)               # = max_span_len
    rounds = [
        (_one(rng.integers(1000, 90000, 300), mask=np.ones(300), wid=0),         # all sensitive, no spans
         _one(long_seg, wid=100)),
        (_one(long_seg, spans=[(0, 1024)], wid=1), _one(long_seg, mask=np.ones(1024), wid=101)),
        (_one(rng.integers(1000, 90000, 50), wid=2), _one(long_seg[:100], wid=102)),
        (_one(np.concatenate([long_seg[:10], long_seg]), spans=[(10, 1024)], wid=3),   # duplicate at another origin
         pack_batches([_one(np.concatenate([rng.integers(1000, 90000, 37), long_seg]), wid=103),
                       _one(rng.integers(1000, 90000, 700), wid=104)])),
    ]
    wl = Workload("degenerate", g, rounds, pool_capacity_tokens=5000, max_span_len=1024)
    res = run_round_parity(Case(wl), score=False)
    _assert(res)
    assert res["hits"] == 1                      # only round 3's first reader reuses the 1024-token entry


def test_zero_uncovered_flag_and_match_error():
    import paper_2605_23640_b200 as cp
    case = Case(make_workload(1))
    wb, rb = case.wl.rounds[0]
    rep = ParityReport()
    case.insert(wb, rep)
    db = case._dev_batch(rb)
    hits = case.dev.match_spans(db, 50)
    dst = case.dst_kv(rb)
    case.dev.gather_rerotate(db, hits, dst, zero_recompute=True, zero_uncovered=True)
    plan = hits.plan.cpu().numpy()[:rb.total_tokens]
    bt = dst.block_tables.cpu().numpy()
    q = np.nonzero(plan == 0)[0]
    assert len(q) > 0
    blk = torch.from_numpy(bt[0, q // 16].astype(np.int64)).cuda()
    slot = torch.from_numpy((q % 16).astype(np.int64)).cuda()
    for l in range(case.g.num_layers):
        assert float(dst.k[l][blk, slot].abs().max()) == 0.0 and float(dst.v[l][blk, slot].abs().max()) == 0.0
    assert case.dev.last_error() == 0
    # a request longer than max_req_tokens raises the sticky device error; later calls no-op
    case = Case(make_workload(2, scale=0.05), sample_reqs=1, sample_layers=[0])
    long = np.arange(1000, 1000 + case.cfg.max_req_tokens + 5, dtype=np.int32)
    bad = cp.DeviceBatch.from_numpy(long, np.array([0, len(long)], np.int64), None)
    bad.max_req_len = case.cfg.max_req_tokens
    case.dev.match_spans(bad, 51, use_mask=False)
    assert case.dev.last_error() == cp._lib.CP_ERR_INVALID_ARG
    assert case.dev.last_error() == 0            # cleared by the read


def test_churn_config5_full_size_oracle_parity():
    """Config 5 at its full batch size (256 requests x ~1.6K tokens per batch, 100K-passage Zipf
    corpus) on one KV-head shard, 6 batches under a 300K-token budget so that LRU eviction runs from
    the second insert on: insert outcomes / ids and the whole live index bit exact, hits / plans /
    stats bit exact, KV rows sampled (2 requests x 2 layers per batch)."""
    from synth.gen import churn_workload
    g = Geometry(32, 8, 128, "bf16", 500000.0)
    wl = churn_workload(batches=6, per_batch=256, corpus=100000, capacity_tokens=300_000, geometry=g)
    case = Case(wl, head_range=(0, 1), sample_reqs=2, sample_layers=[0, 31])
    rep = ParityReport()
    for wb, rb in wl.rounds:
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
    assert rep.stats["duplicate"] > 0 and rep.stats["hits"] > 0
    assert case.orc.num_ids > len(case.orc.live_entries())        # entries were evicted
    par, ser, why = case.dev.commit_stats()
    assert par >= 5, (par, ser, why)                    # the churn batches take the parallel commit


def test_churn_config5_full_batches_invariants():
    """Config 5 at its full batch size (256 requests x ~1.6K tokens, 100K-passage corpus) for a few
    batches on one head shard with a budget that forces LRU eviction; device-side invariants (the
    oracle parity of the same shape is test_churn_config5_full_size_oracle_parity): budget, no device
    error, every stored entry is unmasked in its writer and its tokens equal the writer's span, no
    entry strictly contains another."""
    import paper_2605_23640_b200 as cp
    from synth.gen import churn_workload
    g = Geometry(32, 8, 128, "bf16", 500000.0)
    wl = churn_workload(batches=4, per_batch=256, corpus=100000, capacity_tokens=400_000, geometry=g)
    case = Case(wl, head_range=(0, 1), sample_reqs=1, sample_layers=[0])
    for bi, (wb, rb) in enumerate(wl.rounds):
        db = case._dev_batch(rb)
        hits = case.dev.match_spans(db, 2 * bi + 1)
        nb = [(int(n) + 15) // 16 for n in wb.lens]
        bt = torch.zeros((wb.num_reqs, max(nb)), dtype=torch.int32)
        o = 0
        for r, k in enumerate(nb):
            bt[r, :k] = torch.arange(o, o + k); o += k
        kv = cp.PagedKV.allocate(32, o, 1, 128, torch.bfloat16, bt, "cuda", zero=True)
        sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda() for a in (wb.span_req, wb.span_begin, wb.span_len)]
        ids, oc = case.dev.insert(db, kv, *sp, None, None, 2 * bi + 2)
        assert case.dev.last_error() == 0
        del kv
    snap = case.dev.snapshot()
    assert snap["live_tokens"] <= 400_000 and snap["error"] == 0
    assert snap["next_id"] > snap["num_live"]           # evictions happened
    seqs = {}
    for wb, _ in wl.rounds:
        for s in range(len(wb.span_len)):
            r, b0, m = int(wb.span_req[s]), int(wb.span_begin[s]), int(wb.span_len[s])
            assert not wb.req_mask(r)[b0:b0 + m].any()
            seqs.setdefault(m, set()).add(wb.req_tokens(r)[b0:b0 + m].tobytes())
    strs = []
    for e in snap["entries"]:
        assert e["tokens"].tobytes() in seqs[e["len"]]   # privacy: stored tokens are an unmasked writer span
        strs.append("," + ",".join(map(str, e["tokens"].tolist())) + ",")
    for i in range(0, len(strs), 97):                     # containment-freedom (sampled pairs)
        for j in range(len(strs)):
            if i != j:
                assert strs[i] not in strs[j]


@pytest.mark.parametrize("cfg", [1, 5])
def test_split_insert_prepare_concurrent_with_match_and_gather(cfg):
    """cp_index_insert_prepare on a side stream while cp_match_spans + cp_gather_rerotate of the same
    index run on the main stream, then cp_index_insert_commit: outcomes, entry ids, the whole index
    and the hits must equal the oracle's sequential match-then-insert (the prepare reads the index and
    writes only insert scratch).  Config 5 shape with a small budget: evictions and supersedes."""
    if cfg == 1:
        wl = make_workload(1)
    else:
        from synth.gen import churn_workload
        wl = churn_workload(batches=5, per_batch=24, corpus=60, capacity_tokens=9000,
                            geometry=Geometry(2, 2, 64, "bf16", 500000.0))
    case = Case(wl, seed=11)
    rep = ParityReport()
    rng = np.random.default_rng(cfg)
    first_wb, _ = wl.rounds[0]
    case.insert(first_wb, rep)
    assert rep.ok, rep.notes
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    for k, (wb, rb) in enumerate(wl.rounds[1:]):
        flags = [rng.random(int(m)) < 0.25 for m in wb.span_len]
        words, offs = O.pack_bits(flags)
        kv = case.writer_kv(wb)
        db = case._dev_batch(wb)
        sp = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()
        spans = (sp(wb.span_req), sp(wb.span_begin), sp(wb.span_len))
        dwords = torch.from_numpy(words.view(np.int32).copy() if len(words) else np.zeros(1, np.int32)).cuda()
        doffs = torch.from_numpy(offs.astype(np.int64)).cuda()
        t_match, t_ins = case.t + 1, case.t + 2
        case.t += 2
        rdb = case._dev_batch(rb)
        dst = case.dst_kv(rb)
        ready = torch.cuda.Event()
        ready.record(main)
        side.wait_event(ready)
        with torch.cuda.stream(side):
            case.dev.insert(db, kv, *spans, dwords, doffs, t_ins, phase="prepare")
        hits = case.dev.match_spans(rdb, t_match)
        case.dev.gather_rerotate(rdb, hits, dst)
        main.wait_stream(side)
        ids, oc = case.dev.insert(db, kv, *spans, dwords, doffs, t_ins, phase="commit")
        assert case.dev.last_error() == 0
        res = case.orc.match(rb, t_match)
        rc, oids, ooc = case.orc.insert(wb, words, offs, t_ins)
        assert rc == 0
        h = hits.to_host()
        assert h["num_hits"] == res.num_hits
        for key in ("hit_entry", "hit_dst", "hit_len", "hit_delta"):
            assert np.array_equal(h[key], getattr(res, key)), key
        assert np.array_equal(oc.cpu().numpy(), ooc) and np.array_equal(ids.cpu().numpy(), oids)
        case.compare_index(rep, f"split insert round {k}")
        assert rep.ok, rep.notes


def test_split_insert_misuse_is_rejected_without_side_effects():
    import paper_2605_23640_b200 as cp
    case = Case(make_workload(1))
    wb, _ = case.wl.rounds[0]
    kv = case.writer_kv(wb)
    db = case._dev_batch(wb)
    sp = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()
    spans = (sp(wb.span_req), sp(wb.span_begin), sp(wb.span_len))
    before = case.dev.snapshot()
    with pytest.raises(cp._lib.CacheHitError):
        case.dev.insert(db, kv, *spans, t=1, phase="commit")             # commit without prepare
    case.dev.insert(db, kv, *spans, t=1, phase="prepare")
    with pytest.raises(cp._lib.CacheHitError):
        case.dev.insert(db, kv, *spans, t=1, phase="prepare")            # second prepare while pending
    with pytest.raises(cp._lib.CacheHitError):
        case.dev.insert(db, kv, *spans, t=1)                             # plain insert while pending
    after = case.dev.snapshot()
    assert after["next_id"] == before["next_id"] and after["num_live"] == before["num_live"]
    case.dev.insert(db, kv, *spans, t=1, phase="commit")
    assert case.dev.snapshot()["num_live"] > 0


@pytest.mark.parametrize("n_long", [10241, 30000, 65536])
def test_requests_longer_than_shared_memory(n_long):
    """Requests beyond the shared-memory matcher (max_req_tokens > 10240): the per-request arrays
    live in scratch; hits, plans, stats, the index and sampled KV rows still match the oracle,
    alongside short requests in the same batch."""
    g = Geometry(2, 1, 32, "bf16", 500000.0)
    rng = np.random.default_rng(n_long)
    base = rng.integers(1000, 50000, n_long).astype(np.int32)
    spans = [(0, 3000), (5000, 2047), (n_long - 2000, 2000)]
    w = Batch(tokens=base.copy(), offsets=np.array([0, n_long], np.int64), mask=np.zeros(n_long, np.uint8),
              writer_ids=np.array([0], np.int64), span_req=np.zeros(len(spans), np.int32),
              span_begin=np.array([s_[0] for s_ in spans], np.int32), span_len=np.array([s_[1] for s_ in spans], np.int32))
    shifted = np.concatenate([rng.integers(1000, 50000, 77).astype(np.int32), base])          # every hit moves
    parts = [Batch(tokens=shifted, offsets=np.array([0, len(shifted)], np.int64), mask=np.zeros(len(shifted), np.uint8),
                   writer_ids=np.array([1], np.int64)),
             Batch(tokens=base[5000:7047].copy(), offsets=np.array([0, 2047], np.int64), mask=np.zeros(2047, np.uint8),
                   writer_ids=np.array([2], np.int64)),
             Batch(tokens=base[:50].copy(), offsets=np.array([0, 50], np.int64), mask=np.zeros(50, np.uint8),
                   writer_ids=np.array([3], np.int64))]
    from synth.gen import Workload
    wl = Workload("long", g, [(w, pack_batches(parts))], pool_capacity_tokens=100000, max_span_len=4096)
    case = Case(wl, sample_reqs=2)
    res = run_round_parity(case, score=False)
    _assert(res)
    assert res["hits"] == 4 and res["moved_hits"] == 4


def test_layer_and_head_shards_concatenate_to_the_full_gather():
    """SURVEY §4 multi-GPU layer: each shard's index (layer ranges, head ranges) gathers exactly the
    slice of the one-index gather -- K (moved or not) and V bit for bit -- and the shards' hits,
    plans and index metadata equal the full index's (they replay the same inserts)."""
    wl = make_workload(2, scale=0.05)
    wb, rb = wl.rounds[0]

    def run(**kw):
        case = Case(wl, seed=5, **kw)
        rep = ParityReport()
        case.insert(wb, rep, bits_flags=[np.arange(int(m)) % 4 == 0 for m in wb.span_len])
        assert rep.ok, rep.notes
        db = case._dev_batch(rb)
        hits = case.dev.match_spans(db, 50)
        dst = case.dst_kv(rb)
        case.dev.gather_rerotate(db, hits, dst)
        bt = dst.block_tables.cpu().numpy()
        rows = []
        for r in range(rb.num_reqs):
            q = np.arange(int(rb.lens[r]))
            blk = torch.from_numpy(bt[r, q // 16].astype(np.int64)).cuda()
            sl = torch.from_numpy((q % 16).astype(np.int64)).cuda()
            rows.append((torch.stack([k[blk, sl] for k in dst.k]).cpu(), torch.stack([v[blk, sl] for v in dst.v]).cpu()))
        h = hits.to_host()
        return rows, {k: h[k] for k in ("hit_entry", "hit_dst", "hit_len", "hit_delta", "plan")}

    full_rows, full_hits = run()
    for kw, sel in [(dict(layer_range=(0, 13)), (slice(0, 13), slice(None))),
                    (dict(layer_range=(13, 32)), (slice(13, 32), slice(None))),
                    (dict(head_range=(0, 3)), (slice(None), slice(0, 3))),
                    (dict(head_range=(3, 8)), (slice(None), slice(3, 8)))]:
        rows, hits = run(**kw)
        for key in full_hits:
            assert np.array_equal(hits[key], full_hits[key]), (kw, key)
        for (fk, fv), (sk, sv) in zip(full_rows, rows):
            ls, hsl = sel
            assert torch.equal(sk.view(torch.int16), fk[ls, :, hsl].contiguous().view(torch.int16)), kw
            assert torch.equal(sv.view(torch.int16), fv[ls, :, hsl].contiguous().view(torch.int16)), kw


@pytest.mark.parametrize("placeholders", ["both", "none"])
def test_placeholder_modes_config2_every_request(placeholders):
    """R#14 at full config-2 size, every request, one layer: 'both' = the paper-literal zero placeholders
    (recompute-marked AND unmatched rows +0.0; the unmatched ones through the compacted uncovered list),
    'none' = CP_SKIP_RECOMPUTE (recompute-marked rows left untouched, unmatched rows untouched)."""
    case = Case(make_workload(2), sample_reqs=None, sample_layers=[5], placeholders=placeholders)
    wb, rb = case.wl.rounds[0]
    rep = ParityReport()
    case.insert(wb, rep)
    case.match_and_gather(rb, rep, check_kv=True)
    assert rep.ok, rep.notes[:10]
