"""A balanced-layout rank (one index + pool views) under the config-5 churn shape: every
batch is matched, gathered into every rectangle in ONE launch (cp_gather_rerotate_rects, placeholders
for recompute-marked and unmatched rows) and then inserted under a small LRU budget (stores, evictions,
copy-in into the base and every view -- alternately by cp_index_insert_commit_rects in one launch and
by cp_index_copy_in per view).  Composition pin: after every batch the rank's hits equal a
one-index run's over the full geometry, and every rectangle's gathered K/V rows and pool rows are the
slices of that run's, bit for bit."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from synth.gen import Geometry, churn_workload  # noqa: E402
from tests.harness import SENTINEL, Case  # noqa: E402
from tests.test_gpu_views import _rows, _slice_kv  # noqa: E402


@pytest.mark.parametrize("rank,world", [(1, 3), (2, 5), (2, 3)])
def test_balanced_rank_under_churn_equals_one_index(rank, world):
    import paper_2605_23640_b200 as cp
    from oracle.oracle import pack_bits
    from paper_2605_23640_b200.shard import make_layout
    g = Geometry(4, 4, 64, "bf16", 500000.0)
    wl = churn_workload(seed=11 + rank, batches=5, per_batch=16, corpus=400, capacity_tokens=5000, geometry=g)
    full = Case(wl, seed=rank)
    rects = make_layout(rank, world, g.num_layers, g.num_kv_heads, "balanced", owner_extra_units=1.0)
    assert len(rects) >= 2
    ref = cp.KVIndex(full.cfg)
    r0 = rects[0]
    base = cp.KVIndex(dataclasses.replace(full.cfg, num_layers=r0.num_layers, num_kv_heads=r0.num_heads,
                                          layer_offset=r0.layer_lo, head_offset=r0.head_lo))
    views = [base.view(r.num_layers, r.num_heads, r.layer_lo, r.head_lo) for r in rects[1:]]
    rng = np.random.default_rng(rank)
    sp = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()
    t = 0
    for wb, rb in wl.rounds:
        # ---- match + gather
        t += 1
        rdb = full._dev_batch(rb)
        fh, bh = ref.match_spans(rdb, t), base.match_spans(rdb, t)
        fhh, bhh = fh.to_host(), bh.to_host()
        for key in ("num_hits", "hit_entry", "hit_dst", "hit_len", "hit_delta", "plan", "req_covered"):
            assert np.array_equal(fhh[key], bhh[key]), key
        fdst = full.dst_kv(rb)
        ref.gather_rerotate(rdb, fh, fdst, zero_uncovered=True)
        d2 = []
        for r in rects:
            d = _slice_kv(cp, fdst, r.layer_lo, r.layer_hi, r.head_lo, r.head_hi)
            for x in d.k + d.v:
                x.fill_(SENTINEL)
            d2.append(d)
        base.gather_rerotate_rects(views, rdb, bh, d2, zero_uncovered=True)
        bt = fdst.block_tables.cpu().numpy()
        frows = _rows(fdst, bt, rb.lens)
        for d, r in zip(d2, rects):
            for (fk, fv), (sk, sv) in zip(frows, _rows(d, bt, rb.lens)):
                assert torch.equal(sk.view(torch.int16), fk[r.layer_lo:r.layer_hi, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
                assert torch.equal(sv.view(torch.int16), fv[r.layer_lo:r.layer_hi, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
        # ---- insert: the same batch as writers (stores, duplicates, LRU evictions)
        t += 1
        bits = [rng.random(int(m)) < 0.25 for m in wb.span_len]
        words, offs = pack_bits(bits)
        dwords = torch.from_numpy(words.view(np.int32).copy() if len(words) else np.zeros(1, np.int32)).cuda()
        doffs = torch.from_numpy(offs.astype(np.int64)).cuda()
        spans = (sp(wb.span_req), sp(wb.span_begin), sp(wb.span_len))
        db = full._dev_batch(wb)
        wkv = full.writer_kv(wb)
        ref.insert(db, wkv, *spans, dwords, doffs, t)
        wkvs = [_slice_kv(cp, wkv, r.layer_lo, r.layer_hi, r.head_lo, r.head_hi) for r in rects]
        for x in wkvs[1:]:
            x.block_tables = wkvs[0].block_tables               # one block table object for the rects calls
        if t % 4 == 0:                                          # commit + copy-in of every rectangle in one launch
            base.insert(db, wkvs[0], *spans, dwords, doffs, t, phase="prepare")
            base.insert_commit_rects(views, db, wkvs, *spans, dwords, doffs, t)
        else:                                                   # insert, then each view's share of the copy-in
            base.insert(db, wkvs[0], *spans, dwords, doffs, t)
            for v, x in zip(views, wkvs[1:]):
                v.copy_in(db, x, reuse_worklist=True)
        assert ref.last_error() == 0 and base.last_error() == 0
        fs, bs = ref.snapshot(with_tokens=False), base.snapshot(with_tokens=False)
        assert [(e["id"], e["pages"].tolist(), e["last_used"]) for e in fs["entries"]] == \
            [(e["id"], e["pages"].tolist(), e["last_used"]) for e in bs["entries"]]
        # pools: each rectangle's rows of the live entries are the full pool's slice
        pg = np.concatenate([e["pages"][np.arange(e["len"]) // 16] for e in fs["entries"]]).astype(np.int64)
        sl = np.concatenate([np.arange(e["len"]) % 16 for e in fs["entries"]]).astype(np.int64)
        pg, sl = torch.from_numpy(pg).cuda(), torch.from_numpy(sl).cuda()
        fk, fv = ref.pool_views()
        for ix, r in zip([base] + views, rects):
            k, v = ix.pool_views()
            assert torch.equal(k[:, pg, sl].view(torch.int16),
                               fk[r.layer_lo:r.layer_hi][:, pg, sl][:, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
            assert torch.equal(v[:, pg, sl].view(torch.int16),
                               fv[r.layer_lo:r.layer_hi][:, pg, sl][:, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
    fs = ref.snapshot(with_tokens=False)
    assert int(fs["next_id"]) > fs["num_live"] + 10          # LRU evictions happened
