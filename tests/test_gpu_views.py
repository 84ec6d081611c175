"""Pool views (cp_index_create_view, cp_index_copy_in, CP_REUSE_WORKLIST): the rectangles of one rank of
the load-balanced layout (paper_2605_23640_b200.shard.make_layout 'balanced') served by one index's
metadata.  Composition pin: every rectangle's pool and gathered K/V rows are exactly (bit for bit)
the matching slice of the one-index run over the full geometry, which test_gpu_parity checks against
the oracle; hits / plans come from the base alone.  Also the contract's refusals."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from synth.gen import make_workload  # noqa: E402
from tests.harness import SENTINEL, Case  # noqa: E402


def _slice_kv(cp, kv, l0, l1, h0, h1):
    return cp.PagedKV([t[:, :, h0:h1].contiguous() for t in kv.k[l0:l1]],
                      [t[:, :, h0:h1].contiguous() for t in kv.v[l0:l1]], kv.block_tables)


def _rows(kv, bt, lens):
    out = []
    for r, n in enumerate(lens):
        q = np.arange(int(n))
        blk = torch.from_numpy(bt[r, q // 16].astype(np.int64)).cuda()
        sl = torch.from_numpy((q % 16).astype(np.int64)).cuda()
        out.append((torch.stack([k[blk, sl] for k in kv.k]), torch.stack([v[blk, sl] for v in kv.v])))
    return out


@pytest.mark.parametrize("rank,world", [(3, 8), (1, 4), (7, 8)])
def test_balanced_rank_views_equal_slices_of_the_full_index(rank, world):
    import paper_2605_23640_b200 as cp
    from paper_2605_23640_b200 import _lib as L
    from paper_2605_23640_b200.shard import make_layout
    wl = make_workload(2, scale=0.05)
    wb, rb = wl.rounds[0]
    g = wl.geometry
    full = Case(wl, seed=5)
    rects = make_layout(rank, world, g.num_layers, g.num_kv_heads, "balanced", owner_extra_units=6.0)
    assert len(rects) >= 2
    bits = [np.arange(int(m)) % 4 == 0 for m in wb.span_len]
    wkv = full.writer_kv(wb)
    # one-index reference run with the same writer KV and destination block tables
    from oracle.oracle import pack_bits
    words, offs = pack_bits(bits)
    dwords = torch.from_numpy(words.view(np.int32).copy()).cuda()
    doffs = torch.from_numpy(offs.astype(np.int64)).cuda()
    sp = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()
    spans = (sp(wb.span_req), sp(wb.span_begin), sp(wb.span_len))
    db = full._dev_batch(wb)
    ref = cp.KVIndex(full.cfg)
    ref.insert(db, wkv, *spans, dwords, doffs, 1)
    import dataclasses
    r0 = rects[0]
    base = cp.KVIndex(dataclasses.replace(full.cfg, num_layers=r0.num_layers, num_kv_heads=r0.num_heads,
                                          layer_offset=r0.layer_lo, head_offset=r0.head_lo))
    views = [base.view(r.num_layers, r.num_heads, r.layer_lo, r.head_lo) for r in rects[1:]]
    base.insert(db, _slice_kv(cp, wkv, r0.layer_lo, r0.layer_hi, r0.head_lo, r0.head_hi), *spans, dwords, doffs, 1)
    for v, r in zip(views, rects[1:]):
        v.copy_in(db, _slice_kv(cp, wkv, r.layer_lo, r.layer_hi, r.head_lo, r.head_hi), reuse_worklist=True)
    assert ref.last_error() == 0 and base.last_error() == 0
    # pools: each rectangle's pool is the slice of the full pool (same page ids: shared metadata)
    fk, fv = ref.pool_views()
    snap = ref.snapshot(with_tokens=False)
    assert [e["pages"].tolist() for e in snap["entries"]] == \
        [e["pages"].tolist() for e in base.snapshot(with_tokens=False)["entries"]]
    # the rows the entries hold (t < len; the rest of the pool is uninitialised)
    pg = np.concatenate([e["pages"][np.arange(e["len"]) // 16] for e in snap["entries"]]).astype(np.int64)
    sl = np.concatenate([np.arange(e["len"]) % 16 for e in snap["entries"]]).astype(np.int64)
    pg, sl = torch.from_numpy(pg).cuda(), torch.from_numpy(sl).cuda()
    for ix, r in zip([base] + views, rects):
        k, v = ix.pool_views()
        assert torch.equal(k[:, pg, sl].view(torch.int16),
                           fk[r.layer_lo:r.layer_hi][:, pg, sl][:, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
        assert torch.equal(v[:, pg, sl].view(torch.int16),
                           fv[r.layer_lo:r.layer_hi][:, pg, sl][:, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
    # match once on the base; gather base + views with the reused work list
    rdb = full._dev_batch(rb)
    fh = ref.match_spans(rdb, 50)
    bh = base.match_spans(rdb, 50)
    for key in ("num_hits", "hit_entry", "hit_dst", "hit_len", "hit_delta", "plan", "req_covered"):
        assert np.array_equal(fh.to_host()[key], bh.to_host()[key]), key
    fdst = full.dst_kv(rb)
    ref.gather_rerotate(rdb, fh, fdst)
    dsts = []
    for i, (ix, r) in enumerate(zip([base] + views, rects)):
        d = _slice_kv(cp, fdst, r.layer_lo, r.layer_hi, r.head_lo, r.head_hi)
        for t in d.k + d.v:
            t.fill_(5.0)
        ix.gather_rerotate(rdb, bh, d, reuse_worklist=i > 0)
        dsts.append(d)
    assert base.last_error() == 0
    bt = fdst.block_tables.cpu().numpy()
    frows = _rows(fdst, bt, rb.lens)
    for d, r in zip(dsts, rects):
        for (fk_, fv_), (sk, sv) in zip(frows, _rows(d, bt, rb.lens)):
            assert torch.equal(sk.view(torch.int16), fk_[r.layer_lo:r.layer_hi, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
            assert torch.equal(sv.view(torch.int16), fv_[r.layer_lo:r.layer_hi, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
    # refusals: a view neither matches nor inserts; a reused list needs the same buffers, no match since
    with pytest.raises(L.CacheHitError):
        views[0].match_spans(rdb, 51)
    with pytest.raises(L.CacheHitError):
        views[0].insert(db, wkv, *spans, dwords, doffs, 2)
    base.match_spans(rdb, 52, hits=bh, no_touch=True)
    with pytest.raises(L.CacheHitError):
        views[0].gather_rerotate(rdb, bh, dsts[1], reuse_worklist=True)     # a match ran since
    base.gather_rerotate(rdb, bh, dsts[0])
    other = cp.PagedKV(dsts[1].k, dsts[1].v, dsts[1].block_tables.clone())
    with pytest.raises(L.CacheHitError):
        views[0].gather_rerotate(rdb, bh, other, reuse_worklist=True)       # a different block table
    views[0].gather_rerotate(rdb, bh, dsts[1], reuse_worklist=True)
    assert base.last_error() == 0
    # every rectangle in ONE launch (cp_gather_rerotate_rects): the same rows, bit for bit, with both
    # placeholder modes
    for zu in (False, True):
        ref.gather_rerotate(rdb, fh, fdst, zero_uncovered=zu)
        frows = _rows(fdst, bt, rb.lens)
        d2 = []
        for r in rects:
            d = _slice_kv(cp, fdst, r.layer_lo, r.layer_hi, r.head_lo, r.head_hi)
            d2.append(d)                             # sentinel-filled like fdst: rows no gather writes compare equal
            for t in d.k + d.v:
                t.fill_(SENTINEL)
        base.gather_rerotate_rects(views, rdb, bh, d2, zero_uncovered=zu)
        assert base.last_error() == 0
        for d, r in zip(d2, rects):
            for (fk_, fv_), (sk, sv) in zip(frows, _rows(d, bt, rb.lens)):
                assert torch.equal(sk.view(torch.int16), fk_[r.layer_lo:r.layer_hi, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
                assert torch.equal(sv.view(torch.int16), fv_[r.layer_lo:r.layer_hi, :, r.head_lo:r.head_hi].contiguous().view(torch.int16))
    # refusals: a destination on another block table; a view passed as the base
    with pytest.raises(L.CacheHitError):
        base.gather_rerotate_rects(views, rdb, bh, [d2[0], other] + d2[2:])
    with pytest.raises(L.CacheHitError):
        views[0].gather_rerotate_rects([], rdb, bh, [d2[1]])
    assert base.last_error() == 0
