"""Capacity and bounds guards of the C-ABI (include/cacheprune.h error contract): a call that fails on
the device changes nothing -- no index state, no destination row, no other request's blocks.

  * gather with a block table narrower than a covered position -> CP_ERR_INVALID_ARG, no row written
  * insert whose span reaches past the writer's block table     -> CP_ERR_INVALID_ARG, index unchanged
  * a span strictly containing more than 1024 live segments     -> CP_ERR_CAPACITY, index unchanged
  * overlapping spans whose copy-in list exceeds the chunk list  -> CP_ERR_CAPACITY, index unchanged
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


class _NS:
    pass


def _cp():
    import paper_2605_23640_b200 as cp
    from paper_2605_23640_b200 import _lib as L
    ns = _NS()
    for k in dir(cp):
        setattr(ns, k, getattr(cp, k))
    for k in dir(L):
        if k.startswith("CP_"):
            setattr(ns, k, getattr(L, k))
    return ns


def _index(cp, **kw):
    base = dict(num_layers=2, num_kv_heads=1, head_dim=64, dtype="bf16", window_len=4,
                pool_capacity_tokens=1 << 16, max_entries=4096, max_span_len=8192, max_req_tokens=8192,
                max_batch_reqs=4, max_batch_tokens=8192, max_spans_per_insert=2048)
    base.update(kw)
    return cp.KVIndex(cp.IndexConfig(**base))


def _kv(cp, idx, n_tokens, max_blocks=None):
    nb = (n_tokens + 15) // 16
    mb = nb if max_blocks is None else max_blocks
    bt = torch.arange(mb, dtype=torch.int32).view(1, mb)
    kv = cp.PagedKV.allocate(idx.cfg.num_layers, max(nb, mb) + 1, idx.cfg.num_kv_heads, idx.cfg.head_dim,
                             torch.bfloat16, bt)
    for t in kv.k + kv.v:
        t.normal_()
    return kv


def _sp(xs):
    return torch.tensor(xs, dtype=torch.int32, device="cuda")


def _state(idx):
    s = idx.snapshot(with_tokens=False)
    return (s["num_live"], s["next_id"], s["live_tokens"], s["fifo_count"], tuple(s["fifo"]),
            tuple((e["id"], e["len"], e["last_used"], tuple(e["pages"])) for e in s["entries"]))


def test_gather_rejects_narrow_block_table_and_writes_nothing():
    cp = _cp()
    idx = _index(cp)
    toks = np.arange(100, 164, dtype=np.int32)                     # 64 tokens, 4 blocks
    wb = cp.DeviceBatch.from_numpy(toks, np.array([0, 64], np.int64), np.zeros(64, np.uint8))
    idx.insert(wb, _kv(cp, idx, 64), _sp([0]), _sp([0]), _sp([64]), t=1)
    assert idx.last_error() == 0
    rb = cp.DeviceBatch.from_numpy(toks, np.array([0, 64], np.int64), None)
    hits = idx.match_spans(rb, t=2)
    assert int(hits.num_hits.item()) == 1
    dst = _kv(cp, idx, 64, max_blocks=2)                             # covers 32 of the 64 positions
    before = [t.clone() for t in dst.k + dst.v]
    idx.gather_rerotate(rb, hits, dst)
    assert idx.last_error() == cp.CP_ERR_INVALID_ARG
    for a, b in zip(before, dst.k + dst.v):
        assert torch.equal(a, b), "a rejected gather wrote rows"


def test_insert_rejects_span_past_writer_block_table():
    cp = _cp()
    idx = _index(cp)
    toks = np.arange(100, 164, dtype=np.int32)
    wb = cp.DeviceBatch.from_numpy(toks, np.array([0, 64], np.int64), np.zeros(64, np.uint8))
    idx.insert(wb, _kv(cp, idx, 64), _sp([0]), _sp([0]), _sp([16]), t=1)
    before = _state(idx)
    idx.insert(wb, _kv(cp, idx, 64, max_blocks=3), _sp([0]), _sp([8]), _sp([48]), t=2)   # needs block 3
    assert idx.last_error() == cp.CP_ERR_INVALID_ARG
    assert _state(idx) == before


def test_supersede_over_1024_segments_is_rejected_without_side_effects():
    cp = _cp()
    idx = _index(cp)
    n = 4 * 1030
    toks = np.arange(1000, 1000 + n, dtype=np.int32)
    wb = cp.DeviceBatch.from_numpy(toks, np.array([0, n], np.int64), np.zeros(n, np.uint8))
    kv = _kv(cp, idx, n)
    k = 1025                                                          # 1025 disjoint 4-token segments
    idx.insert(wb, kv, _sp([0] * k), _sp(list(range(0, 4 * k, 4))), _sp([4] * k), t=1)
    assert idx.last_error() == 0
    before = _state(idx)
    assert before[0] == k
    ids, oc = idx.insert(wb, kv, _sp([0]), _sp([0]), _sp([4 * k + 4]), t=2)   # strictly contains all 1025
    assert idx.last_error() == cp.CP_ERR_CAPACITY
    assert _state(idx) == before
    assert int(oc[0].item()) == -1
    # 1024 contained segments are within the limit: the span supersedes them all
    idx2 = _index(cp)
    idx2.insert(wb, kv, _sp([0] * 1024), _sp(list(range(0, 4096, 4))), _sp([4] * 1024), t=1)
    _, oc2 = idx2.insert(wb, kv, _sp([0]), _sp([0]), _sp([4096 + 4]), t=2)
    assert idx2.last_error() == 0
    assert int(oc2[0].item()) == cp.CP_SUPERSEDED
    assert _state(idx2)[0] == 1


def test_overlapping_spans_over_copy_list_capacity_are_rejected():
    cp = _cp()
    # chunk list CH = max_batch_tokens/32 + max(hit cap, spans) + 1 = 32 + 64 + 1 = 97 chunks of 32 tokens
    idx = _index(cp, window_len=128, max_batch_tokens=1024, max_batch_reqs=1, max_spans_per_insert=64,
                 max_req_tokens=1024, max_span_len=1024)
    toks = np.arange(5000, 6024, dtype=np.int32)
    wb = cp.DeviceBatch.from_numpy(toks, np.array([0, 1024], np.int64), np.zeros(1024, np.uint8))
    kv = _kv(cp, idx, 1024)
    before = _state(idx)
    # 24 spans [i, i + 1000): equal length, none contains another, 32 chunks each = 768 > 97
    idx.insert(wb, kv, _sp([0] * 24), _sp(list(range(24))), _sp([1000] * 24), t=1)
    assert idx.last_error() == cp.CP_ERR_CAPACITY
    assert _state(idx) == before
    # a non-overlapping batch of the same call shape still inserts
    idx.insert(wb, kv, _sp([0, 0]), _sp([0, 512]), _sp([512, 512]), t=2)
    assert idx.last_error() == 0
    assert _state(idx)[0] == 2
