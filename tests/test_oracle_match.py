"""Pins for the oracle's matching + greedy assembly.

Independent routes: the SURVEY worked example (computed by brute force), and a
recursive re-statement of the greedy rule using Python's str.find (a library
substring search) on tiny alphabets, plus the SPEC invariants (soundness,
non-overlap, privacy, covered + uncovered = n).
"""
import json
import os

import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import Batch, pack_batches

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FILL = 1_000_000   # filler ids far from the tiny test alphabets


def writer_batch(entries, w):
    """One writer request per entry: [masked filler of length origin][entry tokens]."""
    parts = []
    for i, e in enumerate(entries):
        o, t = e["origin"], np.asarray(e["tokens"], np.int32)
        toks = np.concatenate([np.arange(FILL, FILL + o, dtype=np.int32), t])
        mask = np.concatenate([np.ones(o, np.uint8), np.zeros(len(t), np.uint8)])
        parts.append(Batch(tokens=toks, offsets=np.array([0, len(toks)], np.int64), mask=mask,
                           writer_ids=np.array([i], np.int64), span_req=np.zeros(1, np.int32),
                           span_begin=np.array([o], np.int32), span_len=np.array([len(t)], np.int32)))
    return pack_batches(parts)


def reader_batch(reqs, masks=None):
    parts = []
    for i, r in enumerate(reqs):
        r = np.asarray(r, np.int32)
        m = np.zeros(len(r), np.uint8) if masks is None else np.asarray(masks[i], np.uint8)
        parts.append(Batch(tokens=r, offsets=np.array([0, len(r)], np.int64), mask=m,
                           writer_ids=np.array([1000 + i], np.int64)))
    return pack_batches(parts)


def make_index(entries, w, cap=1 << 20, pages=1 << 16):
    idx = O.OracleIndex(w, 42, cap, pages)
    rc, ids, oc = idx.insert(writer_batch(entries, w), t=1)
    assert rc == 0
    return idx, ids, oc


def test_worked_example():
    ex = json.load(open(os.path.join(GOLD, "match_worked_example.json")))
    w = ex["window_len"]
    idx, ids, oc = make_index(ex["entries"], w)
    assert list(ids) == [0, 1, 2, 3] and list(oc) == [O.STORED] * 4
    rb = reader_batch([ex["request"]])
    res = idx.match(rb, t=2, use_mask=False)
    hits = [[int(res.hit_entry[i]), int(res.hit_dst[i]), int(res.hit_len[i]), int(res.hit_delta[i])]
            for i in range(res.num_hits)]
    assert hits == ex["expect_no_mask"]["hits"]
    assert int(res.req_covered[0]) == ex["expect_no_mask"]["covered"]
    mask = np.zeros(len(ex["request"]), np.uint8)
    mask[ex["reader_mask_positions"]] = 1
    rb2 = reader_batch([ex["request"]], [mask])
    res2 = idx.match(rb2, t=3, use_mask=True)
    hits2 = [[int(res2.hit_entry[i]), int(res2.hit_dst[i]), int(res2.hit_len[i]), int(res2.hit_delta[i])]
             for i in range(res2.num_hits)]
    assert hits2 == ex["expect_with_mask"]["hits"]
    assert int(res2.req_covered[0]) == ex["expect_with_mask"]["covered"]
    # plan codes for the unmasked request: covered positions 1..4 and 6..11
    assert list(res.plan) == [0, 1, 1, 1, 1, 0, 1, 1, 1, 1, 1, 1]


def _s(tokens):
    return "".join(chr(65 + int(t)) for t in tokens)


def greedy_by_find(req, mask, entries, w):
    """Recursive restatement of the greedy rule with str.find (library substring search):
    repeatedly take the earliest unmasked occurrence at or after the cursor, preferring longer
    then smaller id, and move the cursor past it."""
    rs = _s(req)
    hits, cursor = [], 0
    while True:
        best = None
        for eid, e in enumerate(entries):
            es = _s(e["tokens"])
            k = rs.find(es, cursor)
            while k >= 0 and mask is not None and any(mask[k:k + len(es)]):
                k = rs.find(es, k + 1)
            if k < 0:
                continue
            key = (k, -len(es), eid)
            if best is None or key < best[0]:
                best = (key, eid, k, len(es))
        if best is None:
            return hits
        _, eid, k, m = best
        hits.append((eid, k, m, k - entries[eid]["origin"]))
        cursor = k + m


def count_prefix_candidates(req, entries, w):
    rs = _s(req)
    c = 0
    for e in entries:
        pre = _s(e["tokens"][:w])
        k = rs.find(pre)
        while k >= 0:
            c += 1
            k = rs.find(pre, k + 1)
    return c


def _random_case(rng, alphabet, w):
    entries, seen = [], set()
    for i in range(int(rng.integers(1, 7))):
        m = int(rng.integers(w, w + 6))
        t = [int(x) for x in rng.integers(0, alphabet, m)]
        entries.append({"tokens": t, "origin": int(rng.integers(0, 20))})
    # keep only containment-free, distinct entries (the pool invariant)
    kept = []
    for e in entries:
        s = _s(e["tokens"])
        if any(s in _s(k["tokens"]) or _s(k["tokens"]) in s for k in kept):
            continue
        kept.append(e)
    n = int(rng.integers(0, 40))
    req = [int(x) for x in rng.integers(0, alphabet, n)]
    # plant a few entries
    for e in kept:
        if rng.random() < 0.7 and len(e["tokens"]) <= n:
            k = int(rng.integers(0, n - len(e["tokens"]) + 1))
            req[k:k + len(e["tokens"])] = e["tokens"]
    return kept, req


@pytest.mark.parametrize("alphabet,w", [(2, 2), (3, 3), (4, 2), (26, 4)])
def test_greedy_matches_str_find_restatement(alphabet, w):
    rng = np.random.default_rng(alphabet * 100 + w)
    for trial in range(150):
        entries, req = _random_case(rng, alphabet, w)
        if not entries:
            continue
        idx, ids, oc = make_index(entries, w)
        assert list(oc) == [O.STORED] * len(entries)
        use_mask = trial % 2 == 1
        mask = (rng.random(len(req)) < 0.1).astype(np.uint8) if use_mask else None
        res = idx.match(reader_batch([req], [mask] if use_mask else None), t=5, use_mask=use_mask)
        got = [(int(res.hit_entry[i]), int(res.hit_dst[i]), int(res.hit_len[i]), int(res.hit_delta[i]))
               for i in range(res.num_hits)]
        assert got == greedy_by_find(req, mask, entries, w)
        assert int(res.req_candidates[0]) == count_prefix_candidates(req, entries, w)
        # invariants: soundness, non-overlap, covered + uncovered = n
        cov = np.zeros(len(req), bool)
        for (e, k, m, d) in got:
            assert req[k:k + m] == entries[e]["tokens"]
            assert not cov[k:k + m].any()
            cov[k:k + m] = True
            if use_mask:
                assert not mask[k:k + m].any()
        assert int(res.req_covered[0]) == int(cov.sum())
        assert np.array_equal(res.plan > 0, cov)


def test_plan_recompute_codes_and_touch():
    w = 4
    ents = [{"tokens": [1, 2, 3, 4, 5, 6], "origin": 3}]
    idx = O.OracleIndex(w, 42, 1 << 20, 1 << 10)
    bits, offs = O.pack_bits([np.array([0, 1, 0, 0, 1, 1], bool)])
    rc, ids, oc = idx.insert(writer_batch(ents, w), bits, offs, t=10)
    assert rc == 0
    res = idx.match(reader_batch([[9, 1, 2, 3, 4, 5, 6, 9]]), t=20)
    assert list(res.plan) == [0, 1, 2, 1, 1, 2, 2, 0]
    assert int(res.req_recompute[0]) == 3 and int(res.req_covered[0]) == 6
    assert idx.entry(0)["last_used"] == 20                  # LRU touch of accepted hits
    idx.match(reader_batch([[1, 2, 3, 4, 5, 6]]), t=30, no_touch=True)
    assert idx.entry(0)["last_used"] == 20
    idx.match(reader_batch([[1, 2, 3, 4, 5, 6]]), t=5)
    assert idx.entry(0)["last_used"] == 20                  # max(last_used, t)


def test_empty_and_short_requests():
    w = 4
    idx, _, _ = make_index([{"tokens": [1, 2, 3, 4], "origin": 0}], w)
    rb = reader_batch([[], [1, 2, 3], [1, 2, 3, 4]])
    res = idx.match(rb, t=2)
    assert res.num_hits == 1 and list(res.req_hit_offsets) == [0, 0, 0, 1]
    assert list(res.req_candidates) == [0, 0, 1]
    # empty pool -> match rate 0
    idx2 = O.OracleIndex(w, 42, 1 << 20, 1 << 10)
    res2 = idx2.match(reader_batch([[1, 2, 3, 4, 5]]), t=1)
    assert res2.num_hits == 0 and int(res2.req_covered[0]) == 0


def test_identical_unmasked_prompt_is_prefix_reuse():
    """Invariant (north star): an unmasked identical prompt reproduces ordinary prefix reuse:
    one hit at dst 0 with delta 0 covering the whole prompt."""
    rng = np.random.default_rng(9)
    p = [int(x) for x in rng.integers(0, 128256, 300)]
    idx, _, _ = make_index([{"tokens": p, "origin": 0}], 128)
    res = idx.match(reader_batch([p]), t=2)
    assert res.num_hits == 1
    assert (int(res.hit_dst[0]), int(res.hit_len[0]), int(res.hit_delta[0])) == (0, 300, 0)
