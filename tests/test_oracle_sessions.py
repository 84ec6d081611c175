"""Pins for the oracle's same-user session reuse (NEXT-2 remainder; "If the request
belongs to the same user session, all KV cache can be reused without restriction.  If the request
originates from a different user, it applies the selective cross-user sharing policy"; DESIGN.md
R#33, modelled as SPEC S:L419-420 does: exact-prefix reuse of the user's own last request).

Pinned here: a worked example (the same session reuses its own sensitive tokens, nobody else sees them),
replacement of the session entry, a Python restatement of match-with-sessions over randomized
workloads, and the privacy probe run with private entries in the pool (cross-user direct recovery
stays 0 while the owner's own probes do recover them)."""
import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import Batch, pack_batches
from tests import privacy_probe as P


def req(tokens, mask=None):
    t = np.asarray(tokens, np.int32)
    m = np.zeros(len(t), np.uint8) if mask is None else np.asarray(mask, np.uint8)
    return Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=m, writer_ids=np.zeros(1, np.int64))


def test_session_reuses_its_own_sensitive_prefix_and_nobody_else_does():
    rng = np.random.default_rng(1)
    w = 8
    first = rng.integers(100, 200, 40).astype(np.int32)
    mask = np.zeros(40, np.uint8); mask[10:13] = 1                  # the user's own PII
    idx = O.OracleIndex(w, 0, 10_000, 4096)
    rc, ids, oc = idx.insert_session(req(first, mask), [5], t=1)
    assert rc == 0 and oc[0] == O.STORED and ids[0] == 0
    nxt = np.concatenate([first[:30], rng.integers(300, 400, 20)]).astype(np.int32)   # follow-up turn
    res = idx.match(req(nxt), t=2, sessions=[5])
    assert res.num_hits == 1 and (res.hit_entry[0], res.hit_dst[0], res.hit_len[0], res.hit_delta[0]) == (0, 0, 30, 0)
    assert res.plan[:30].tolist() == [1] * 30 and res.plan[30:].tolist() == [0] * 20
    for other in ([6], [0], None):                                   # another session, anonymous, no sessions
        assert idx.match(req(nxt), t=3, sessions=other).num_hits == 0
    assert idx.match(req(first[:w - 1]), t=4, sessions=[5]).num_hits == 0                # shorter than w


def test_session_entry_is_replaced_and_lives_in_the_shared_budget():
    rng = np.random.default_rng(2)
    idx = O.OracleIndex(8, 0, 100, 4096)
    a, b = rng.integers(100, 200, 60), rng.integers(200, 300, 70)
    assert idx.insert_session(req(a), [3], t=1)[2][0] == O.STORED
    pages_a = idx.live_entries()[0]["pages"].tolist()
    assert idx.insert_session(req(b), [3], t=2)[2][0] == O.STORED
    live = idx.live_entries()
    assert [(e["id"], e["owner"], e["len"]) for e in live] == [(1, 3, 70)]
    assert idx.fifo().tolist()[-len(pages_a):] == pages_a               # the old entry's pages, to the FIFO tail
    # a second session: 70 + 60 > 100 -> LRU evicts session 3's entry (private and shared share one budget)
    assert idx.insert_session(req(a), [4], t=3)[2][0] == O.STORED
    assert [(e["owner"], e["len"]) for e in idx.live_entries()] == [(4, 60)]
    # shared inserts never dedup against a private entry: the same tokens are stored again as shared
    w = req(a); w.span_req = np.zeros(1, np.int32); w.span_begin = np.zeros(1, np.int32); w.span_len = np.array([60], np.int32)
    rc, ids, oc = idx.insert(w, t=4)
    assert rc == 0 and oc[0] == O.STORED


def _py_match(entries, q, sess, w):
    """Plain restatement: the session's LCP hit (>= w) first, then greedy (k asc, m desc, id asc) over the
    exact occurrences of shared entries at k >= that prefix (R#7, R#33)."""
    hits, cursor = [], 0
    for e in entries:
        if sess and e["owner"] == sess:
            l = 0
            while l < min(e["len"], len(q)) and q[l] == e["tokens"][l]:
                l += 1
            if l >= w:
                hits.append((e["id"], 0, l)); cursor = l
    occ = []
    for e in entries:
        if e["owner"]:
            continue
        m = e["len"]
        for k in range(0, len(q) - m + 1):
            if list(q[k:k + m]) == list(e["tokens"]):
                occ.append((k, -m, e["id"]))
    for k, negm, eid in sorted(occ):
        if k >= cursor:
            hits.append((eid, k, -negm)); cursor = k - negm
    return hits


@pytest.mark.parametrize("seed", range(10))
def test_match_with_sessions_vs_restatement(seed):
    rng = np.random.default_rng(50 + seed)
    w = 4
    base = rng.integers(0, 5, 200).astype(np.int32)
    idx = O.OracleIndex(w, seed, 100_000, 8192)
    t = 0
    for step in range(12):
        t += 1
        a = int(rng.integers(0, 150)); n = int(rng.integers(w, 40))
        toks = base[a:a + n]
        if rng.random() < 0.5:
            assert idx.insert_session(req(toks), [int(rng.integers(1, 4))], t=t)[0] == 0
        else:
            wb = req(toks); wb.span_req = np.zeros(1, np.int32); wb.span_begin = np.zeros(1, np.int32)
            wb.span_len = np.array([len(toks)], np.int32)
            assert idx.insert(wb, t=t)[0] == 0
        entries = idx.live_entries()
        for _ in range(4):
            a = int(rng.integers(0, 150)); n = int(rng.integers(w, 60))
            q = base[a:a + n]
            sess = int(rng.integers(0, 4))
            res = idx.match(req(q), t=t, no_touch=True, sessions=[sess])
            got = [(int(res.hit_entry[i]), int(res.hit_dst[i]), int(res.hit_len[i])) for i in range(res.num_hits)]
            assert got == _py_match(entries, q, sess, w), (seed, step)


def test_private_entries_leak_nothing_to_other_users():
    """The privacy probe (tests/privacy_probe.py) with every writer ALSO stored as its own session's
    private entry (sensitive tokens included): cross-user probes (no session, and a foreign session)
    recover no sensitive token; the owner's own probes do (same-user reuse is unrestricted)."""
    for seed in range(10):
        wl = P.make_workload(seed)
        idx = O.OracleIndex(P.W, 42, 1 << 20, (1 << 20) // 16 + (1 << 20) // P.W + 64)
        assert idx.insert(wl.writers, t=1)[0] == 0
        wb = wl.writers
        sess = np.arange(1, wb.num_reqs + 1, dtype=np.int32)
        assert idx.insert_session(wb, sess, t=2)[0] == 0
        for who in (0, 10_000):
            R = lambda b, who=who: (idx.match(b, t=3, no_touch=True, use_mask=False,
                                              sessions=np.full(b.num_reqs, who, np.int32)).req_covered > 0).astype(np.uint8)
            rec, total, _ = P.attack(wl, R, "sensitive")
            assert total > 0 and rec == 0, (seed, who, rec)
    # the owner: writer 0's session probing its own prompt recovers its sensitive tokens
    wl = P.make_workload(3)
    idx = O.OracleIndex(P.W, 42, 1 << 20, (1 << 20) // 16 + (1 << 20) // P.W + 64)
    assert idx.insert_session(wl.writers, np.arange(1, wl.writers.num_reqs + 1), t=1)[0] == 0
    n0 = int(wl.writers.offsets[1])
    own = req(wl.writers.tokens[:n0])
    res = idx.match(own, t=2, no_touch=True, use_mask=False, sessions=[1])
    assert res.num_hits == 1 and res.hit_len[0] == n0 and wl.truth[:n0].any()
