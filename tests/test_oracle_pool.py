"""Pins for the oracle's KV-pool insert / dedup / LRU / page allocation.

Independent routes: the SPEC worked examples, a Python restatement of the pool
rules that uses str-containment (library substring search) and sorts for LRU,
and exhaustive invariants (containment-freedom, budget, privacy, page
conservation).
"""
import json
import os

import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import Batch

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def one_writer(tokens, spans, mask=None):
    t = np.asarray(tokens, np.int32)
    m = np.zeros(len(t), np.uint8) if mask is None else np.asarray(mask, np.uint8)
    sb = np.array([s[0] for s in spans], np.int32)
    sl = np.array([s[1] for s in spans], np.int32)
    return Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=m, writer_ids=np.zeros(1, np.int64),
                 span_req=np.zeros(len(spans), np.int32), span_begin=sb, span_len=sl)


def test_spec_examples():
    ex = json.load(open(os.path.join(GOLD, "pool_spec_examples.json")))
    w = 64
    A = np.arange(1, 201, dtype=np.int32)          # A = [1..200]
    B = np.arange(50, 151, dtype=np.int32)         # B = [50..150]
    # insert A then B (B is a contiguous substring of A) -> DroppedAsContained
    idx = O.OracleIndex(w, 1, 1 << 20, 1 << 12)
    rc, ids, oc = idx.insert(one_writer(A, [(0, 200)]), t=1); assert rc == 0 and oc[0] == O.STORED
    rc, ids, oc = idx.insert(one_writer(B, [(0, 101)]), t=2)
    assert rc == 0 and oc[0] == O.DROPPED_CONTAINED and ids[0] == 0
    assert [e["len"] for e in idx.live_entries()] == [200]
    # insert B then A -> SupersededExisting([B])
    idx = O.OracleIndex(w, 1, 1 << 20, 1 << 12)
    idx.insert(one_writer(B, [(0, 101)]), t=1)
    rc, ids, oc = idx.insert(one_writer(A, [(0, 200)]), t=2)
    assert rc == 0 and oc[0] == O.SUPERSEDED and ids[0] == 1
    live = idx.live_entries()
    assert [(e["id"], e["len"]) for e in live] == [(1, 200)]
    # B's pages were freed to the FIFO tail and A got fresh pages from the head
    assert list(live[0]["pages"]) == list(range(7, 20))
    # LRU: capacity 300, three disjoint 128-token segments with distinct touch times
    cap = ex["lru"]["capacity"]
    idx = O.OracleIndex(128, 1, cap, 1 << 12)
    segs = [np.arange(1000 * (i + 1), 1000 * (i + 1) + 128, dtype=np.int32) for i in range(3)]
    idx.insert(one_writer(segs[0], [(0, 128)]), t=1)
    idx.insert(one_writer(segs[1], [(0, 128)]), t=2)
    rb = Batch(tokens=segs[0], offsets=np.array([0, 128], np.int64), mask=np.zeros(128, np.uint8),
               writer_ids=np.zeros(1, np.int64))
    idx.match(rb, t=3)                                  # touch segment 0 -> segment 1 is LRU
    idx.insert(one_writer(segs[2], [(0, 128)]), t=4)
    assert sorted(e["id"] for e in idx.live_entries()) == [0, 2]
    assert idx.live_tokens == 256


def test_duplicate_refreshes_and_validation_has_no_side_effects():
    w = 16
    idx = O.OracleIndex(w, 1, 1 << 20, 1 << 12)
    t = np.arange(100, 164, dtype=np.int32)
    rc, ids, oc = idx.insert(one_writer(t, [(0, 64)]), t=5)
    rc, ids, oc = idx.insert(one_writer(np.concatenate([[7, 7], t]), [(2, 64)]), t=9)
    assert oc[0] == O.DUPLICATE and ids[0] == 0
    assert idx.entry(0)["last_used"] == 9 and idx.entry(0)["origin_pos"] == 0
    before = (idx.num_ids, idx.live_tokens, list(idx.fifo()))
    mask = np.zeros(80, np.uint8); mask[40] = 1
    wb = one_writer(np.arange(500, 580), [(0, 20), (30, 20)], mask)
    rc, _, _ = idx.insert(wb, t=11)
    assert rc == O.ERR_SENSITIVE_SPAN                       # P:L403-405 selective sharing
    assert (idx.num_ids, idx.live_tokens, list(idx.fifo())) == before
    rc, _, _ = idx.insert(one_writer(np.arange(500, 580), [(0, 20), (30, 15)]), t=11)
    assert rc == O.ERR_SPAN_TOO_SHORT                       # P:L646-648 min length
    rc, _, _ = idx.insert(one_writer(np.arange(500, 580), [(70, 20)]), t=11)
    assert rc == O.ERR_INVALID_ARG
    assert (idx.num_ids, idx.live_tokens, list(idx.fifo())) == before


# ---------------------------------------------------------------------------
# Python restatement of the pool rules (str containment + sorted LRU)
# ---------------------------------------------------------------------------
class PyPool:
    def __init__(self, w, cap, pages, block=16):
        self.w, self.cap, self.block = w, cap, block
        self.e = {}          # id -> dict
        self.next = 0
        self.fifo = list(range(pages))

    @staticmethod
    def s(t):
        return ",".join(str(int(x)) for x in t) + ","

    def _rm(self, i):
        e = self.e.pop(i)
        self.fifo.extend(e["pages"])

    def insert(self, tau, origin, t):
        S = "," + self.s(tau)
        for i, e in self.e.items():
            if e["tokens"] == list(tau):
                e["last_used"] = t
                return O.DUPLICATE, i
        cont = [i for i, e in self.e.items() if len(e["tokens"]) > len(tau) and S in "," + self.s(e["tokens"])]
        if cont:
            return O.DROPPED_CONTAINED, min(cont)
        sup = sorted(i for i, e in self.e.items() if len(e["tokens"]) < len(tau) and "," + self.s(e["tokens"]) in S)
        for i in sup:
            self._rm(i)
        npg = -(-len(tau) // self.block)
        pages, self.fifo = self.fifo[:npg], self.fifo[npg:]
        i = self.next; self.next += 1
        self.e[i] = dict(tokens=list(tau), last_used=t, pages=pages, origin=origin)
        while sum(len(e["tokens"]) for e in self.e.values()) > self.cap:
            v = min(self.e, key=lambda j: (self.e[j]["last_used"], j))
            self._rm(v)
        return (O.SUPERSEDED if sup else O.STORED), i

    def touch(self, i, t):
        self.e[i]["last_used"] = max(self.e[i]["last_used"], t)


@pytest.mark.parametrize("seed", range(6))
def test_pool_vs_python_restatement(seed):
    rng = np.random.default_rng(100 + seed)
    w, cap, pages = 8, 120 + 40 * seed, 4096
    idx = O.OracleIndex(w, seed, cap, pages)
    py = PyPool(w, cap, pages)
    base = [int(x) for x in rng.integers(0, 6, 80)]          # small alphabet -> many containments
    t = 0
    for step in range(60):
        t += 1
        if rng.random() < 0.25 and py.e:
            # touch through a match of an existing entry's tokens
            i = int(rng.choice(sorted(py.e)))
            toks = py.e[i]["tokens"]
            rb = Batch(tokens=np.array(toks, np.int32), offsets=np.array([0, len(toks)], np.int64),
                       mask=np.zeros(len(toks), np.uint8), writer_ids=np.zeros(1, np.int64))
            res = idx.match(rb, t=t)
            for h in range(res.num_hits):
                py.touch(int(res.hit_entry[h]), t)
            continue
        a = int(rng.integers(0, 60)); m = int(rng.integers(w, 21))
        tau = (base + base)[a:a + m]
        wb = one_writer(tau, [(0, m)])
        rc, ids, oc = idx.insert(wb, t=t)
        assert rc == 0
        exp_oc, exp_id = py.insert(tau, 0, t)
        assert (int(oc[0]), int(ids[0])) == (exp_oc, exp_id)
        live = idx.live_entries()
        assert sorted(e["id"] for e in live) == sorted(py.e)
        for e in live:
            assert list(e["pages"]) == py.e[e["id"]]["pages"]
            assert e["last_used"] == py.e[e["id"]]["last_used"]
        assert list(idx.fifo()) == py.fifo
        # invariants
        strs = ["," + PyPool.s(e["tokens"]) for e in live]
        for i in range(len(strs)):
            for j in range(len(strs)):
                if i != j:
                    assert strs[i] not in strs[j]                  # containment-freedom
        assert idx.live_tokens <= cap                              # budget
        used = sorted(p for e in live for p in e["pages"])
        assert len(set(used)) == len(used)                        # pages owned exclusively
        assert sorted(used + list(idx.fifo())) == list(range(pages))   # page conservation


def test_entry_hashes_and_digest():
    w = 16
    idx = O.OracleIndex(w, 77, 1 << 20, 1 << 12)
    t = np.arange(3000, 3050, dtype=np.int32)
    idx.insert(one_writer(t, [(0, 50)]), t=1)
    e = idx.entry(0)
    assert e["prefix_hash"] == O.poly_hash(t[:w], idx.B)
    assert e["full_hash"] == O.poly_hash(t, idx.B)
    assert e["digest"] == O.sha256_tokens(t)
    assert list(e["pages"]) == [0, 1, 2, 3]                       # FIFO starts at ascending page ids
