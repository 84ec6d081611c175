"""Pins for the oracle's linked-page lifetime (NEXT-2 remainder; "link reusable segments
without touching the actual KV", R#32): an engine that links a request block to a pool page
pins it (orc_pin_pages +1 per linked block) until it releases it (-1).  While an entry is pinned it is
never evicted (LRU victims are the unpinned live entries) nor superseded (a span that would remove it,
or whose length with the pinned tokens exceeds the budget, is DEFERRED_PINNED and changes nothing), so
a pinned page is never recycled.  Pinned here: worked cases, a Python restatement of the pool rules
with pins over randomized sequences, and the never-recycled invariant."""
import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import Batch


def writer(tokens, spans):
    t = np.asarray(tokens, np.int32)
    return Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=np.zeros(len(t), np.uint8),
                 writer_ids=np.zeros(1, np.int64), span_req=np.zeros(len(spans), np.int32),
                 span_begin=np.array([a for a, _ in spans], np.int32), span_len=np.array([m for _, m in spans], np.int32))


def reader(tokens):
    t = np.asarray(tokens, np.int32)
    return Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=np.zeros(len(t), np.uint8),
                 writer_ids=np.zeros(1, np.int64))


def seg(seed, n):
    return [int(x) for x in np.random.default_rng(seed).integers(1000, 90000, n)]


def pin_entry(idx, toks, t, delta=1):
    """Link the entry equal to `toks` through a match of it at offset 0 (delta 0, page aligned) and pin
    the linked pages; returns the link table."""
    rb = reader(toks)
    res = idx.match(rb, t=t, no_touch=True)
    link = idx.link_blocks(rb, res)
    assert (link >= 0).any()
    assert idx.pin_pages(link, delta) == 0
    return link


def test_pinned_entry_is_not_evicted():
    A, C, D = seg(1, 200), seg(2, 200), seg(3, 200)
    idx = O.OracleIndex(16, 0, 500, 4096)
    for t, toks in enumerate([A, C], 1):
        assert idx.insert(writer(toks, [(0, 200)]), t=t)[0] == 0
    pin_entry(idx, A, 3)
    rc, ids, oc = idx.insert(writer(D, [(0, 200)]), t=4)
    assert rc == 0 and oc[0] == O.STORED
    live = [e["id"] for e in idx.live_entries()]
    assert live == [0, 2]                  # C (id 1) evicted although A (id 0) is older: A is pinned
    assert idx.entry_pin(0) > 0


def test_superseding_a_pinned_entry_is_deferred_until_unpinned():
    A = seg(4, 160)
    big = seg(5, 40) + A + seg(6, 40)
    idx = O.OracleIndex(16, 0, 10_000, 4096)
    assert idx.insert(writer(A, [(0, 160)]), t=1)[0] == 0
    link = pin_entry(idx, A, 2)
    before = [(e["id"], e["len"], e["pages"].tolist()) for e in idx.live_entries()]
    fifo = idx.fifo().tolist()
    rc, ids, oc = idx.insert(writer(big, [(0, len(big))]), t=3)
    assert rc == 0 and oc[0] == O.DEFERRED_PINNED and ids[0] == 0
    assert [(e["id"], e["len"], e["pages"].tolist()) for e in idx.live_entries()] == before
    assert idx.fifo().tolist() == fifo and idx.num_ids == 1
    assert idx.pin_pages(link, -1) == 0
    rc, ids, oc = idx.insert(writer(big, [(0, len(big))]), t=4)
    assert rc == 0 and oc[0] == O.SUPERSEDED
    assert [e["len"] for e in idx.live_entries()] == [len(big)]


def test_pinned_tokens_plus_span_over_budget_is_deferred():
    A, B = seg(7, 300), seg(8, 250)
    idx = O.OracleIndex(16, 0, 500, 4096)
    assert idx.insert(writer(A, [(0, 300)]), t=1)[0] == 0
    pin_entry(idx, A, 2)
    rc, ids, oc = idx.insert(writer(B, [(0, 250)]), t=3)
    assert rc == 0 and oc[0] == O.DEFERRED_PINNED and ids[0] == -1      # 300 pinned + 250 > 500
    assert [e["id"] for e in idx.live_entries()] == [0]


def test_pin_validation_has_no_side_effects():
    A = seg(9, 64)
    idx = O.OracleIndex(16, 0, 1000, 4096)
    assert idx.insert(writer(A, [(0, 64)]), t=1)[0] == 0
    pages = idx.live_entries()[0]["pages"]
    free_page = int(idx.fifo()[0])
    assert idx.pin_pages([pages[0], free_page], 1) == O.ERR_INVALID_ARG      # a page of no live entry
    assert idx.entry_pin(0) == 0
    assert idx.pin_pages([pages[0], pages[1]], -1) == O.ERR_INVALID_ARG      # below zero
    assert idx.pin_pages([pages[0], pages[1]], 1) == 0 and idx.entry_pin(0) == 2
    assert idx.pin_pages([pages[0], pages[1], pages[2]], -1) == O.ERR_INVALID_ARG
    assert idx.entry_pin(0) == 2
    assert idx.pin_pages([-1, pages[0], -1, pages[1]], -1) == 0 and idx.entry_pin(0) == 0


class PyPinnedPool:
    """The pool rules (R#20-22) written out again with pins (R#32), on Python lists."""

    def __init__(self, cap, pages, block=16):
        self.cap, self.block = cap, block
        self.e, self.next, self.fifo = {}, 0, list(range(pages))

    def insert(self, tau, t):
        tau = list(tau)
        s = lambda x: "," + ",".join(map(str, x)) + ","
        for i, e in self.e.items():
            if e["tokens"] == tau:
                e["last"] = t
                return O.DUPLICATE, i
        cont = [i for i, e in self.e.items() if len(e["tokens"]) > len(tau) and s(tau) in s(e["tokens"])]
        if cont:
            return O.DROPPED_CONTAINED, min(cont)
        blocked = [i for i, e in self.e.items() if e["pin"] and len(e["tokens"]) < len(tau) and s(e["tokens"]) in s(tau)]
        pinned = sum(len(e["tokens"]) for e in self.e.values() if e["pin"])
        if blocked or pinned + len(tau) > self.cap:
            return O.DEFERRED_PINNED, (min(blocked) if blocked else -1)
        sup = sorted(i for i, e in self.e.items() if len(e["tokens"]) < len(tau) and s(e["tokens"]) in s(tau))
        for i in sup:
            self.fifo.extend(self.e.pop(i)["pages"])
        npg = -(-len(tau) // self.block)
        pages, self.fifo = self.fifo[:npg], self.fifo[npg:]
        i = self.next; self.next += 1
        self.e[i] = dict(tokens=tau, last=t, pages=pages, pin=0)
        while sum(len(e["tokens"]) for e in self.e.values()) > self.cap:
            v = min((j for j in self.e if not self.e[j]["pin"]), key=lambda j: (self.e[j]["last"], j))
            self.fifo.extend(self.e.pop(v)["pages"])
        return (O.SUPERSEDED if sup else O.STORED), i


@pytest.mark.parametrize("seed", range(8))
def test_pins_vs_python_restatement(seed):
    rng = np.random.default_rng(300 + seed)
    cap, pages = 200 + 40 * seed, 4096
    idx = O.OracleIndex(8, seed, cap, pages)
    py = PyPinnedPool(cap, pages)
    base = [int(x) for x in rng.integers(0, 5, 90)]
    held = []                                   # (pages list, owner id) pinned so far
    for t in range(1, 80):
        r = rng.random()
        if r < 0.2 and py.e:
            i = int(rng.choice(sorted(py.e)))
            pg = [int(x) for x in rng.choice(py.e[i]["pages"], size=min(2, len(py.e[i]["pages"])), replace=False)]
            assert idx.pin_pages(pg, 1) == 0
            py.e[i]["pin"] += len(pg)
            held.append((pg, i))
            continue
        if r < 0.32 and held:
            pg, i = held.pop(int(rng.integers(0, len(held))))
            assert idx.pin_pages(pg, -1) == 0
            py.e[i]["pin"] -= len(pg)
            continue
        a = int(rng.integers(0, 70)); m = int(rng.integers(8, 21))
        tau = base[a:a + m]
        if len(tau) < 8:
            continue
        rc, ids, oc = idx.insert(writer(tau, [(0, len(tau))]), t=t)
        assert rc == 0
        exp_oc, exp_id = py.insert(tau, t)
        assert (int(oc[0]), int(ids[0])) == (exp_oc, exp_id), (t, int(oc[0]), int(ids[0]), exp_oc, exp_id)
        live = idx.live_entries()
        assert [e["id"] for e in live] == sorted(py.e)
        assert [e["pages"].tolist() for e in live] == [py.e[i]["pages"] for i in sorted(py.e)]
        assert idx.fifo().tolist() == py.fifo
        # invariant: a pinned entry's pages are never free
        free = set(py.fifo)
        for e in py.e.values():
            if e["pin"]:
                assert not free.intersection(e["pages"])
        assert sum(e["len"] for e in live) <= cap
