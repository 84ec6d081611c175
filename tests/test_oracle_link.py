"""Pins for the oracle's zero-copy page linking (NEXT-2; "link reusable segments
without touching the actual KV", L245-252 prefix sharing; R#31).

Independent routes: closed forms on a fresh index (the FIFO hands out ascending pages, R#22), the
special cases that must not link (moved keys, misaligned pages, recompute marks, partial pages), and
a restatement through the gather's addressing rule (position q of hit h reads
page_list[e][(q - dst)/16], slot (q - dst) % 16): a block links iff its 16 positions read one page,
slots 0..15 in order, with delta 0 and plan code 1."""
import numpy as np

import oracle.oracle as O
from tests.test_oracle_match import make_index, reader_batch


def test_identical_unmasked_prompt_links_every_full_page():
    rng = np.random.default_rng(9)
    p = [int(x) for x in rng.integers(0, 128256, 300)]          # 18 full pages + 12 tokens
    idx, _, _ = make_index([{"tokens": p, "origin": 0}], 128)
    rb = reader_batch([p])
    res = idx.match(rb, t=2)
    link = idx.link_blocks(rb, res)
    assert link.shape == (1, 19)
    assert list(link[0]) == list(range(18)) + [-1]             # fresh FIFO: the entry owns pages 0..18


def test_no_link_for_moved_misaligned_recomputed_or_partial_blocks():
    rng = np.random.default_rng(1)
    a = [int(x) for x in rng.integers(0, 128256, 64)]
    b = [int(x) for x in rng.integers(0, 128256, 64)]
    c = [int(x) for x in rng.integers(0, 128256, 40)]
    # entry A stored at origin 16, B at origin 5, C at origin 0 (40 tokens: 2 full pages + 8)
    idx, ids, _ = make_index([{"tokens": a, "origin": 16}, {"tokens": b, "origin": 5},
                              {"tokens": c, "origin": 0}], 32)
    filler = lambda n: [int(x) for x in rng.integers(0, 128256, n)]
    reqs = [filler(32) + a,                                   # A at 32: delta 16, aligned -> no link
            filler(5) + b + filler(11),                      # B at 5: delta 0, misaligned -> no link
            filler(16) + a,                                  # A at 16: delta 0, aligned -> 4 links
            c]                                               # C at 0: pages 0, 1 linked, tail not
    rb = reader_batch(reqs)
    res = idx.match(rb, t=3)
    assert res.num_hits == 4
    link = idx.link_blocks(rb, res)
    pa = idx.entry(int(ids[0]))["pages"]
    pc = idx.entry(int(ids[2]))["pages"]
    assert (link[0] == -1).all() and (link[1] == -1).all()
    assert list(link[2][:5]) == [-1] + list(pa[:4])
    assert list(link[3][:3]) == [pc[0], pc[1], -1]


def test_recompute_mark_unlinks_only_its_block():
    rng = np.random.default_rng(2)
    p = [int(x) for x in rng.integers(0, 128256, 96)]
    flags = np.zeros(96, bool)
    flags[50] = True                                          # block 3 (positions 48..63)
    idx = O.OracleIndex(32, 42, 1 << 20, 1 << 10)
    from tests.test_oracle_match import writer_batch
    bits, offs = O.pack_bits([flags])
    rc, ids, _ = idx.insert(writer_batch([{"tokens": p, "origin": 0}], 32), bits, offs, t=1)
    assert rc == 0
    rb = reader_batch([p])
    res = idx.match(rb, t=2)
    link = idx.link_blocks(rb, res)
    pages = idx.entry(int(ids[0]))["pages"]
    assert list(link[0]) == [pages[0], pages[1], pages[2], -1, pages[4], pages[5]]


def _links_by_gather_rule(idx, rb, res):
    """Restatement via the gather's addressing (step 6), not the linking code."""
    R = rb.num_reqs
    nb = [int((rb.offsets[r + 1] - rb.offsets[r] + 15) // 16) for r in range(R)]
    out = np.full((R, max(nb)), -1, np.int32)
    src = {}                                                   # (r, q) -> (page, slot, delta)
    for h in range(res.num_hits):
        e = idx.entry(int(res.hit_entry[h]))
        for t in range(int(res.hit_len[h])):
            src[(int(res.hit_req[h]), int(res.hit_dst[h]) + t)] = (int(e["pages"][t // 16]), t % 16,
                                                                   int(res.hit_delta[h]))
    for r in range(R):
        for b in range(nb[r]):
            qs = range(16 * b, 16 * b + 16)
            got = [src.get((r, q)) for q in qs]
            if any(g is None for g in got):
                continue
            if any(int(res.plan[rb.offsets[r] + q]) != 1 for q in qs if rb.offsets[r] + q < rb.offsets[r + 1]):
                continue
            if 16 * b + 16 > rb.offsets[r + 1] - rb.offsets[r]:
                continue
            if len({g[0] for g in got}) == 1 and [g[1] for g in got] == list(range(16)) and got[0][2] == 0:
                out[r, b] = got[0][0]
    return out


def test_random_workloads_match_gather_addressing_restatement():
    from synth.gen import make_workload
    for cfg, scale in ((1, 1.0), (2, 0.05), (3, 0.05)):
        wl = make_workload(cfg, scale=scale)
        wb, rb = wl.rounds[0]
        g = wl.geometry
        num_pages = (wl.pool_capacity_tokens + wl.max_span_len + 15) // 16 + wl.pool_capacity_tokens // g.window_len + 2
        idx = O.OracleIndex(g.window_len, 42, wl.pool_capacity_tokens, num_pages)
        rng = np.random.default_rng(cfg)
        flags = [rng.random(int(m)) < 0.02 for m in wb.span_len]  # sparse marks: many linkable pages
        words, offs = O.pack_bits(flags)
        rc, _, _ = idx.insert(wb, words, offs, t=1)
        assert rc == 0
        for readers in (rb, wb):                                  # shifted readers and the writers themselves
            res = idx.match(readers, t=2)
            link = idx.link_blocks(readers, res)
            exp = _links_by_gather_rule(idx, readers, res)
            assert np.array_equal(link, exp[:, :link.shape[1]]), cfg
        # the writers re-reading their own prompts do link pages (delta 0 at their origins)
        assert (idx.link_blocks(wb, idx.match(wb, t=3)) >= 0).any() or cfg != 1
