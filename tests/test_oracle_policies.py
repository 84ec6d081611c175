"""Pins for the oracle's NEXT-3 baseline policies (R#28-29).

FixedChunk and PrefixOnly are restated here independently of the oracle's C code:
- FixedChunk (Fig. 4-b): a reader chunk [c*L, (c+1)*L) is
  covered iff it has no mask-1 token and its exact content equals some mask-free aligned chunk of a
  prior (writer) request.  Restated with Python sets of token tuples.
- PrefixOnly (Fig. 4-a): the covered prefix ends where the tokens
  diverge from a prior request's stored prefix or at the first mask-1 token.  Restated as a max of
  longest-common-prefix loops over the writers' prefixes.
Also pinned: the SPEC's worked construction and the directional criterion 7.
"""
import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import Batch, pack_batches

VOCAB = 128256


def batch_of(reqs, masks):
    parts = []
    for i, (r, m) in enumerate(zip(reqs, masks)):
        parts.append(Batch(tokens=np.asarray(r, np.int32), offsets=np.array([0, len(r)], np.int64),
                           mask=np.asarray(m, np.uint8), writer_ids=np.array([i], np.int64)))
    return pack_batches(parts)


def store(writers, policy, L, max_len=1 << 20):
    idx = O.OracleIndex(L, 42, 1 << 24, 1 << 20)
    sr, sb, sl = O.policy_spans(writers, policy, L, max_len)
    if len(sr):
        rc, _, oc = idx.insert(writers, t=1, spans=(sr, sb, sl))
        assert rc == 0
    return idx, (sr, sb, sl)


# ---------------------------------------------------------------------------- policy_spans
def test_policy_spans_hand_example():
    L = 4
    toks = [list(range(10)), list(range(20, 33)), list(range(40, 43))]
    masks = [[0] * 10,
             [0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0],
             [0, 0, 0]]
    b = batch_of(toks, masks)
    sr, sb, sl = O.policy_spans(b, "fixed_chunk", L, 100)
    # request 0: chunks [0,4) [4,8) (the tail 8..9 is not a full chunk); request 1: chunk [4,8) holds
    # the mask-1 token 5, [0,4) and [8,12) are clean; request 2: shorter than one chunk
    assert list(zip(sr, sb, sl)) == [(0, 0, 4), (0, 4, 4), (1, 0, 4), (1, 8, 4)]
    sr, sb, sl = O.policy_spans(b, "prefix_only", L, 100)
    assert list(zip(sr, sb, sl)) == [(0, 0, 10), (1, 0, 5)]
    sr, sb, sl = O.policy_spans(b, "prefix_only", L, 7)        # max_len truncates the stored prefix
    assert list(zip(sr, sb, sl)) == [(0, 0, 7), (1, 0, 5)]


# ---------------------------------------------------------------------------- FixedChunk
def fixed_chunk_brute(writers_t, writers_m, reader_t, reader_m, L):
    """Covered reader positions and, per covered chunk, the writer chunk it reuses (first
    occurrence in writer order)."""
    first = {}
    for wi, (t, m) in enumerate(zip(writers_t, writers_m)):
        for c in range(len(t) // L):
            ch = tuple(t[c * L:(c + 1) * L])
            if not any(m[c * L:(c + 1) * L]) and ch not in first:
                first[ch] = (wi, c * L)
    cov = np.zeros(len(reader_t), bool)
    hits = []
    for c in range(len(reader_t) // L):
        ch = tuple(reader_t[c * L:(c + 1) * L])
        if not any(reader_m[c * L:(c + 1) * L]) and ch in first:
            cov[c * L:(c + 1) * L] = True
            hits.append((c * L, first[ch][1]))
    return cov, hits


def _chunky_case(rng, L, alphabet):
    """Writers and a reader built from a small library of chunks, so that aligned and shifted reuse
    both occur; random masks."""
    lib_ = [[int(x) for x in rng.integers(0, alphabet, L)] for _ in range(6)]
    def req(nchunks):
        t = []
        for _ in range(nchunks):
            t += lib_[int(rng.integers(0, len(lib_)))] if rng.random() < 0.7 else \
                [int(x) for x in rng.integers(0, alphabet, L)]
        shift = int(rng.integers(0, L)) if rng.random() < 0.3 else 0
        t = [int(x) for x in rng.integers(0, alphabet, shift)] + t + \
            [int(x) for x in rng.integers(0, alphabet, int(rng.integers(0, L)))]
        m = (rng.random(len(t)) < 0.02).astype(np.uint8)
        return t, m
    writers = [req(int(rng.integers(1, 6))) for _ in range(int(rng.integers(1, 5)))]
    reader = req(int(rng.integers(0, 7)))
    return writers, reader


@pytest.mark.parametrize("L,alphabet", [(4, 3), (8, 50), (16, VOCAB)])
def test_fixed_chunk_vs_set_restatement(L, alphabet):
    rng = np.random.default_rng(L * 7 + alphabet)
    for trial in range(120):
        writers, (rt, rm) = _chunky_case(rng, L, alphabet)
        wb = batch_of([w[0] for w in writers], [w[1] for w in writers])
        idx, _ = store(wb, "fixed_chunk", L)
        res = idx.match(batch_of([rt], [rm]), t=5, policy="fixed_chunk")
        cov, hits = fixed_chunk_brute([w[0] for w in writers], [w[1] for w in writers], rt, rm, L)
        assert np.array_equal(res.plan > 0, cov), trial
        assert int(res.req_covered[0]) == int(cov.sum())
        got = [(int(res.hit_dst[i]), int(res.hit_dst[i]) - int(res.hit_delta[i])) for i in range(res.num_hits)]
        assert got == hits                                       # (dst, writer origin) per covered chunk
        assert all(int(x) == L for x in res.hit_len)


def test_fixed_chunk_ignores_longer_entries_and_unaligned_windows():
    """The FixedChunk flag on a selective store: only aligned windows, only length-L entries."""
    L = 4
    rng = np.random.default_rng(3)
    a = [int(x) for x in rng.integers(0, VOCAB, 4)]
    b = [int(x) for x in rng.integers(0, VOCAB, 6)]
    wb = batch_of([a + b], [[0] * 10])
    idx = O.OracleIndex(L, 42, 1 << 20, 1 << 12)
    rc, _, _ = idx.insert(wb, t=1, spans=(np.array([0, 0], np.int32), np.array([0, 4], np.int32),
                                          np.array([4, 6], np.int32)))
    assert rc == 0
    r = [7, 7, 7, 7] + a + [7] + b + [7]
    res = idx.match(batch_of([r], [[0] * len(r)]), t=2, policy="fixed_chunk")
    assert [(int(res.hit_dst[i]), int(res.hit_len[i])) for i in range(res.num_hits)] == [(4, 4)]
    sel = idx.match(batch_of([r], [[0] * len(r)]), t=2)               # the method finds both
    assert [(int(sel.hit_dst[i]), int(sel.hit_len[i])) for i in range(sel.num_hits)] == [(4, 4), (9, 6)]


# ---------------------------------------------------------------------------- PrefixOnly
def lcp(a, b, m):
    n = 0
    while n < len(a) and n < len(b) and a[n] == b[n] and not m[n]:
        n += 1
    return n


@pytest.mark.parametrize("L", [4, 16])
def test_prefix_only_vs_lcp_restatement(L):
    rng = np.random.default_rng(100 + L)
    for trial in range(150):
        sysp = [int(x) for x in rng.integers(0, VOCAB, int(rng.integers(0, 3 * L)))]
        writers = []
        for _ in range(int(rng.integers(1, 5))):
            t = sysp + [int(x) for x in rng.integers(0, VOCAB, int(rng.integers(0, 3 * L)))]
            m = np.zeros(len(t), np.uint8)
            if rng.random() < 0.5 and len(t):
                m[int(rng.integers(0, len(t))):] = 1                # a sensitive suffix (Fig. 4-a)
            writers.append((t, m))
        if rng.random() < 0.5 and writers:                          # a writer whose prefix extends another's
            t0, m0 = writers[0]
            t = list(t0) + [int(x) for x in rng.integers(0, VOCAB, L)]
            writers.append((t, np.zeros(len(t), np.uint8)))
        src = writers[int(rng.integers(0, len(writers)))][0]
        cut = int(rng.integers(0, len(src) + 1))
        rt = list(src[:cut]) + [int(x) for x in rng.integers(0, VOCAB, int(rng.integers(0, 2 * L)))]
        rm = np.zeros(len(rt), np.uint8)
        if rng.random() < 0.3 and len(rt):
            rm[int(rng.integers(0, len(rt)))] = 1
        max_len = int(rng.integers(L, 6 * L))
        wb = batch_of([w[0] for w in writers], [w[1] for w in writers])
        idx, _ = store(wb, "prefix_only", L, max_len)
        res = idx.match(batch_of([rt], [rm]), t=5, policy="prefix_only")
        # restatement: max over writers of LCP(reader, stored prefix), stopped at the reader's first
        # mask-1 token, covered only if >= L (R#29)
        best = 0
        for t, m in writers:
            first = int(np.argmax(m)) if m.any() else len(t)
            p = t[:min(first, len(t), max_len)]
            if len(p) >= L:
                best = max(best, lcp(rt, p, rm))
        want = best if best >= L else 0
        assert int(res.req_covered[0]) == want, trial
        assert np.array_equal(res.plan > 0, np.arange(len(rt)) < want)
        if want:
            assert res.num_hits == 1 and int(res.hit_dst[0]) == 0 and int(res.hit_delta[0]) == 0
            e = idx.entry(int(res.hit_entry[0]))
            assert e["origin_pos"] == 0 and list(e["tokens"][:want]) == rt[:want]
        else:
            assert res.num_hits == 0


def test_identical_unmasked_prompt_prefix_only_covers_all():
    """A1 invariant under PrefixOnly: an unmasked identical prompt is covered whole."""
    rng = np.random.default_rng(4)
    p = [int(x) for x in rng.integers(0, VOCAB, 300)]
    wb = batch_of([p], [[0] * 300])
    idx, _ = store(wb, "prefix_only", 128)
    res = idx.match(batch_of([p], [[0] * 300]), t=2, policy="prefix_only")
    assert (res.num_hits, int(res.hit_len[0]), int(res.req_covered[0])) == (1, 300, 300)


# ---------------------------------------------------------------------------- granularity gap
def straddle_pair(rng, shift, span_len=200, pos=60, n=400, L=128):
    """a shared span straddling a chunk boundary, shifted by `shift` tokens between writer
    and reader; everything outside the span is the writer's private (masked) text."""
    span = [int(x) for x in rng.integers(0, VOCAB, span_len)]
    wt = [int(x) for x in rng.integers(0, VOCAB, pos)] + span
    wt += [int(x) for x in rng.integers(0, VOCAB, n - len(wt))]
    wm = np.ones(n, np.uint8)
    wm[pos:pos + span_len] = 0
    rt = [int(x) for x in rng.integers(0, VOCAB, pos + shift)] + span
    rt += [int(x) for x in rng.integers(0, VOCAB, n - len(rt))]
    return (wt, wm), (rt, np.zeros(n, np.uint8))


def selective_store(wb, L):
    """The method's store: every maximal mask-0 run of length >= L (coarse segments)."""
    idx = O.OracleIndex(L, 42, 1 << 24, 1 << 20)
    sr, sb, sl = [], [], []
    for r in range(wb.num_reqs):
        a, b = int(wb.offsets[r]), int(wb.offsets[r + 1])
        m = wb.mask[a:b]
        i = 0
        while i < b - a:
            if m[i]:
                i += 1
                continue
            j = i
            while j < b - a and not m[j]:
                j += 1
            if j - i >= L:
                sr.append(r); sb.append(i); sl.append(j - i)
            i = j
    rc, _, _ = idx.insert(wb, t=1, spans=(np.array(sr, np.int32), np.array(sb, np.int32), np.array(sl, np.int32)))
    assert rc == 0
    return idx


def test_spec_straddling_example():
    """selective covers the 200-token span, FixedChunk covers 0."""
    rng = np.random.default_rng(401)
    (wt, wm), (rt, rm) = straddle_pair(rng, shift=1)
    wb, rb = batch_of([wt], [wm]), batch_of([rt], [rm])
    sel = selective_store(wb, 128).match(rb, t=2)
    fc, (sr, sb, sl) = store(wb, "fixed_chunk", 128)
    assert list(sb) == [128]                  # the writer's only clean aligned chunk is [128, 256)
    fix = fc.match(rb, t=2, policy="fixed_chunk")
    assert int(sel.req_covered[0]) == 200 and int(fix.req_covered[0]) == 0


def test_criterion7_granularity_gap_direction():
    """S:L645 criterion 7: on boundary-straddling pairs shifted by 1-64 tokens, CrossUserSelective's
    match rate strictly exceeds FixedChunk(128)'s on >= 95% of 200 seeded pairs."""
    wins = 0
    for seed in range(200):
        rng = np.random.default_rng(10_000 + seed)
        shift = int(rng.integers(1, 65))
        span_len = int(rng.integers(160, 320))
        pos = int(rng.integers(0, 128))
        (wt, wm), (rt, rm) = straddle_pair(rng, shift, span_len, pos, n=pos + shift + span_len + 64)
        wb, rb = batch_of([wt], [wm]), batch_of([rt], [rm])
        s = int(selective_store(wb, 128).match(rb, t=2).req_covered[0])
        f = int(store(wb, "fixed_chunk", 128)[0].match(rb, t=2, policy="fixed_chunk").req_covered[0])
        wins += s > f
    assert wins >= 190
