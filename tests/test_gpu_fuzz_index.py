"""Randomized GPU-vs-oracle stress of the index (a7) and the matcher / gather (a1-a5).

Tiny alphabets make windows collide, segments repeat, contain one another and supersede; a small
token budget forces LRU eviction every round (candidate-list pops, deferred FIFO traffic and its
flushes, slot recycling); writers and readers are drawn from a shared pool of token "motifs" so hits
are frequent and shifted.  Every round the harness compares insert outcomes and entry ids, the whole
live index (ids, lengths, origins, hashes, digests, last_used, page lists, tokens, recompute bits,
free-page FIFO), hits, plan codes, stats and the gathered KV rows against the oracle."""
import numpy as np
import pytest

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.gen import Batch, Geometry, Workload, pack_batches  # noqa: E402
from tests.harness import Case, ParityReport  # noqa: E402


def _request(rng, motifs, alphabet, wid, writer, w=8):
    parts, mask = [], []
    for _ in range(int(rng.integers(2, 6))):
        if rng.random() < 0.7:
            m = motifs[int(rng.integers(len(motifs)))]
        else:
            m = rng.integers(0, alphabet, int(rng.integers(3, 5 * w))).astype(np.int32)
        parts.append(m)
        mask.append(np.zeros(len(m), np.uint8))
        if rng.random() < 0.4:                                     # a sensitive run between pieces
            k = int(rng.integers(1, 4))
            parts.append(rng.integers(0, alphabet, k).astype(np.int32))
            mask.append(np.ones(k, np.uint8))
    toks, msk = np.concatenate(parts)[:9000], np.concatenate(mask)[:9000]   # within cfg.max_req_tokens
    spans_b, spans_l = [], []
    if writer:                                                     # spans: maximal mask-free runs >= w, maybe trimmed
        i, n = 0, len(toks)
        while i < n:
            if msk[i]:
                i += 1
                continue
            a = i
            while i < n and not msk[i]:
                i += 1
            if i - a >= w:
                b0 = a + int(rng.integers(0, max(1, (i - a - w) // 3 + 1)))
                spans_b.append(b0)
                ln = i - b0 if rng.random() < 0.6 else int(rng.integers(w, i - b0 + 1))
                spans_l.append(min(ln, 12 * w))                    # <= the smallest budget below
    return Batch(tokens=toks, offsets=np.array([0, len(toks)], np.int64), mask=msk,
                 writer_ids=np.array([wid], np.int64), span_req=np.zeros(len(spans_b), np.int32),
                 span_begin=np.array(spans_b, np.int32), span_len=np.array(spans_l, np.int32))


def _workload(seed, dtype, heavy=False, w=8):
    rng = np.random.default_rng(seed)
    alphabet = int(rng.integers(3, 9))
    motifs = [rng.integers(0, alphabet, int(rng.integers(w, 8 * w))).astype(np.int32) for _ in range(3 if heavy else 6)]
    motifs += [np.concatenate([motifs[0], motifs[1]]), motifs[2][: max(w, len(motifs[2]) // 2)]]
    rounds, wid = [], 0
    for _ in range(5):
        nw = int(rng.integers(8, 17)) if heavy else int(rng.integers(2, 6))
        ws = [_request(rng, motifs, alphabet, wid + k, True, w) for k in range(nw)]
        wid += len(ws)
        rs = [_request(rng, motifs, alphabet, 10000 + wid + k, False, w) for k in range(int(rng.integers(1, 5)))]
        rounds.append((pack_batches(ws), pack_batches(rs)))
    L, H, d = [(1, 1, 16), (2, 2, 32), (1, 3, 16), (3, 1, 64)][seed % 4]
    g = Geometry(L, H, d, dtype, 10000.0 if seed % 3 else 500000.0, window_len=w,
                 rope_style="gptj" if seed % 5 == 0 else "neox")
    return Workload(f"fuzz{seed}", g, rounds, pool_capacity_tokens=int(rng.integers(15 * w, 50 * w)),
                    max_span_len=max(256, 16 * w))


@pytest.mark.parametrize("seed", range(64))
def test_index_fuzz_rounds(seed):
    wl = _workload(seed, "fp32" if seed % 2 else "bf16")
    case = Case(wl, seed=seed, sample_reqs=None, use_reader_mask=seed % 7 != 0)
    rep = ParityReport()
    for wb, rb in wl.rounds:
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
        case.match_and_gather(wb, rep, no_touch=True)            # writers re-read their own prompts
        assert rep.ok, rep.notes[:6]
    assert rep.stats.get("stored", 0) > 0


@pytest.mark.parametrize("seed", range(100, 164))
def test_index_fuzz_heavy_in_batch_repetition(seed):
    """Few motifs and 8-16 writers per batch: the same content recurs inside one insert call (first
    Dropped, later Stored after its container is evicted or superseded, ...) -- the batch-dedup /
    representative paths of the commit."""
    wl = _workload(seed, "bf16" if seed % 2 else "fp32", heavy=True)
    case = Case(wl, seed=seed, sample_reqs=None)
    rep = ParityReport()
    for wb, rb in wl.rounds:
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
    assert rep.stats.get("stored", 0) > 0


@pytest.mark.parametrize("seed", range(200, 216))
def test_index_fuzz_long_windows(seed):
    """The same generators at the paper's window sizes (w = 32 and 128): long motifs, spans of
    hundreds to ~1.5K tokens, budgets of 15-50 windows."""
    w = 32 if seed % 2 else 128
    wl = _workload(seed, "bf16" if seed % 4 < 2 else "fp32", heavy=seed % 3 == 0, w=w)
    case = Case(wl, seed=seed, sample_reqs=None)
    rep = ParityReport()
    for wb, rb in wl.rounds:
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
    assert rep.stats.get("stored", 0) > 0


_COMMITS = {"parallel": 0, "serial": 0}


@pytest.mark.parametrize("seed", list(range(300, 316)))
def test_index_fuzz_commit_paths(seed):
    """Both commit paths on the fuzz generators (the parallel apply where the batch's segments do not
    interact, the sequential loop otherwise), each against the oracle; the last case checks that
    both paths were taken over the set."""
    wl = _workload(seed, "bf16", heavy=seed % 2 == 0, w=[4, 8, 32][seed % 3])
    case = Case(wl, seed=seed, sample_reqs=None)
    rep = ParityReport()
    for wb, rb in wl.rounds:
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
    par, ser, why = case.dev.commit_stats()
    _COMMITS["parallel"] += par
    _COMMITS["serial"] += ser
    if seed == 315:
        assert _COMMITS["parallel"] > 0 and _COMMITS["serial"] > 0, _COMMITS
