"""GPU parity for the linked-page lifetime (NEXT-2 remainder, R#32): cp_pin_links pins /
unpins the entries owning pool pages; with pins in the index, every insert -- outcomes (incl.
CP_DEFERRED_PINNED), entry ids, the whole live index with its pin counts, the free-page FIFO -- equals
the oracle's (tests/test_oracle_pins.py pins the oracle), and a pinned page's pool rows and tokens stay
bit-identical across the inserts that would otherwise have evicted or superseded it."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from tests.harness import Case, ParityReport  # noqa: E402
from tests.test_gpu_fuzz_index import _workload  # noqa: E402


@pytest.mark.parametrize("seed", range(12))
def test_pins_gpu_vs_oracle(seed):
    wl = _workload(400 + seed, "bf16", heavy=seed % 2 == 0, w=8)
    case = Case(wl, seed=seed, sample_reqs=None)
    rep = ParityReport()
    rng = np.random.default_rng(seed)
    held = []                                              # (pages, pool rows of those pages, tokens) pinned
    pinned_rounds = 0
    for wb, rb in wl.rounds:
        snap = case.dev.snapshot()
        ents = snap["entries"]
        for _ in range(int(rng.integers(1, 4))):           # pin a few pages of random live entries
            if not ents:
                break
            e = ents[int(rng.integers(0, len(ents)))]
            pg = [int(x) for x in rng.choice(e["pages"], size=min(2, len(e["pages"])), replace=False)]
            d = torch.tensor(pg, dtype=torch.int32, device="cuda")
            case.dev.pin_links(d, 1)
            assert case.dev.last_error() == 0
            assert case.orc.pin_pages(pg, 1) == 0
            k, v = case.dev.pool_views()
            held.append((pg, k[:, pg].clone(), v[:, pg].clone()))
        if held and rng.random() < 0.3:                    # release one pin set
            pg, _, _ = held.pop(int(rng.integers(0, len(held))))
            case.dev.pin_links(torch.tensor(pg, dtype=torch.int32, device="cuda"), -1)
            assert case.dev.last_error() == 0
            assert case.orc.pin_pages(pg, -1) == 0
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
        pinned_rounds += int(sum(1 for e in case.orc.live_entries() if e["pin"]) > 0)
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
        k, v = case.dev.pool_views()
        for pg, k0, v0 in held:                            # pinned pages never recycled or overwritten
            assert torch.equal(k[:, pg].view(torch.int16), k0.view(torch.int16))
            assert torch.equal(v[:, pg].view(torch.int16), v0.view(torch.int16))
    assert pinned_rounds > 0


def test_pin_errors_change_nothing():
    import paper_2605_23640_b200 as cp
    wl = _workload(450, "bf16", w=8)
    case = Case(wl, seed=0, sample_reqs=None)
    rep = ParityReport()
    case.insert(wl.rounds[0][0], rep)
    assert rep.ok
    snap = case.dev.snapshot()
    e = snap["entries"][0]
    free = int(snap["fifo"][0])
    case.dev.pin_links(torch.tensor([int(e["pages"][0]), free], dtype=torch.int32, device="cuda"), 1)
    assert case.dev.last_error() == cp._lib.CP_ERR_INVALID_ARG                 # a free page
    case.dev.pin_links(torch.tensor([int(e["pages"][0])] * 2, dtype=torch.int32, device="cuda"), -1)
    assert case.dev.last_error() == cp._lib.CP_ERR_INVALID_ARG                 # below zero
    assert [x["pin"] for x in case.dev.snapshot()["entries"]] == [0] * len(snap["entries"])
    case.dev.pin_links(torch.tensor([int(e["pages"][0]), -1], dtype=torch.int32, device="cuda"), 1)
    assert case.dev.last_error() == 0
    assert case.dev.snapshot()["entries"][0]["pin"] == 1


def _idx(cap):
    import paper_2605_23640_b200 as cp
    return cp, cp.KVIndex(cp.IndexConfig(num_layers=1, num_kv_heads=1, head_dim=16, dtype="fp32", rope_theta=1e4,
                                         window_len=16, pool_capacity_tokens=cap, max_entries=256, max_span_len=512,
                                         max_req_tokens=1024, max_batch_reqs=4, max_batch_tokens=4096,
                                         max_spans_per_insert=8))


def _ins(cp, idx, toks, t):
    toks = np.asarray(toks, np.int32)
    n = len(toks)
    db = cp.DeviceBatch.from_numpy(toks, np.array([0, n], np.int64), np.zeros(n, np.uint8))
    nb = (n + 15) // 16
    kv = cp.PagedKV.allocate(1, nb, 1, 16, torch.float32, torch.arange(nb, dtype=torch.int32).view(1, nb))
    sp = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    ids, oc = idx.insert(db, kv, sp([0]), sp([0]), sp([n]), None, None, t)
    assert idx.last_error() == 0
    return int(ids[0].item()), int(oc[0].item())


def test_deferred_outcomes_match_the_oracle_worked_cases():
    rng = np.random.default_rng(7)
    A, big = rng.integers(1000, 9000, 160), None
    big = np.concatenate([rng.integers(1000, 9000, 40), A, rng.integers(1000, 9000, 40)])
    cp, idx = _idx(10_000)
    assert _ins(cp, idx, A, 1) == (0, cp._lib.CP_STORED)
    pages = torch.tensor(idx.snapshot()["entries"][0]["pages"], dtype=torch.int32, device="cuda")
    idx.pin_links(pages, 1)
    assert _ins(cp, idx, big, 2) == (0, cp._lib.CP_DEFERRED_PINNED)      # would supersede the pinned entry
    assert [e["id"] for e in idx.snapshot()["entries"]] == [0]
    idx.pin_links(pages, -1)
    assert _ins(cp, idx, big, 3) == (1, cp._lib.CP_SUPERSEDED)
    # pinned tokens + span over the budget
    cp, idx = _idx(500)
    assert _ins(cp, idx, rng.integers(1000, 9000, 300), 1)[1] == cp._lib.CP_STORED
    idx.pin_links(torch.tensor(idx.snapshot()["entries"][0]["pages"], dtype=torch.int32, device="cuda"), 1)
    assert _ins(cp, idx, rng.integers(1000, 9000, 250), 2) == (-1, cp._lib.CP_DEFERRED_PINNED)
    # LRU evicts the unpinned entry although the pinned one is older
    cp, idx = _idx(500)
    for t in (1, 2):
        _ins(cp, idx, rng.integers(1000, 9000, 200), t)
    idx.pin_links(torch.tensor(idx.snapshot()["entries"][0]["pages"][:1], dtype=torch.int32, device="cuda"), 1)
    assert _ins(cp, idx, rng.integers(1000, 9000, 200), 3) == (2, cp._lib.CP_STORED)
    assert [e["id"] for e in idx.snapshot()["entries"]] == [0, 2]
