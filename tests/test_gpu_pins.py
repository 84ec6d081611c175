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
    deferred = 0
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
        deferred += int(sum(1 for e in case.orc.live_entries() if e["pin"]) > 0)
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
        k, v = case.dev.pool_views()
        for pg, k0, v0 in held:                            # pinned pages never recycled or overwritten
            assert torch.equal(k[:, pg].view(torch.int16), k0.view(torch.int16))
            assert torch.equal(v[:, pg].view(torch.int16), v0.view(torch.int16))
    assert deferred > 0


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
