"""The commit's LRU candidate list is prepared beside match + gather (cp_index_insert_prepare, k_lru_*)
from a snapshot that may precede the step's match touches, and is discarded after a pin.  These tests
put exactly those operations between the device prepare and commit -- a touching match of the same
step (the serving order: match at t, then the insert's commit at t), or pins of the oldest entries --
and require the oracle's sequential result (match / pin first, then the insert): outcomes, ids and
the whole live index, under LRU eviction every round (R#21, R#32)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from tests.harness import Case, ParityReport  # noqa: E402
from tests.test_gpu_fuzz_index import _workload  # noqa: E402


@pytest.mark.parametrize("seed", range(16))
def test_touching_match_between_prepare_and_commit(seed):
    wl = _workload(700 + seed, "bf16" if seed % 2 else "fp32", heavy=seed % 3 == 0, w=8)
    case = Case(wl, seed=seed, sample_reqs=None)
    rep = ParityReport()
    for i, (wb, rb) in enumerate(wl.rounds):
        def between(rb=rb):
            case.t -= 1                        # the match runs at the insert's logical time t
            case.match_and_gather(rb, rep)
        case.insert(wb, rep, between=between if i > 0 else None)
        assert rep.ok, rep.notes[:6]
    assert rep.stats.get("stored", 0) > 0


@pytest.mark.parametrize("seed", range(8))
def test_pin_between_prepare_and_commit(seed):
    wl = _workload(800 + seed, "bf16", heavy=seed % 2 == 0, w=8)
    case = Case(wl, seed=seed, sample_reqs=None)
    rep = ParityReport()
    rng = np.random.default_rng(seed)
    for i, (wb, rb) in enumerate(wl.rounds):
        def between():
            ents = sorted(case.dev.snapshot()["entries"], key=lambda e: (e["last_used"], e["id"]))
            for e in ents[:2]:                 # the two LRU-oldest entries: the next evictions' victims
                pg = [int(e["pages"][0])]
                case.dev.pin_links(torch.tensor(pg, dtype=torch.int32, device="cuda"), 1)
                assert case.dev.last_error() == 0
                assert case.orc.pin_pages(pg, 1) == 0
        case.insert(wb, rep, between=between if i > 0 else None)
        assert rep.ok, rep.notes[:6]
        case.match_and_gather(rb, rep)
        assert rep.ok, rep.notes[:6]
