"""GPU parity for NEXT-2, zero-copy page linking (R#31):
cp_link_blocks vs the oracle's link table, bit exact; and the data contract behind a link: with
CP_SKIP_LINKED the gather leaves exactly the linked destination blocks unwritten, every other row
is bit-identical to the full gather, and the linked pool page holds bit-for-bit the rows the full
gather would have copied (so pointing a block table at it is equivalent to copying)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.gen import make_workload  # noqa: E402
from tests.harness import SENTINEL, Case, ParityReport  # noqa: E402


def _check(case, readers, t, rep_links):
    cp = case.cp
    db = case._dev_batch(readers, with_mask=True)
    hits = case.dev.match_spans(db, t, no_touch=True)
    res = case.orc.match(readers, t, no_touch=True)
    maxb = int(max((readers.offsets[r + 1] - readers.offsets[r] + 15) // 16 for r in range(readers.num_reqs)))
    link = case.dev.link_blocks(db, hits, maxb + 3).cpu().numpy()
    assert case.dev.last_error() == 0
    olink = case.orc.link_blocks(readers, res, maxb + 3)
    nb = [(int(n) + 15) // 16 for n in readers.lens]
    for r in range(readers.num_reqs):                        # blocks beyond a request are not written
        assert (link[r, nb[r]:] == -1).all()
    assert np.array_equal(link, olink)
    full = case.dst_kv(readers)
    case.dev.gather_rerotate(db, hits, full, zero_recompute=True)
    skip = cp.PagedKV([t.clone().fill_(SENTINEL) for t in full.k], [t.clone().fill_(SENTINEL) for t in full.v],
                      full.block_tables)
    case.dev.gather_rerotate(db, hits, skip, zero_recompute=True, skip_linked=True)
    assert case.dev.last_error() == 0
    pk, pv = case.dev.pool_views()
    bt = full.block_tables.cpu().numpy()
    rr, bb = np.nonzero(link >= 0)
    lb = torch.from_numpy(bt[rr, bb].astype(np.int64)).cuda()
    pages = torch.from_numpy(link[rr, bb].astype(np.int64)).cuda()
    linked = torch.zeros(full.k[0].shape[0], dtype=torch.bool, device="cuda")
    linked[lb] = True
    for l in range(case.g.num_layers):
        for F, S, P in ((full.k[l], skip.k[l], pk[l]), (full.v[l], skip.v[l], pv[l])):
            assert torch.equal(F[~linked], S[~linked])                       # every other row: identical
            assert (S[linked] == SENTINEL).all()                             # linked blocks: untouched
            assert torch.equal(P[pages], F[lb])                              # pool page == copied rows
    rep_links.append(int((link >= 0).sum()))


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 0.05), (3, 0.04)])
def test_link_blocks_parity_and_skip_contract(cfg, scale):
    wl = make_workload(cfg, scale=scale)
    case = Case(wl, seed=cfg)
    wb, rb = wl.rounds[0]
    rng = np.random.default_rng(cfg)
    rep = ParityReport()
    case.insert(wb, rep, bits_flags=[rng.random(int(m)) < 0.02 for m in wb.span_len])   # sparse marks
    assert rep.ok, rep.notes
    links = []
    _check(case, rb, 100, links)           # shifted readers
    _check(case, wb, 101, links)           # the writers re-reading their own prompts (delta 0)
    assert links[1] > 0


def test_identical_unmasked_prompt_links_all_full_pages():
    """Ordinary prefix reuse as block-table edits: a stored unmasked prompt without
    recompute marks, read again, links every full page to the entry's pages (ascending on a fresh
    index, R#22) and leaves nothing for the gather to copy but the partial tail page."""
    import dataclasses
    wl = make_workload(1)
    wb, _ = wl.rounds[0]
    one = wb.subset([0])
    n = int(one.lens[0])
    one = dataclasses.replace(one, mask=np.zeros(n, np.uint8), span_req=np.zeros(1, np.int32),
                              span_begin=np.zeros(1, np.int32), span_len=np.array([n], np.int32))
    case = Case(wl, seed=3)
    rep = ParityReport()
    case.insert(one, rep, bits_flags=[np.zeros(n, bool)])
    assert rep.ok, rep.notes
    db = case._dev_batch(one)
    hits = case.dev.match_spans(db, 50, no_touch=True)
    link = case.dev.link_blocks(db, hits, (n + 15) // 16).cpu().numpy()[0]
    full = n // 16
    assert list(link[:full]) == list(range(full))
    assert (link[full:] == -1).all()
