"""GPU parity for same-user session reuse (NEXT-2 remainder; R#33):
cp_index_insert_session and cp_match_spans with per-request sessions against the oracle -- outcomes,
ids, the whole live index with owners and pins, hits / plans / stats and the gathered K/V rows of the
private prefix hits and the cross-user hits after them -- on randomized mixes of shared inserts,
session inserts and session-tagged readers; and the privacy probe with private entries in the pool
(no sensitive token reaches another user through cp_match_spans)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle.oracle as O  # noqa: E402
from synth.gen import Batch, pack_batches  # noqa: E402
from tests import privacy_probe as P  # noqa: E402
from tests.harness import Case, ParityReport  # noqa: E402
from tests.test_gpu_fuzz_index import _request, _workload  # noqa: E402


@pytest.mark.parametrize("seed", range(12))
def test_sessions_gpu_vs_oracle(seed):
    wl = _workload(500 + seed, "bf16" if seed % 2 else "fp32", heavy=seed % 3 == 0, w=8)
    case = Case(wl, seed=seed, sample_reqs=None, max_sessions=4, batch_slack=64)
    rep = ParityReport()
    rng = np.random.default_rng(seed)
    for wb, rb in wl.rounds:
        case.insert(wb, rep)
        assert rep.ok, rep.notes[:6]
        # each writer (that fits an entry's page list, max_span_len) is also its session's last turn
        keep = [r for r in range(wb.num_reqs) if int(wb.lens[r]) <= wl.max_span_len]
        sw = wb.subset(keep)
        sess = rng.integers(1, 5, sw.num_reqs).astype(np.int32)
        case.insert_session(sw, sess, rep)
        assert rep.ok, rep.notes[:6]
        # readers: follow-up turns of those sessions (a writer's prompt, then new tokens) and other readers
        follow = []
        for r in range(min(sw.num_reqs, 3)):
            base = sw.tokens[sw.offsets[r]:sw.offsets[r + 1]]
            cut = int(rng.integers(1, len(base) + 1))
            t = np.concatenate([base[:cut], rng.integers(0, 9, int(rng.integers(0, 30)))]).astype(np.int32)
            follow.append(Batch(tokens=t, offsets=np.array([0, len(t)], np.int64), mask=np.zeros(len(t), np.uint8),
                                writer_ids=np.array([90000 + r], np.int64)))
        rr = pack_batches(follow + [rb])
        reader_sess = np.concatenate([sess[:len(follow)], rng.integers(0, 5, rb.num_reqs)]).astype(np.int32)
        case.match_and_gather(rr, rep, sessions=reader_sess)
        assert rep.ok, rep.notes[:6]
    assert rep.stats.get("session_stored", 0) > 0 and rep.stats.get("hits", 0) > 0


def test_gpu_private_entries_leak_nothing_to_other_users():
    import paper_2605_23640_b200 as cp
    for seed in range(6):
        wl = P.make_workload(seed)
        wb = wl.writers
        cfg = cp.IndexConfig(num_layers=1, num_kv_heads=1, head_dim=16, dtype="fp32", rope_theta=1e4, window_len=P.W,
                             pool_capacity_tokens=1 << 16, max_entries=4096, max_span_len=256, max_req_tokens=256,
                             max_batch_reqs=1 << 19, max_batch_tokens=1 << 23, max_spans_per_insert=64, max_sessions=64)
        idx = cp.KVIndex(cfg)
        nb = [(int(n) + 15) // 16 for n in wb.lens]
        bt = torch.zeros((wb.num_reqs, max(nb)), dtype=torch.int32)
        o = 0
        for r, k in enumerate(nb):
            bt[r, :k] = torch.arange(o, o + k); o += k
        kv = cp.PagedKV.allocate(1, o, 1, 16, torch.float32, bt)
        sess = np.arange(1, wb.num_reqs + 1, dtype=np.int32)
        db = cp.DeviceBatch.from_numpy(wb.tokens, wb.offsets, wb.mask, session=sess)
        sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda() for a in (wb.span_req, wb.span_begin, wb.span_len)]
        idx.insert(db, kv, *sp, None, None, 1)
        idx.insert_session(db, kv, 2)
        assert idx.last_error() == 0
        orc = O.OracleIndex(P.W, 42, 1 << 16, (1 << 16) // 16 + (1 << 16) // P.W + 64)
        assert orc.insert(wb, t=1)[0] == 0 and orc.insert_session(wb, sess, t=2)[0] == 0
        for who in (0, 63):
            def R(batch, who=who):
                ss = np.full(batch.num_reqs, who, np.int32)
                h = idx.match_spans(cp.DeviceBatch.from_numpy(batch.tokens, batch.offsets, None, session=ss), 3,
                                    no_touch=True, use_mask=False)
                g = (h.req_covered.cpu().numpy() > 0).astype(np.uint8)
                o_ = (orc.match(batch, t=3, no_touch=True, use_mask=False, sessions=ss).req_covered > 0).astype(np.uint8)
                assert np.array_equal(g, o_)
                return g
            rec, total, _ = P.attack(wl, R, "sensitive")
            assert total > 0 and rec == 0, (seed, who, rec)
