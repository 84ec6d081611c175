"""Privacy pin end to end on the GPU path: the index built by cp_index_insert and probed through
cp_match_spans gives, probe for probe, the same binary reuse signal as the oracle, and the exhaustive
desk-scale attack of tests/privacy_probe.py recovers no sensitive token on 50 seeded workloads (PAPER
Table 4: "Direct Recovery" 0%; SPEC acceptance 1), while recovery of
detector-missed tokens grows with the miss rate (SPEC acceptance 2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle.oracle as O  # noqa: E402
from tests import privacy_probe as P  # noqa: E402


def _gpu_index(wl):
    import paper_2605_23640_b200 as cp
    wb = wl.writers
    cfg = cp.IndexConfig(num_layers=1, num_kv_heads=1, head_dim=16, dtype="fp32", rope_theta=10000.0,
                         window_len=P.W, pool_capacity_tokens=1 << 16, max_entries=4096, max_span_len=256,
                         max_req_tokens=256, max_batch_reqs=1 << 19, max_batch_tokens=1 << 23,
                         max_spans_per_insert=max(1, len(wb.span_len)))
    idx = cp.KVIndex(cfg)
    nb = [(int(n) + 15) // 16 for n in wb.lens]
    bt = torch.zeros((wb.num_reqs, max(nb)), dtype=torch.int32)
    o = 0
    for r, k in enumerate(nb):
        bt[r, :k] = torch.arange(o, o + k); o += k
    kv = cp.PagedKV.allocate(1, o, 1, 16, torch.float32, bt)
    db = cp.DeviceBatch.from_numpy(wb.tokens, wb.offsets, wb.mask)
    sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda() for a in (wb.span_req, wb.span_begin, wb.span_len)]
    idx.insert(db, kv, *sp, None, None, 1)
    assert idx.last_error() == 0
    return idx, cp


def _reuse_gpu(idx, cp):
    def R(batch):
        db = cp.DeviceBatch.from_numpy(batch.tokens, batch.offsets, None)
        h = idx.match_spans(db, 2, no_touch=True, use_mask=False)
        assert idx.last_error() == 0
        return (h.req_covered.cpu().numpy() > 0).astype(np.uint8)
    return R


def _reuse_oracle(wl):
    idx = O.OracleIndex(P.W, 42, 1 << 16, (1 << 16) // 16 + (1 << 16) // P.W + 64)
    assert idx.insert(wl.writers, t=1)[0] == 0

    def R(batch):
        return (idx.match(batch, t=2, no_touch=True, use_mask=False).req_covered > 0).astype(np.uint8)
    return R


@pytest.mark.parametrize("block", range(5))
def test_gpu_reuse_oracle_leaks_no_sensitive_token(block):
    for seed in range(10 * block, 10 * block + 10):
        wl = P.make_workload(seed)
        idx, cp = _gpu_index(wl)
        Rg, Ro = _reuse_gpu(idx, cp), _reuse_oracle(wl)
        seen = []

        def both(batch):
            g, o = Rg(batch), Ro(batch)
            assert np.array_equal(g, o), f"seed {seed}: GPU and oracle reuse signals differ"
            seen.append(int(g.sum()))
            return g
        rec, total, probes = P.attack(wl, both, "sensitive")
        assert total > 0 and probes > 0
        assert rec == 0, f"seed {seed}: {rec}/{total} sensitive tokens recovered through cp_match_spans"


def test_gpu_positive_control_recovers_public_tokens():
    """The same attack through cp_match_spans recovers public tokens inside stored segments (and the
    GPU signal equals the oracle's on those probes too)."""
    got = tot = 0
    for seed in range(6):
        wl = P.make_workload(seed)
        idx, cp = _gpu_index(wl)
        Rg, Ro = _reuse_gpu(idx, cp), _reuse_oracle(wl)

        def both(batch):
            g = Rg(batch)
            assert np.array_equal(g, Ro(batch))
            return g
        rec, total, _ = P.attack(wl, both, "public")
        got += rec; tot += total
    assert tot > 0 and got / tot > 0.5, (got, tot)


def test_gpu_false_negative_sweep_is_monotone():
    rates = []
    for fn in (0.0, 0.05, 0.10, 0.15, 0.20):
        wl = P.make_workload(100, n_writers=8, fn_rate=fn)
        idx, cp = _gpu_index(wl)
        rec, total, _ = P.attack(wl, _reuse_gpu(idx, cp), "sensitive")
        rates.append(rec / total)
    assert rates[0] == 0.0 and rates[-1] > 0.0
    assert all(a <= b for a, b in zip(rates, rates[1:])), rates
