"""The matcher's work is O(n + c) ("the retriever scans each request once ... and
verifies only the c candidates that pass the prefix filter"; SPEC acceptance 10: window-scan
counts fit c * n).  cp_index_match_work counts, per call: windows probed, prefix-filter candidates c,
candidates that pass the O(1) full-hash pre-check, and the tokens their verification may compare.
Pinned here against what the workload fixes: windows = sum (n - w + 1) exactly (linear in n, the
constant is 1), candidates = sum of the per-request counts the matcher reports, full-hash-passed =
the number of request offsets where some stored segment occurs (brute-force search: no false
positive reaches verification), verification tokens = the total length of those occurrences."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _setup(seed=0, n_seg=1000, w=128):
    import paper_2605_23640_b200 as cp
    rng = np.random.default_rng(seed)
    segs = [rng.integers(1000, 120000, int(rng.integers(w, 4 * w))).astype(np.int32) for _ in range(n_seg)]
    toks = np.concatenate(segs)
    offs = np.concatenate([[0], np.cumsum([len(s) for s in segs])]).astype(np.int64)
    cfg = cp.IndexConfig(num_layers=1, num_kv_heads=1, head_dim=16, dtype="fp32", rope_theta=1e4, window_len=w,
                         pool_capacity_tokens=1 << 21, max_entries=8192, max_span_len=4 * w, max_req_tokens=8192,
                         max_batch_reqs=n_seg, max_batch_tokens=int(offs[-1]) + 8192 * 8, max_spans_per_insert=n_seg)
    idx = cp.KVIndex(cfg)
    nb = [(len(s) + 15) // 16 for s in segs]
    bt = torch.zeros((n_seg, max(nb)), dtype=torch.int32)
    o = 0
    for r, k in enumerate(nb):
        bt[r, :k] = torch.arange(o, o + k); o += k
    kv = cp.PagedKV.allocate(1, o, 1, 16, torch.float32, bt)
    db = cp.DeviceBatch.from_numpy(toks, offs, np.zeros(len(toks), np.uint8))
    sp = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    idx.insert(db, kv, sp(list(range(n_seg))), sp([0] * n_seg), sp([len(s) for s in segs]), None, None, 1)
    assert idx.last_error() == 0
    return cp, idx, segs, rng, w


def test_matcher_work_is_linear_in_n_plus_c():
    cp, idx, segs, rng, w = _setup()
    by_prefix = {}
    for s in segs:
        by_prefix.setdefault(s[:w].tobytes(), []).append(s)
    per_n = {}
    for n in (512, 1024, 2048, 4096, 8192):
        reqs = []
        for _ in range(16):
            r = rng.integers(1000, 120000, n).astype(np.int32)
            for _ in range(n // 1024 + 1):                      # plant stored segments
                s = segs[int(rng.integers(0, len(segs)))]
                if len(s) < n:
                    k = int(rng.integers(0, n - len(s) + 1))
                    r[k:k + len(s)] = s
            reqs.append(r)
        toks = np.concatenate(reqs)
        offs = np.arange(0, n * 17, n, dtype=np.int64)[:17]
        db = cp.DeviceBatch.from_numpy(toks, offs, None)
        idx.match_work(reset=True)
        h = idx.match_spans(db, 2, no_touch=True, use_mask=False)
        win, cand, passed, vtok = idx.match_work()
        assert win == 16 * (n - w + 1)
        assert cand == int(h.req_candidates.sum().item())
        # brute force: offsets where some stored segment occurs, and their lengths
        occ, occ_tok = 0, 0
        for r in reqs:
            for k in range(n - w + 1):
                cands = by_prefix.get(r[k:k + w].tobytes())
                if not cands:
                    continue
                found = [len(s) for s in cands if k + len(s) <= n and np.array_equal(r[k:k + len(s)], s)]
                if found:
                    occ += 1
                    occ_tok += found[0]          # the pool is containment-free: one segment per offset
        assert passed == occ, (n, passed, occ)
        assert vtok == occ_tok
        per_n[n] = win / (16 * n)
    # window scans per request token: the same constant at every n (within the n - w + 1 edge term)
    ratios = [per_n[n] * n / (n - w + 1) for n in per_n]
    assert max(ratios) - min(ratios) < 1e-12
