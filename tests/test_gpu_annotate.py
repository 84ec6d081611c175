"""GPU parity for NEXT-1, the on-device KV Annotator (C1 Steps 1-2):
cp_annotate_spans vs the oracle's summed-area-table search, bit exact (spans and fixed-point
scores), on random causal matrices with random masks and on config-2-shaped writer attention."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle.oracle as O  # noqa: E402
import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import attention_torch, make_workload  # noqa: E402


def _run(mats, masks, heads, min_len, max_segments=64):
    dA = [torch.from_numpy(np.ascontiguousarray(A, np.float32)).cuda() for A in mats]
    dM = [torch.from_numpy(np.ascontiguousarray(m, np.uint8)).cuda() for m in masks]
    return cp.annotate_spans(dA, dM, heads, min_len=min_len, max_segments=max_segments)


@pytest.mark.parametrize("variant", ["0", "1", "2"])     # auto / flat (thread per start) / split rows
@pytest.mark.parametrize("seed", range(4))
def test_random_causal_matrices(seed, variant, monkeypatch):
    monkeypatch.setenv("CP_ANN_VARIANT", variant)
    rng = np.random.default_rng(seed)
    mats, masks, heads, exp = [], [], [], []
    min_len = [1, 3, 8, 17][seed]
    for _ in range(12):
        n = int(rng.integers(1, 300))
        h = int(rng.integers(1, 3))
        A = np.tril(rng.uniform(0, 1, (h, n, n)) ** 2).astype(np.float32)
        if rng.random() < 0.5:
            A /= A.sum(-1, keepdims=True)
        m = (rng.random(n) < rng.uniform(0, 0.1)).astype(np.uint8)
        mats.append(A); masks.append(m); heads.append(h)
        exp.append(O.annotate(A, m, min_len))
    got = _run(mats, masks, heads, min_len)
    assert got == exp


def test_config2_writer_attention():
    wl = make_workload(2, scale=0.05)
    wb, _ = wl.rounds[0]
    mats, masks = [], []
    for r in range(wb.num_reqs):
        A = attention_torch(int(wb.lens[r]), wb.segments[r], 0.01, seed=r)
        mats.append(A)
        masks.append(torch.from_numpy(wb.req_mask(r).copy()).cuda())
    got = cp.annotate_spans(mats, masks, [1] * len(mats), min_len=128)
    for r in range(wb.num_reqs):
        exp = O.annotate(mats[r].cpu().numpy(), wb.req_mask(r), 128)
        assert got[r] == exp, r
    # every reported span lies inside its coarse segment and respects min_len
    for r in range(wb.num_reqs):
        for (l, rr, d) in got[r]:
            if l >= 0:
                assert rr - l + 1 >= 128 and d > 0 and not wb.req_mask(r)[l:rr + 1].any()


def test_all_masked_and_short():
    I = np.eye(40, dtype=np.float32)
    got = _run([I, I, I], [np.ones(40, np.uint8), np.zeros(40, np.uint8), np.zeros(40, np.uint8)], [1, 1, 1], 50)
    assert got == [[], [(-1, -1, 0)], [(-1, -1, 0)]]


@pytest.mark.parametrize("variant", ["1", "2"])
def test_many_segments_beside_long_request(variant, monkeypatch):
    """A short request with hundreds of coarse segments in the same call as a long one: the partial
    bests of each request stay inside its own workspace slice (stride ceil(n/32) per segment)."""
    monkeypatch.setenv("CP_ANN_VARIANT", variant)
    rng = np.random.default_rng(11)
    mats, masks, heads, exp = [], [], [], []
    for n, alt in ((2600, False), (700, True), (1900, False), (650, True)):
        A = np.tril(rng.uniform(0, 1, (1, n, n))).astype(np.float32)
        m = np.zeros(n, np.uint8)
        if alt:
            m[1::3] = 1                                  # ~n/3 segments of 2 tokens
        else:
            m[rng.integers(0, n, 6)] = 1
        mats.append(A); masks.append(m); heads.append(1)
        exp.append(O.annotate(A, m, 1))
    got = _run(mats, masks, heads, 1, max_segments=256)
    assert got == exp


@pytest.mark.parametrize("n", [7500, 10000])
def test_long_requests_at_the_timed_sizes(n):
    """The 7.5K / 10K-token requests the annotator is timed at (M6 sizes): row-stochastic
    segment-local attention plus a perturbation that makes the optimal span a strict sub-range of its
    segment, two masked runs; bit exact against the oracle's summed-area-table search."""
    g = torch.Generator(device="cuda").manual_seed(n)
    segs = [(0, 1000), (1003, 4000), (4002, n)]
    A = attention_torch(n, segs, 0.01, seed=n)
    A = A * (1.0 + 0.5 * torch.rand(A.shape, generator=g, device="cuda")).tril()
    A = (A / A.sum(-1, keepdim=True)).contiguous()                 # rows still sum to 1 (domain, header)
    m = np.zeros(n, np.uint8); m[1000:1003] = 1; m[4000:4002] = 1
    got = cp.annotate_spans([A], [torch.from_numpy(m).cuda()], [1], min_len=128)[0]
    exp = O.annotate(A.cpu().numpy(), m, 128)
    assert got == exp
    assert len(got) == 3 and all(l >= 0 for l, _, _ in got)
