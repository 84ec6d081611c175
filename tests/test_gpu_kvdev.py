"""GPU parity for NEXT-4, CacheBlend's KV-deviation selector (R#30):
cp_score_kv_deviation vs the oracle, bit exact on deviations and selection bits.  Paged caches with
random block tables (reused and fresh tables differ), ragged span lengths (1 .. 2000, several spans
per request, spans not page aligned), bf16 Llama-3-8B geometry and fp32 toy geometry, ties."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle.oracle as O  # noqa: E402
import paper_2605_23640_b200 as cp  # noqa: E402


def _paged(rng, lens, H, d, dtype, gen):
    nb = [(n + 15) // 16 for n in lens]
    perm = torch.from_numpy(rng.permutation(sum(nb)).astype(np.int32))
    bt = torch.zeros((len(lens), max(nb)), dtype=torch.int32)
    o = 0
    for r, k in enumerate(nb):
        bt[r, :k] = perm[o:o + k]
        o += k
    K = torch.randn((sum(nb), 16, H, d), generator=gen, device="cuda").to(dtype)
    V = torch.randn((sum(nb), 16, H, d), generator=gen, device="cuda").to(dtype)
    return K, V, bt.cuda()


def _rows(K, bt, r, lo, hi):
    """Rows [lo, hi] of request r as fp32 numpy [m, H*d] (exact widening; plumbing only)."""
    q = torch.arange(lo, hi + 1, device=K.device)
    blk = bt[r, q // 16].long()
    return K[blk, q % 16].float().reshape(len(q), -1).cpu().numpy()


@pytest.mark.parametrize("H,d,dtype", [(8, 128, torch.bfloat16), (2, 64, torch.float32), (1, 8, torch.bfloat16)])
def test_kv_deviation_random(H, d, dtype):
    rng = np.random.default_rng(H * 1000 + d)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    lens = [1, 40, 517, 2100, 300]
    rK, rV, rbt = _paged(rng, lens, H, d, dtype, gen)
    fK, fV, fbt = _paged(rng, lens, H, d, dtype, gen)
    # fresh = reused (through each side's block table) except on a random subset of tokens, so that
    # many deviations tie at 0 and the rest vary in size
    for r, n in enumerate(lens):
        q = torch.arange(n, device="cuda")
        rb, fb = rbt[r, q // 16].long(), fbt[r, q // 16].long()
        keep = torch.from_numpy(rng.random(n) < 0.6).cuda()
        scale = torch.from_numpy(rng.uniform(0, 0.3, n).astype(np.float32)).cuda()[:, None, None]
        base_k, base_v = rK[rb, q % 16].float(), rV[rb, q % 16].float()
        noise_k = torch.randn(base_k.shape, generator=gen, device="cuda") * scale
        noise_v = torch.randn(base_v.shape, generator=gen, device="cuda") * scale
        fK[fb, q % 16] = torch.where(keep[:, None, None], base_k, base_k + noise_k).to(dtype)
        fV[fb, q % 16] = torch.where(keep[:, None, None], base_v, base_v + noise_v).to(dtype)
    spans = [(0, 0, 0), (1, 3, 39), (2, 0, 516), (2, 5, 5), (3, 17, 2016), (3, 2050, 2099), (4, 0, 299)]
    req, ls, rs = zip(*spans)
    for num, den in [(3, 20), (1, 4), (0, 20), (20, 20)]:
        dev, bits, so, bo = cp.score_kv_deviation(req, ls, rs, rK, rV, rbt, fK, fV, fbt, num, den)
        dev, bits = dev.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
        for s, (r, lo, hi) in enumerate(spans):
            m = hi - lo + 1
            od, ob = O.kv_deviation(_rows(rK, rbt, r, lo, hi), _rows(rV, rbt, r, lo, hi),
                                    _rows(fK, fbt, r, lo, hi), _rows(fV, fbt, r, lo, hi), num, den)
            assert np.array_equal(dev[so[s]:so[s] + m], od), (s, num, den)
            assert np.array_equal(bits[bo[s]:bo[s] + (m + 31) // 32], ob), (s, num, den)


def test_kv_deviation_identical_caches_selects_first_tokens():
    rng = np.random.default_rng(0)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    K, V, bt = _paged(rng, [700], 8, 128, torch.bfloat16, gen)
    dev, bits, so, bo = cp.score_kv_deviation([0], [100], [699], K, V, bt, K, V, bt)
    assert not dev.cpu().numpy().any()
    m, k = 600, -(-3 * 600 // 20)
    exp = np.zeros((m + 31) // 32, np.uint32)
    for i in range(k):
        exp[i // 32] |= np.uint32(1 << (i % 32))
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), exp)


def test_kv_deviation_rejects_bad_arguments_without_launch():
    rng = np.random.default_rng(0)
    gen = torch.Generator(device="cuda")
    K, V, bt = _paged(rng, [40], 2, 64, torch.float32, gen)
    with pytest.raises(Exception):
        cp.score_kv_deviation([0], [0], [48], K, V, bt, K, V, bt)        # beyond the block table
    with pytest.raises(Exception):
        cp.score_kv_deviation([0], [5], [4], K, V, bt, K, V, bt)         # empty span
