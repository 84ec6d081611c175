"""Pins for the oracle's RoPE re-rotation (readings R#11-13; the paper is silent on RoPE)
and recompute score / top-k.

Independent routes: numpy complex exponentials (RoPE as multiplication by
e^{i*p*theta}), group identities R(a)R(b) = R(a+b) and R(d)R(-d) = I,
closed-form single-pair values, math.fsum scores, lexsort top-k, and the
closed forms of SPEC.md L184-186.
"""
import math

import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import bf16_round_np, payload_np


def rope_complex(x, pos, theta, H, d):
    """NeoX rotation written as complex multiplication: (x_i + i x_{i+d/2}) * exp(i pos theta_i)."""
    x = np.asarray(x, np.float64).reshape(H, d)
    z = x[:, :d // 2] + 1j * x[:, d // 2:]
    th = theta ** (-np.arange(d // 2) * 2.0 / d)
    z = z * np.exp(1j * pos * th)
    return np.concatenate([z.real, z.imag], axis=1).reshape(-1)


def test_delta_zero_is_bit_copy():
    x = np.array([-0.0, 1.5, np.float32(1e-30), -3.25] * 32, np.float32)
    y = O.rerotate_row(x, 2, 64, 10000.0, 0, bf16=False)
    assert y.tobytes() == x.tobytes()                      # -0.0 preserved (R#13)


def test_single_pair_closed_form():
    # d = 2: one pair, theta_0 = base^0 = 1, so the angle is delta itself
    for delta in [1, -1, 5, 1000, -8191]:
        y = O.rerotate_row(np.array([1.0, 0.0], np.float32), 1, 2, 500000.0, delta, bf16=False)
        assert y[0] == np.float32(math.cos(delta)) and y[1] == np.float32(math.sin(delta))


@pytest.mark.parametrize("H,d,theta", [(2, 64, 10000.0), (8, 128, 500000.0), (1, 128, 500000.0)])
def test_matches_complex_rope_and_group_laws(H, d, theta):
    rng = np.random.default_rng(H * d)
    for trial in range(8):
        x = rng.uniform(-2, 2, H * d).astype(np.float32)
        a, b = (int(v) for v in rng.integers(-8192, 8192, 2))
        ra = O.rerotate_row(x, H, d, theta, a, bf16=False)
        ref = rope_complex(x, a, theta, H, d)
        assert np.max(np.abs(ra - ref)) <= 2e-7 * max(1.0, np.max(np.abs(ref)))
        # R(a) R(b) = R(a + b) and R(d) R(-d) = I  (fp32 rounding only)
        rab = O.rerotate_row(ra, H, d, theta, b, bf16=False)
        rsum = O.rerotate_row(x, H, d, theta, a + b, bf16=False)
        assert np.max(np.abs(rab - rsum)) <= 1e-6
        back = O.rerotate_row(ra, H, d, theta, -a, bf16=False)
        assert np.max(np.abs(back - x)) <= 1e-6
        # pair norms preserved
        xr = x.reshape(H, d).astype(np.float64); yr = ra.reshape(H, d).astype(np.float64)
        n0 = xr[:, :d // 2] ** 2 + xr[:, d // 2:] ** 2
        n1 = yr[:, :d // 2] ** 2 + yr[:, d // 2:] ** 2
        assert np.max(np.abs(n0 - n1)) <= 1e-5


def test_gptj_is_permuted_neox():
    H, d = 2, 64
    rng = np.random.default_rng(5)
    x = rng.uniform(-2, 2, H * d).astype(np.float32)
    perm = np.concatenate([np.arange(0, d, 2), np.arange(1, d, 2)])       # gptj (2i, 2i+1) -> neox (i, i+d/2)
    xp = x.reshape(H, d)[:, perm].reshape(-1)
    y_neox = O.rerotate_row(xp, H, d, 10000.0, 123, bf16=False)
    y_gptj = O.rerotate_row(x, H, d, 10000.0, 123, bf16=False, gptj=True)
    assert np.array_equal(y_gptj.reshape(H, d)[:, perm].reshape(-1), y_neox)


def test_bf16_rounding_is_single_rne():
    x = np.array([1.0, 0.0], np.float32)
    y = O.rerotate_row(x, 1, 2, 10000.0, 1, bf16=True)
    assert y[0] == bf16_round_np(np.array([math.cos(1)], np.float32))[0]   # cos(1)=0.5403 -> 0.5390625
    assert y[1] == np.float32(0.83984375)                                   # sin(1)=0.8415 -> bf16


def test_fresh_prefill_pin():
    """Writer K at origin p is R(p) k_raw (rounded to bf16); after re-rotation by delta = q - p the
    key must equal R(q) k_raw up to two bf16 roundings, independent of the oracle's code path."""
    H, d, theta = 8, 128, 500000.0
    rng = np.random.default_rng(11)
    for trial in range(10):
        p, q = (int(v) for v in rng.integers(0, 8192, 2))
        kraw = payload_np(3, trial, 0, np.arange(H)[:, None], np.arange(d)[None], 0).reshape(-1)
        k_writer = bf16_round_np(rope_complex(kraw, p, theta, H, d).astype(np.float32))
        got = O.rerotate_row(k_writer, H, d, theta, q - p, bf16=True)
        want = rope_complex(kraw, q, theta, H, d)
        assert np.max(np.abs(got - want)) <= 2 * 0.0078125 + 1e-6       # <= 2 half-ulps at |k| < 4


# ---------------------------------------------------------------------------- score / top-k
def fsum_scores(A, l, r):
    return np.array([math.fsum(A[i, :l]) - math.fsum(A[i, l:i + 1]) for i in range(l, r + 1)])


def causal_stochastic(n, rng):
    A = np.tril(rng.uniform(0.01, 1.0, (n, n)))
    return (A / A.sum(1, keepdims=True)).astype(np.float32)


def test_rho_zero_and_one():
    rng = np.random.default_rng(0)
    A = causal_stochastic(50, rng)
    _, b0 = O.score(A, 10, 40, 0, 4)
    assert not O.bits_to_bool(b0, 31).any()
    _, b1 = O.score(A, 10, 40, 4, 4)
    assert O.bits_to_bool(b1, 31).all()


def test_score_equals_fsum_and_row_stochastic_form():
    rng = np.random.default_rng(1)
    n = 200
    A = causal_stochastic(n, rng)
    l, r = 37, 180
    sc, _ = O.score(A, l, r)
    got = sc.astype(np.float64) / 2.0 ** 40
    ref = fsum_scores(A, l, r)
    assert np.max(np.abs(got - ref)) <= n * 2.0 ** -40 * 2
    # row-stochastic causal A: intra = rowsum - inter, so score = 2*inter - rowsum (~ 2*inter - 1)
    inter = np.array([math.fsum(A[i, :l]) for i in range(l, r + 1)])
    rows = np.array([math.fsum(A[i, :i + 1]) for i in range(l, r + 1)])
    assert np.max(np.abs(got - (2 * inter - rows))) <= n * 2.0 ** -39
    assert np.max(np.abs(rows - 1.0)) < 1e-5


@pytest.mark.parametrize("seed", range(5))
def test_topk_is_sorted_selection(seed):
    rng = np.random.default_rng(10 + seed)
    n = int(rng.integers(40, 300))
    heads = int(rng.integers(1, 4))
    A = np.stack([causal_stochastic(n, rng) for _ in range(heads)])
    l = int(rng.integers(0, n // 2)); r = int(rng.integers(l, n))
    num, den = [(1, 4), (1, 10), (3, 7), (1, 3)][seed % 4]
    sc, bits = O.score(A, l, r, num, den)
    m = r - l + 1
    ref = sum(fsum_scores(A[h], l, r) for h in range(heads))
    order = np.lexsort((np.arange(m), -sc))            # score desc, index asc
    k = -(-num * m // den)
    exp = np.zeros(m, bool); exp[order[:k]] = True
    assert np.array_equal(O.bits_to_bool(bits, m), exp)
    # ranks by the exact fixed-point score agree with the fsum ranking up to 2^-39-close pairs
    top = np.sort(ref[exp]); rest = np.sort(ref[~exp])
    if len(top) and len(rest):
        assert top[0] >= rest[-1] - heads * n * 2.0 ** -39


def test_ties_take_smaller_index_and_ceil_rule():
    # segment-local attention: nothing before l, so every token's inter is 0; all mass on the
    # diagonal makes intra = 1 exactly for every i -> all scores tie -> the first ceil(rho*m)
    # indices.
    n, l, r = 64, 10, 39
    A = np.eye(n, dtype=np.float32)
    sc, bits = O.score(A, l, r, 1, 10)                 # m = 30, rho = 1/10 -> k = 3 exactly (R#15)
    got = O.bits_to_bool(bits, 30)
    assert list(np.nonzero(got)[0]) == [0, 1, 2]


def test_hand_example():
    # 3x3 causal matrix, span [1, 2]: score_1 = A10 - A11, score_2 = A20 - (A21 + A22)
    A = np.array([[1, 0, 0], [0.75, 0.25, 0], [0.5, 0.25, 0.25]], np.float32)
    sc, bits = O.score(A, 1, 2, 1, 2)
    assert list(sc) == [int(0.5 * 2 ** 40), 0]
    assert list(O.bits_to_bool(bits, 2)) == [True, False]
