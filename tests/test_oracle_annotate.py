"""Pins for the oracle's C1 Steps 1-2 (summed-area table + optimal substring; PAPER.md L600-639,
SPEC.md sat/annotator L84-217).

Independent routes: numpy cumulative sums of the fixed-point matrix (SAT definition), SPEC worked
examples (all-ones 3x3, zero matrix, short segment, block-local attention), and an exhaustive
double-loop evaluation of the paper's IntraAttn/InterAttn equation for every
substring on tiny inputs.
"""
import numpy as np
import pytest

import oracle.oracle as O

ONE = 1 << 40


def q(A):
    """2^-40 fixed point with truncation toward zero (R#17), computed in Python big ints."""
    A = np.asarray(A, np.float32)
    return np.vectorize(lambda x: int(np.float64(x) * ONE), otypes=[object])(A)


def test_sat_spec_examples():
    T = O.sat(np.ones((3, 3), np.float32))
    assert (T[1:, 1:] == np.array([[1, 2, 3], [2, 4, 6], [3, 6, 9]]) * ONE).all()
    assert (O.sat(np.zeros((5, 5), np.float32)) == 0).all()
    rng = np.random.default_rng(0)
    A = np.tril(rng.uniform(0, 1, (8, 8))).astype(np.float32)
    T = O.sat(A)
    ref = np.cumsum(np.cumsum(q(A).astype(np.int64), axis=0), axis=1)
    assert (T[1:, 1:] == ref).all()
    # rect with x1 = y1 = 1 is exactly T[x2, y2]; 1x1 rects recover the entries
    qa = q(A)
    for i in range(1, 9):
        for j in range(1, 9):
            assert T[i, j] - T[i - 1, j] - T[i, j - 1] + T[i - 1, j - 1] == qa[i - 1, j - 1]


def brute(A, mask, min_len):
    """Exhaustive: every substring of every coarse segment, IntraAttn/InterAttn by the equation."""
    qa = q(A)
    n = len(mask)
    out = []
    i = 0
    while i < n:
        if mask[i]:
            i += 1
            continue
        a = i
        while i < n and not mask[i]:
            i += 1
        b = i - 1
        best = None
        for l in range(a, b + 1):
            for r in range(l + min_len - 1, b + 1):
                intra = sum(qa[x, y] for x in range(l, r + 1) for y in range(l, x + 1))
                inter = sum(qa[x, y] for x in range(l, r + 1) for y in range(0, l))
                key = (intra - inter, r - l + 1, -l)
                if best is None or key > best[0]:
                    best = (key, l, r)
        if best is None or best[0][0] <= 0:
            out.append((-1, -1, 0))
        else:
            out.append((best[1], best[2], best[0][0]))
    return out


def causal_stochastic(n, rng):
    A = np.tril(rng.uniform(0.0, 1.0, (n, n)) ** 3)
    return (A / A.sum(1, keepdims=True)).astype(np.float32)


def test_select_reusable_examples():
    rng = np.random.default_rng(1)
    A = causal_stochastic(24, rng)
    m = np.zeros(24, np.uint8)
    m[4] = 1
    m[21] = 1
    got = O.annotate(A, m, 4)
    assert got == brute(A, m, 4)                           # S:L177 random 24-token matrix, min_len 4
    assert got[1][0] >= 5 and got[1][1] <= 20               # span inside seg (5, 20) [0-based]
    assert got[2] == (-1, -1, 0)                            # segment shorter than min_len
    # block-local attention, min_len 1: the whole segment, score = |seg|
    I = np.eye(12, dtype=np.float32)
    m2 = np.zeros(12, np.uint8); m2[5] = 1
    assert O.annotate(I, m2, 1) == [(0, 4, 5 * ONE), (6, 11, 6 * ONE)]
    # all-sensitive -> no segments
    assert O.annotate(I, np.ones(12, np.uint8), 1) == []


@pytest.mark.parametrize("seed", range(12))
def test_oracle_equivalence_small(seed):                   # n <= 48 vs exhaustive reference
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(4, 49))
    A = causal_stochastic(n, rng)
    if seed % 3 == 0:
        A = np.tril(rng.uniform(0, 1, (n, n))).astype(np.float32)         # non-row-stochastic (R#27)
    mask = (rng.random(n) < 0.15).astype(np.uint8)
    min_len = int(rng.integers(1, 6))
    assert O.annotate(A, mask, min_len) == brute(A, mask, min_len)


def test_segment_starting_at_position_one_is_selected_whole():
    """Prefix-reuse special case: with inter = 0 for l = 1 and every row adding a
    positive amount, the first coarse segment selects its whole length."""
    rng = np.random.default_rng(3)
    for n in (30, 64):
        A = causal_stochastic(n, rng)
        m = np.zeros(n, np.uint8); m[n - 7] = 1
        got = O.annotate(A, m, 5)
        assert got[0][:2] == (0, n - 8)
