"""Pins for the oracle's CacheBlend KV-deviation selector (NEXT-4; R#30).

The paper gives no norm, so the definition (L1 over K and V in 2^-24 fixed point, trunc toward zero)
is a reading; these tests pin the oracle against facts that do not restate its code: closed forms on
constructed inputs, the metric axioms, the truncation special cases, and the selection rule against
numpy's lexsort (a different algorithm)."""
import numpy as np
import pytest

import oracle.oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")
U = 2.0 ** -24                      # one fixed-point unit


def rows(rng, m, w, scale=2.0 ** -10):
    """fp32 rows that are integer multiples of 2^-10 (so of 2^-24): q24 is exact on them."""
    return (rng.integers(-4096, 4096, size=(m, w)) * scale).astype(np.float32)


def first_k_bits(order, m, k):
    bits = np.zeros((m + 31) // 32, np.uint32)
    for i in order[:k]:
        bits[i // 32] |= np.uint32(1 << (i % 32))
    return bits


def test_identical_caches_all_ties_first_indices():
    rng = np.random.default_rng(0)
    K, V = rows(rng, 70, 32), rows(rng, 70, 32)
    dev, bits = O.kv_deviation(K, V, K, V, 3, 20)
    assert not dev.any()
    k = -(-3 * 70 // 20)                                 # ceil(0.15 * 70) = 11
    assert np.array_equal(bits, first_k_bits(np.arange(70), 70, k))


def test_constructed_offsets_closed_form_and_selection():
    rng = np.random.default_rng(1)
    m, w = 45, 24
    K, V = rows(rng, m, w, 2.0 ** -16), rows(rng, m, w, 2.0 ** -16)     # |x| <= 2^-4: offsets stay exact
    c = rng.permutation(np.arange(1, m + 1)).astype(np.int64)        # distinct per-token offsets (units)
    sign = rng.choice([-1.0, 1.0], size=(m, w))
    Kf = (K.astype(np.float64) + sign * c[:, None] * U).astype(np.float32)
    Vf = (V.astype(np.float64) - 3 * sign * c[:, None] * U).astype(np.float32)
    assert np.array_equal(Kf.astype(np.float64) - K, sign * c[:, None] * U)      # offsets exact in fp32
    dev, bits = O.kv_deviation(K, V, Kf, Vf, 1, 4)
    assert np.array_equal(dev, 4 * w * c)                # |c| per K element + |3c| per V element
    k = -(-m // 4)
    assert np.array_equal(bits, first_k_bits(np.argsort(-c, kind="stable"), m, k))


def test_metric_axioms():
    rng = np.random.default_rng(2)
    m, w = 33, 16
    A = [(rng.standard_normal((m, w)) * 3).astype(np.float32) for _ in range(6)]
    dab, _ = O.kv_deviation(A[0], A[1], A[2], A[3])
    dba, _ = O.kv_deviation(A[2], A[3], A[0], A[1])
    assert np.array_equal(dab, dba)                                           # symmetry
    dbc, _ = O.kv_deviation(A[2], A[3], A[4], A[5])
    dac, _ = O.kv_deviation(A[0], A[1], A[4], A[5])
    assert (dac <= dab + dbc).all()                                           # triangle inequality
    assert (dab >= 0).all()
    # K and V enter symmetrically: swapping them in both caches changes nothing
    dswap, _ = O.kv_deviation(A[1], A[0], A[3], A[2])
    assert np.array_equal(dab, dswap)


def test_truncation_toward_zero_special_cases():
    z = np.zeros((1, 4), np.float32)
    x = np.array([[2.0 ** -25, -(2.0 ** -25), 1.5 * U, -1.5 * U]], np.float32)
    dev, _ = O.kv_deviation(x, z, z, z, 1, 1)
    assert dev.tolist() == [0 + 0 + 1 + 1]              # |trunc(0.5)| = 0, |trunc(+-1.5)| = 1
    big = np.array([[1000.0, -1000.0, 0.0, 0.0]], np.float32)
    dev, _ = O.kv_deviation(big, z, z, z, 1, 1)
    assert dev.tolist() == [2000 * 2 ** 24]


def test_selection_matches_lexsort_and_rho_limits():
    rng = np.random.default_rng(3)
    for m in (1, 7, 32, 33, 100):
        K, V, Kf, Vf = (rows(rng, m, 8, 2.0 ** -4) for _ in range(4))
        Kf[: m // 2] = K[: m // 2]; Vf[: m // 2] = V[: m // 2]          # force ties at zero
        for num, den in ((0, 20), (3, 20), (1, 4), (20, 20), (1, 3)):
            dev, bits = O.kv_deviation(K, V, Kf, Vf, num, den)
            k = -(-num * m // den)
            order = np.lexsort((np.arange(m), -dev))
            assert np.array_equal(bits, first_k_bits(order, m, k)), (m, num, den)
