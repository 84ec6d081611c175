"""Pins for the oracle's hashing.

Independent routes: Python arbitrary-precision integers (a textbook modmul), the
rolling recurrence of SPEC.md L256-259 (different algorithm from the oracle's
Horner fold), hashlib's SHA-256 and the FIPS 180-2 example digests.
"""
import hashlib
import os
import struct

import numpy as np

import oracle.oracle as O

P = (1 << 61) - 1
M64 = (1 << 64) - 1
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _py_splitmix(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _golden_lines(name):
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                lhs, rhs = line.split(" = ")
                yield lhs, rhs


def test_golden_hash_vectors():
    n = 0
    for lhs, rhs in _golden_lines("hash_vectors.txt"):
        kind, *kv = lhs.split()
        kv = dict(x.split("=") for x in kv)
        if kind == "base":
            assert O.hash_base(int(kv["seed"])) == int(rhs)
        elif kind == "prefix":
            B = O.hash_base(int(kv["seed"]))
            toks = [int(x) for x in kv["tokens"].split(",")]
            assert [int(v) for v in O.prefix_hashes(toks, B)] == [int(x) for x in rhs.split(",")]
        elif kind == "window":
            B = O.hash_base(int(kv["seed"]))
            lo, hi = (int(x) for x in kv["range"].split(".."))
            toks = np.arange(lo, hi + 1, dtype=np.int32)
            w, k = int(kv["w"]), int(kv["k"])
            assert O.poly_hash(toks[k:k + w], B) == int(rhs)
        elif kind == "mulmod":
            assert O.mulmod(int(kv["a"]), int(kv["b"])) == int(rhs)
        n += 1
    assert n == 9


def test_base_matches_bigint_splitmix_and_range():
    rng = np.random.default_rng(0)
    bases = set()
    for s in [0, 1, 2, 42, M64, 1 << 63] + [int(x) for x in rng.integers(0, 1 << 62, 100)]:
        B = O.hash_base(s)
        assert B == 2 + _py_splitmix(s) % (P - 3)
        assert 2 <= B <= P - 2
        bases.add(B)
    assert len(bases) >= 100          # SPEC.md L278 base randomization


def test_mulmod_vs_bigint():
    rng = np.random.default_rng(1)
    edge = [0, 1, P - 1, P, P + 1, (1 << 61), M64, M64 - 1, 1 << 63]
    vals = edge + [int(x) for x in rng.integers(0, 1 << 63, 300)] + [int(x) | (1 << 63) for x in rng.integers(0, 1 << 63, 100)]
    for i, a in enumerate(vals):
        b = vals[(i * 7 + 3) % len(vals)]
        assert O.mulmod(a, b) == (a * b) % P       # SPEC.md L277 "equals schoolbook big-integer result"


def _py_prefix(t, B):
    h = [0]
    for x in t:
        h.append((h[-1] * B + int(x) + 1) % P)
    return h


def test_prefix_array_closed_forms():
    B = O.hash_base(7)
    assert list(O.prefix_hashes([], B)) == [0]                       # S:L244 empty -> h=[0]
    for t in [0, 5, 128255, (1 << 31) - 2]:
        assert O.poly_hash([t], B) == (t + 1) % P                    # S:L245/L254 single token
    rng = np.random.default_rng(2)
    toks = rng.integers(0, 128256, 257).astype(np.int32)
    h = O.prefix_hashes(toks, B)
    assert [int(x) for x in h] == _py_prefix(toks, B)
    assert int(h[-1]) == O.poly_hash(toks, B)                        # S:L253 sub(1,n) = h[n]
    # every substring hash equals a from-scratch fold (textbook sum of powers)
    for l, r in [(1, 1), (1, 257), (5, 130), (100, 228), (257, 257), (20, 21)]:
        sub = (int(h[r]) - int(h[l - 1]) * pow(B, r - l + 1, P)) % P
        direct = sum((int(toks[k - 1]) + 1) * pow(B, r - k, P) for k in range(l, r + 1)) % P
        assert sub == direct == O.poly_hash(toks[l - 1:r], B)


def test_rolling_window_equals_prefix_array():
    """SPEC.md L256-264 / L276: the roll_window chain equals substring hashes (exact)."""
    B = O.hash_base(3)
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = int(rng.integers(130, 600))
        w = int(rng.choice([1, 2, 7, 128]))
        toks = rng.integers(0, 50 if trial % 2 else 128256, n)
        Bw1 = pow(B, w - 1, P)
        cur = O.poly_hash(toks[:w], B)
        for k in range(1, n - w + 1):
            cur = ((cur - (int(toks[k - 1]) + 1) * Bw1) * B + int(toks[k + w - 1]) + 1) % P
            if k % 17 == 0 or k == n - w:
                assert cur == O.poly_hash(toks[k:k + w], B)
    # constant sequence -> rolling hash unchanged
    c = np.full(300, 9, np.int32)
    assert O.poly_hash(c[:128], B) == O.poly_hash(c[50:178], B)


def test_sha256_golden_and_hashlib():
    for lhs, rhs in _golden_lines("sha256_vectors.txt"):
        if lhs.startswith("bytes:"):
            assert O.sha256_bytes(lhs[6:].encode()).hex() == rhs
        else:
            toks = [int(x) for x in lhs[7:].split(",")]
            assert O.sha256_tokens(toks).hex() == rhs
    rng = np.random.default_rng(4)
    for n in list(range(0, 140)) + [1000, 4096]:
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert O.sha256_bytes(b) == hashlib.sha256(b).digest()
    for m in [0, 1, 7, 8, 9, 63, 64, 65, 128, 1000]:
        toks = rng.integers(0, 128256, m)
        enc = b"".join(struct.pack(">q", int(t)) for t in toks)       # S:L233 big-endian u64
        assert O.sha256_tokens(toks) == hashlib.sha256(enc).digest()


def test_digest_distinguishes_one_token():
    t = np.arange(200, dtype=np.int32)
    u = t.copy(); u[137] += 1
    assert O.sha256_tokens(t) != O.sha256_tokens(u)
    assert O.sha256_tokens(t) == O.sha256_tokens(t.copy())
