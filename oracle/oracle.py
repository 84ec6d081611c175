"""ctypes front-end of the plain CPU oracle (oracle/cp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2605_23640_b200) never imports this module, and this module never
imports the product package.  Every function here marshals arguments only; the
arithmetic lives in cp_oracle.c (see its header for the paper citations).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cp_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

STORED, SUPERSEDED, DUPLICATE, DROPPED_CONTAINED, DEFERRED_PINNED = 0, 1, 2, 3, 4
OK, ERR_INVALID_ARG, ERR_SENSITIVE_SPAN, ERR_SPAN_TOO_SHORT, ERR_CAPACITY = 0, -1, -2, -3, -4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u64, i64, i32, vp = C.c_uint64, C.c_int64, C.c_int32, C.c_void_p
        sig = {
            "orc_splitmix64": (u64, [u64]),
            "orc_hash_base": (u64, [u64]),
            "orc_mulmod": (u64, [u64, u64]),
            "orc_poly_hash": (u64, [vp, i64, u64]),
            "orc_prefix_hashes": (None, [vp, i64, u64, vp]),
            "orc_sha256_bytes": (None, [vp, u64, vp]),
            "orc_sha256_tokens": (None, [vp, i64, vp]),
            "orc_index_new": (vp, [i32, u64, i64, i32, i32]),
            "orc_index_free": (None, [vp]),
            "orc_index_base": (u64, [vp]),
            "orc_index_insert": (i32, [vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, u64, vp, vp]),
            "orc_match": (i32, [vp, vp, vp, vp, vp, i32, u64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "orc_index_insert_session": (i32, [vp, vp, vp, i32, vp, u64, vp, vp]),
            "orc_num_ids": (i32, [vp]),
            "orc_live_tokens": (i64, [vp]),
            "orc_fifo_count": (i32, [vp]),
            "orc_entry_get": (i32, [vp, i32, vp, vp, vp, vp, vp, vp]),
            "orc_fifo_get": (None, [vp, vp]),
            "orc_rerotate_row": (None, [vp, i32, i32, i32, C.c_double, i64, i32, vp]),
            "orc_score": (i32, [vp, i64, i32, i32, i32, i32, i32, vp, vp]),
            "orc_kv_deviation": (i32, [vp, vp, vp, vp, i64, i32, i32, i32, vp, vp]),
            "orc_link_blocks": (i32, [vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, i32, vp]),
            "orc_pin_pages": (i32, [vp, vp, i64, i32]),
            "orc_entry_pin": (i32, [vp, i32]),
            "orc_rerotate_rows": (None, [vp, i64, i32, i32, i32, C.c_double, i64, i32, vp]),
            "orc_annotate": (i32, [vp, i64, i32, vp, i32, i32, vp, vp, vp]),
            "orc_sat": (None, [vp, i64, i32, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# --- hashing -------------------------------------------------------------------
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def hash_base(seed: int) -> int:
    return int(lib().orc_hash_base(seed))


def mulmod(a: int, b: int) -> int:
    return int(lib().orc_mulmod(a, b))


def poly_hash(tokens, B: int) -> int:
    t = _c(tokens, np.int32)
    return int(lib().orc_poly_hash(_p(t), len(t), B))


def prefix_hashes(tokens, B: int) -> np.ndarray:
    t = _c(tokens, np.int32)
    h = np.zeros(len(t) + 1, np.uint64)
    lib().orc_prefix_hashes(_p(t), len(t), B, _p(h))
    return h


def sha256_bytes(b: bytes) -> bytes:
    buf = np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8)
    out = np.zeros(32, np.uint8)
    lib().orc_sha256_bytes(_p(buf), len(b), _p(out))
    return out.tobytes()


def sha256_tokens(tokens) -> bytes:
    t = _c(tokens, np.int32)
    if len(t) == 0:
        t = np.zeros(1, np.int32)
        out = np.zeros(32, np.uint8)
        lib().orc_sha256_tokens(_p(t), 0, _p(out))
        return out.tobytes()
    out = np.zeros(32, np.uint8)
    lib().orc_sha256_tokens(_p(t), len(t), _p(out))
    return out.tobytes()


# --- re-rotation / score -------------------------------------------------------------
def rerotate_row(row, H: int, d: int, theta: float, delta: int, bf16: bool, gptj: bool = False) -> np.ndarray:
    x = _c(row, np.float32)
    out = np.zeros_like(x)
    lib().orc_rerotate_row(_p(x), H, d, int(gptj), float(theta), int(delta), int(bf16), _p(out))
    return out


def rerotate_rows(rows, H, d, theta, delta, bf16, gptj=False) -> np.ndarray:
    rows = _c(rows, np.float32)
    out = np.empty_like(rows)
    n = rows.size // (H * d)
    lib().orc_rerotate_rows(_p(rows), n, H, d, int(gptj), float(theta), int(delta), int(bf16), _p(out))
    return out


def score(A, l: int, r: int, rho_num: int = 1, rho_den: int = 4):
    """A: fp32 [n, n] or [heads, n, n]. Returns (scores int64 [m], bits uint32 [ceil(m/32)])."""
    A = _c(A, np.float32)
    if A.ndim == 2:
        A = A[None]
    heads, n = A.shape[0], A.shape[1]
    m = r - l + 1
    sc = np.zeros(max(m, 1), np.int64)
    bits = np.zeros(max((m + 31) // 32, 1), np.uint32)
    rc = lib().orc_score(_p(A), n, heads, l, r, rho_num, rho_den, _p(sc), _p(bits))
    if rc != OK:
        raise ValueError(f"orc_score rc={rc}")
    return sc[:m], bits[:(m + 31) // 32]


def kv_deviation(Kr, Vr, Kf, Vf, rho_num: int = 3, rho_den: int = 20):
    """NEXT-4 (CacheBlend selector; R#30): rows [m, width] (any float dtype that widens to fp32
    exactly).  Returns (dev int64 [m], bits uint32 [ceil(m/32)])."""
    Kr, Vr, Kf, Vf = (_c(np.asarray(x, np.float32).reshape(np.shape(x)[0], -1), np.float32) for x in (Kr, Vr, Kf, Vf))
    m, width = Kr.shape
    dev = np.zeros(max(m, 1), np.int64)
    bits = np.zeros(max((m + 31) // 32, 1), np.uint32)
    rc = lib().orc_kv_deviation(_p(Kr), _p(Vr), _p(Kf), _p(Vf), m, width, rho_num, rho_den, _p(dev), _p(bits))
    if rc != OK:
        raise ValueError(f"orc_kv_deviation rc={rc}")
    return dev[:m], bits[:(m + 31) // 32]


def sat(A) -> np.ndarray:
    """C1 Step 1 on the 2^-40 fixed-point matrix: int64 [(n+1), (n+1)] with zero border."""
    A = _c(A, np.float32)
    if A.ndim == 2:
        A = A[None]
    n = A.shape[1]
    T = np.zeros((n + 1, n + 1), np.int64)
    lib().orc_sat(_p(A), n, A.shape[0], _p(T))
    return T


def annotate(A, mask, min_len: int = 128, max_segments: int = 4096):
    """C1 Steps 1-2: list of (l, r, diff) per coarse segment (l = r = -1 if none)."""
    A = _c(A, np.float32)
    if A.ndim == 2:
        A = A[None]
    n = A.shape[1]
    m = _c(mask, np.uint8)
    ol = np.zeros(max_segments, np.int32); orr = np.zeros(max_segments, np.int32); od = np.zeros(max_segments, np.int64)
    k = lib().orc_annotate(_p(A), n, A.shape[0], _p(m), min_len, max_segments, _p(ol), _p(orr), _p(od))
    if k < 0:
        raise ValueError("too many coarse segments")
    return [(int(ol[i]), int(orr[i]), int(od[i])) for i in range(k)]


def bits_to_bool(bits: np.ndarray, m: int) -> np.ndarray:
    b = np.asarray(bits, np.uint32)
    return ((b[np.arange(m) // 32] >> (np.arange(m) % 32).astype(np.uint32)) & 1).astype(bool)


def pack_bits(flags_per_span):
    """list of bool arrays -> (uint32 words, int64 word offsets [S+1])"""
    words, offs = [], [0]
    for f in flags_per_span:
        f = np.asarray(f, bool)
        nw = (len(f) + 31) // 32
        w = np.zeros(nw, np.uint32)
        idx = np.nonzero(f)[0]
        np.bitwise_or.at(w, idx // 32, (np.uint32(1) << (idx % 32).astype(np.uint32)))
        words.append(w)
        offs.append(offs[-1] + nw)
    return (np.concatenate(words) if words else np.zeros(0, np.uint32)), np.array(offs, np.int64)


# --- NEXT-3 baseline stores (R#28-29) ------------------------
def policy_spans(batch, policy: str, chunk_len: int, max_len: int):
    """Spans a baseline policy stores for a writer batch, in (request, position) order.
    fixed_chunk: every chunk [c*L, (c+1)*L) of the request with no mask-1 token (Fig. 4-b).
    prefix_only: [0, min(first mask-1 position, n, max_len)) if at least L long (Fig. 4-a)."""
    req, beg, ln = [], [], []
    for r in range(batch.num_reqs):
        a, b = int(batch.offsets[r]), int(batch.offsets[r + 1])
        m = [int(x) for x in batch.mask[a:b]]
        n = b - a
        if policy == "fixed_chunk":
            for c in range(n // chunk_len):
                if not any(m[c * chunk_len:(c + 1) * chunk_len]):
                    req.append(r); beg.append(c * chunk_len); ln.append(chunk_len)
        elif policy == "prefix_only":
            first = m.index(1) if 1 in m else n
            p = min(first, n, max_len)
            if p >= chunk_len:
                req.append(r); beg.append(0); ln.append(p)
        else:
            raise ValueError(policy)
    return np.array(req, np.int32), np.array(beg, np.int32), np.array(ln, np.int32)


# --- index ---------------------------------------------------------------------------
@dataclass
class MatchResult:
    num_hits: int
    req_hit_offsets: np.ndarray
    hit_req: np.ndarray
    hit_entry: np.ndarray
    hit_dst: np.ndarray
    hit_len: np.ndarray
    hit_delta: np.ndarray
    plan: np.ndarray
    req_covered: np.ndarray
    req_recompute: np.ndarray
    req_candidates: np.ndarray


class OracleIndex:
    def __init__(self, window_len: int, hash_seed: int, capacity_tokens: int, num_pages: int,
                 block_size: int = 16):
        self.w, self.block = window_len, block_size
        self.h = lib().orc_index_new(window_len, hash_seed, capacity_tokens, block_size, num_pages)
        self.B = int(lib().orc_index_base(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_index_free(self.h)
            self.h = None

    def insert(self, batch, bits_words=None, bits_offsets=None, t: int = 0, spans=None):
        sr, sb, sl = spans if spans is not None else (batch.span_req, batch.span_begin, batch.span_len)
        sr, sb, sl = _c(sr, np.int32), _c(sb, np.int32), _c(sl, np.int32)
        S = len(sr)
        tok, off, msk = _c(batch.tokens, np.int32), _c(batch.offsets, np.int64), _c(batch.mask, np.uint8)
        bw = None if bits_words is None else _c(bits_words, np.uint32)
        bo = None if bits_offsets is None else _c(bits_offsets, np.int64)
        out_id = np.full(max(S, 1), -1, np.int32)
        out_oc = np.full(max(S, 1), -1, np.int32)
        rc = lib().orc_index_insert(self.h, _p(tok), _p(off), _p(msk), batch.num_reqs, S,
                                    _p(sr), _p(sb), _p(sl), _p(bw), _p(bo), t, _p(out_id), _p(out_oc))
        return rc, out_id[:S], out_oc[:S]

    def insert_session(self, batch, sessions, t: int = 0):
        """R#33: each request replaces its session's private entry (whole request, sensitive tokens too)."""
        tok, off = _c(batch.tokens, np.int32), _c(batch.offsets, np.int64)
        ss = _c(np.asarray(sessions), np.int32)
        R = batch.num_reqs
        out_id = np.full(max(R, 1), -1, np.int32)
        out_oc = np.full(max(R, 1), -1, np.int32)
        rc = lib().orc_index_insert_session(self.h, _p(tok), _p(off), R, _p(ss), t, _p(out_id), _p(out_oc))
        return rc, out_id[:R], out_oc[:R]

    def match(self, batch, t: int = 0, no_touch: bool = False, use_mask: bool = True,
              max_hits: Optional[int] = None, policy: Optional[str] = None, sessions=None) -> MatchResult:
        """policy None: CrossUserSelective (the method); "fixed_chunk" / "prefix_only": NEXT-3
        baselines (R#28-29)."""
        R, T = batch.num_reqs, batch.total_tokens
        tok, off = _c(batch.tokens, np.int32), _c(batch.offsets, np.int64)
        msk = _c(batch.mask, np.uint8) if use_mask else None
        mh = max_hits if max_hits is not None else T // self.w + R + 1
        o = lambda n, dt=np.int32: np.zeros(max(n, 1), dt)
        rho = o(R + 1)
        hr, he, hd, hl, hdl = o(mh), o(mh), o(mh), o(mh), o(mh)
        plan = o(T, np.uint8)
        cov, rec, cand = o(R), o(R), o(R)
        flags = int(no_touch) | {None: 0, "fixed_chunk": 2, "prefix_only": 4}[policy]
        ss = None if sessions is None else _c(np.asarray(sessions), np.int32)
        nh = lib().orc_match(self.h, _p(tok), _p(off), _p(msk), _p(ss), R, t, flags, mh, _p(rho),
                             _p(hr), _p(he), _p(hd), _p(hl), _p(hdl), _p(plan), _p(cov), _p(rec), _p(cand))
        if nh < 0:
            raise RuntimeError("oracle match: hit buffer overflow")
        return MatchResult(nh, rho[:R + 1], hr[:nh], he[:nh], hd[:nh], hl[:nh], hdl[:nh], plan[:T],
                           cov[:R], rec[:R], cand[:R])

    def link_blocks(self, batch, res: "MatchResult", max_blocks: Optional[int] = None) -> np.ndarray:
        """NEXT-2 (R#31): int32 [R, max_blocks] pool page linked to each request block, -1 if none."""
        R = batch.num_reqs
        off = _c(batch.offsets, np.int64)
        mb = max_blocks if max_blocks is not None else int(max((off[r + 1] - off[r] + 15) // 16 for r in range(R)))
        link = np.full((R, max(mb, 1)), -1, np.int32)
        rc = lib().orc_link_blocks(self.h, R, _p(off), res.num_hits, _p(_c(res.hit_req, np.int32)),
                                   _p(_c(res.hit_entry, np.int32)), _p(_c(res.hit_dst, np.int32)),
                                   _p(_c(res.hit_len, np.int32)), _p(_c(res.hit_delta, np.int32)),
                                   _p(_c(res.plan, np.uint8)), max(mb, 1), _p(link))
        if rc != OK:
            raise ValueError(f"orc_link_blocks rc={rc}")
        return link[:, :mb]

    def pin_pages(self, pages, delta: int) -> int:
        """R#32: pin (+1) / unpin (-1) the entries owning the listed pool pages (a link table; -1 skipped)."""
        p = _c(np.asarray(pages).reshape(-1), np.int32)
        return int(lib().orc_pin_pages(self.h, _p(p), len(p), int(delta)))

    def entry_pin(self, eid: int) -> int:
        return int(lib().orc_entry_pin(self.h, int(eid)))

    @property
    def num_ids(self) -> int:
        return int(lib().orc_num_ids(self.h))

    @property
    def live_tokens(self) -> int:
        return int(lib().orc_live_tokens(self.h))

    def fifo(self) -> np.ndarray:
        n = int(lib().orc_fifo_count(self.h))
        out = np.zeros(max(n, 1), np.int32)
        lib().orc_fifo_get(self.h, _p(out))
        return out[:n]

    def entry(self, eid: int) -> dict:
        info = np.zeros(10, np.int32)
        hs = np.zeros(3, np.uint64)
        lib().orc_entry_get(self.h, eid, _p(info), _p(hs), None, None, None, None)
        ln, npg = int(info[1]), int(info[5])
        dg = np.zeros(32, np.uint8)
        pages = np.zeros(max(npg, 1), np.int32)
        toks = np.zeros(max(ln, 1), np.int32)
        rec = np.zeros(max(ln, 1), np.uint8)
        lib().orc_entry_get(self.h, eid, _p(info), _p(hs), _p(dg), _p(pages), _p(toks), _p(rec))
        return dict(id=eid, live=bool(info[0]), len=ln, origin_pos=int(info[2]), origin_call=int(info[3]),
                    origin_req=int(info[4]), prefix_hash=int(hs[0]), full_hash=int(hs[1]),
                    last_used=int(hs[2]), digest=dg.tobytes(), pages=pages[:npg].copy(),
                    tokens=toks[:ln].copy(), recompute=rec[:ln].astype(bool), pin=int(info[6]), owner=int(info[7]))

    def live_entries(self):
        return [e for e in (self.entry(i) for i in range(self.num_ids)) if e["live"]]
