"""Synthetic workloads shaped like CachePrune's evaluation (§5).

Everything here is a seeded generator:
  * token ids / sensitivity masks / insert spans for the five BASELINE configs,
  * a counter-based KV payload (splitmix64 of a packed coordinate key) that the
    numpy side and the torch-on-device side reproduce bit-for-bit,
  * causal row-stochastic exp-decay attention matrices for the recompute score.

Workload shapes (citations are PAPER.md line numbers):
  * user text is 8.8% of a prompt and 2.3% of user text is sensitive (L350, L356);
  * the writer ("constructed request") populates the pool and the reader
    ("original request") is matched against it (L1248-1250), with the
    sensitive tokens replaced by substitutes -- here of a different length,
    which shifts every later segment and forces RoPE re-rotation;
  * strict masking (Policy 3, L757-760) marks all user text sensitive so only
    system prompts / retrieved passages are shared (configs 3-5);
  * insert spans are whole coarse segments (maximal mask-0 runs, L556-558) of
    length >= window_len (min segment length 128, L646-648).  The generator
    knows where it put every sensitive run, so it emits the spans from its own
    layout; it never runs the method's segmentation.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Geometry", "Batch", "Workload", "CONFIGS", "make_workload",
    "splitmix64_np", "payload_np", "bf16_round_np", "bf16_bits_np",
    "payload_torch", "fill_paged_kv_torch", "attention_np", "attention_torch",
    "VOCAB", "pack_batches",
]

VOCAB = 128256          # Llama-3 vocabulary size (SURVEY §8(d) input recipe)
FILLER_LO = 1000        # filler ids are uniform in [FILLER_LO, VOCAB)
M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
PAYLOAD_SALT = 0x243F6A8885A308D3   # fixed salt of the KV payload generator


# ----------------------------------------------------------------------------
# geometry / batches
# ----------------------------------------------------------------------------
@dataclass
class Geometry:
    num_layers: int
    num_kv_heads: int
    head_dim: int
    dtype: str                 # "fp32" | "bf16"
    rope_theta: float
    window_len: int = 128
    block_size: int = 16
    rope_style: str = "neox"   # "neox" (pairs i, i+d/2) | "gptj" (pairs 2i, 2i+1)

    @property
    def elem_bytes(self) -> int:
        return 4 if self.dtype == "fp32" else 2

    @property
    def row_bytes(self) -> int:
        """bytes of one token's K (or V) row for one layer: H*d*e"""
        return self.num_kv_heads * self.head_dim * self.elem_bytes

    def shard(self, layer_lo: int, layer_hi: int, head_lo: int, head_hi: int) -> "Geometry":
        return dataclasses.replace(self, num_layers=layer_hi - layer_lo,
                                   num_kv_heads=head_hi - head_lo)


@dataclass
class Batch:
    """A CSR batch of requests plus (for writers) the spans to insert."""
    tokens: np.ndarray          # int32 [T]
    offsets: np.ndarray         # int64 [R+1]
    mask: np.ndarray            # uint8 [T], 1 = sensitive
    writer_ids: np.ndarray      # int64 [R], payload identity of each request
    span_req: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    span_begin: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    span_len: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    # layout annotations (used only by generators/tests, never by the method)
    segments: List[List[Tuple[int, int]]] = field(default_factory=list)

    @property
    def num_reqs(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def total_tokens(self) -> int:
        return int(self.offsets[-1])

    @property
    def lens(self) -> np.ndarray:
        return np.diff(self.offsets)

    def req_tokens(self, r: int) -> np.ndarray:
        return self.tokens[self.offsets[r]:self.offsets[r + 1]]

    def req_mask(self, r: int) -> np.ndarray:
        return self.mask[self.offsets[r]:self.offsets[r + 1]]

    def subset(self, reqs: Sequence[int]) -> "Batch":
        reqs = list(reqs)
        return pack_batches([_single(self, r) for r in reqs])


def _single(b: Batch, r: int) -> Batch:
    sel = b.span_req == r
    return Batch(tokens=b.req_tokens(r).copy(),
                 offsets=np.array([0, b.lens[r]], np.int64),
                 mask=b.req_mask(r).copy(),
                 writer_ids=b.writer_ids[r:r + 1].copy(),
                 span_req=np.zeros(int(sel.sum()), np.int32),
                 span_begin=b.span_begin[sel].copy(),
                 span_len=b.span_len[sel].copy(),
                 segments=[b.segments[r]] if b.segments else [])


def pack_batches(parts: Sequence[Batch]) -> Batch:
    toks, masks, wids, sr, sb, sl, segs = [], [], [], [], [], [], []
    offs = [0]
    r0 = 0
    for p in parts:
        toks.append(p.tokens); masks.append(p.mask); wids.append(p.writer_ids)
        for r in range(p.num_reqs):
            offs.append(offs[-1] + int(p.lens[r]))
        sr.append(p.span_req + r0); sb.append(p.span_begin); sl.append(p.span_len)
        segs.extend(p.segments)
        r0 += p.num_reqs
    cat = lambda xs, dt: (np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    return Batch(tokens=cat(toks, np.int32), offsets=np.array(offs, np.int64),
                 mask=cat(masks, np.uint8), writer_ids=cat(wids, np.int64),
                 span_req=cat(sr, np.int32), span_begin=cat(sb, np.int32),
                 span_len=cat(sl, np.int32), segments=segs)


def _build_request(parts: Sequence[Tuple[np.ndarray, int]]):
    """parts: list of (tokens, sensitive_flag). Returns tokens, mask, clear runs."""
    toks = np.concatenate([p[0] for p in parts]).astype(np.int32)
    mask = np.concatenate([np.full(len(p[0]), p[1], np.uint8) for p in parts])
    runs = []
    pos = 0
    cur = None
    for t, s in parts:
        n = len(t)
        if n == 0:
            continue
        if s == 0:
            cur = (cur[0], pos + n) if cur is not None else (pos, pos + n)
        else:
            if cur is not None:
                runs.append(cur)
            cur = None
        pos += n
    if cur is not None:
        runs.append(cur)
    return toks, mask, runs


def _make_batch(reqs, writer_ids, w: int) -> Batch:
    """reqs: list of (tokens, mask, clear_runs). Spans = clear runs of length >= w."""
    offs = [0]
    sr, sb, sl, segs = [], [], [], []
    for r, (t, m, runs) in enumerate(reqs):
        offs.append(offs[-1] + len(t))
        segs.append(runs)
        for a, b in runs:
            if b - a >= w:
                sr.append(r); sb.append(a); sl.append(b - a)
    return Batch(tokens=np.concatenate([q[0] for q in reqs]).astype(np.int32) if reqs else np.zeros(0, np.int32),
                 offsets=np.array(offs, np.int64),
                 mask=np.concatenate([q[1] for q in reqs]).astype(np.uint8) if reqs else np.zeros(0, np.uint8),
                 writer_ids=np.asarray(writer_ids, np.int64),
                 span_req=np.array(sr, np.int32), span_begin=np.array(sb, np.int32),
                 span_len=np.array(sl, np.int32), segments=segs)


def _fill(rng: np.random.Generator, n: int) -> np.ndarray:
    return rng.integers(FILLER_LO, VOCAB, size=n, dtype=np.int64).astype(np.int32)


def _passage(seed: int, pid: int, lo: int, hi: int) -> np.ndarray:
    r = np.random.default_rng([seed, 7919, pid])
    n = int(r.integers(lo, hi + 1))
    return _fill(r, n)


_ZIPF_CDF = {}


def _zipf(rng: np.random.Generator, n_items: int, s: float, size: int) -> np.ndarray:
    key = (n_items, s)
    if key not in _ZIPF_CDF:
        p = 1.0 / np.power(np.arange(1, n_items + 1, dtype=np.float64), s)
        _ZIPF_CDF[key] = np.cumsum(p / p.sum())
    cdf = _ZIPF_CDF[key]
    return np.minimum(np.searchsorted(cdf, rng.random(size), side="right"), n_items - 1)


# ----------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    geometry: Geometry
    # sequential rounds: each round = (writer batch to insert, reader batch to match)
    rounds: List[Tuple[Optional[Batch], Batch]]
    pool_capacity_tokens: int
    max_span_len: int
    notes: str = ""


def toy_workload(seed: int = 1, pairs: int = 4) -> Workload:
    """Config 1: L=2, H=2, d=64, fp32, theta=1e4; 8 requests x ~512 tokens.

    Prompt = [system 128 (shared)] [PII1 2-6] [body A 150] [PII2] [body B 150]
    [PII3] [tail < 128].  The reader is the writer with each PII run replaced by
    fresh tokens whose length differs by 0..3, so bodies A and B move (delta != 0)
    while the system prefix is reused in place (delta == 0).
    """
    g = Geometry(2, 2, 64, "fp32", 10000.0)
    rng = np.random.default_rng(seed)
    system = _fill(rng, 128)
    rounds = []
    for p in range(pairs):
        pii = [int(x) for x in rng.integers(2, 7, size=3)]
        a, b = _fill(rng, 150), _fill(rng, 150)
        tail_n = 512 - (128 + 300 + sum(pii))
        tail = _fill(rng, tail_n)
        wpii = [_fill(rng, k) for k in pii]
        rpii = [_fill(rng, max(1, k + int(rng.integers(-3, 4)))) for k in pii]
        wreq = _build_request([(system, 0), (wpii[0], 1), (a, 0), (wpii[1], 1), (b, 0), (wpii[2], 1), (tail, 0)])
        rreq = _build_request([(system, 0), (rpii[0], 1), (a, 0), (rpii[1], 1), (b, 0), (rpii[2], 1), (tail, 0)])
        wb = _make_batch([wreq], [2 * p], g.window_len)
        rb = _make_batch([rreq], [2 * p + 1], g.window_len)
        rounds.append((wb, rb))
    return Workload("toy", g, rounds, pool_capacity_tokens=1 << 20, max_span_len=512,
                    notes="4 writer/reader pairs processed sequentially")


def msmarco_workload(seed: int = 2, pairs: int = 256, geometry: Optional[Geometry] = None) -> Workload:
    """Config 2: Llama-3-8B-shaped KV, MSMARCO-style RAG prompts of ~1.5K tokens.

    Prompt = [system 160 (shared)] [question ~135 tokens = 8.8% of the prompt,
    holding 1-2 PII runs of ~3 tokens = 2.3% of user text] [10 passages of
    100-148 tokens].  Writers are the constructed requests; readers replace each
    PII run with one whose length differs by -2..+2 (>= 1).
    """
    g = geometry or Geometry(32, 8, 128, "bf16", 500000.0)
    rng = np.random.default_rng(seed)
    system = _fill(rng, 160)
    wreqs, rreqs = [], []
    for p in range(pairs):
        n_pii = int(rng.integers(1, 3))
        pii = [int(x) for x in rng.integers(2, 5, size=n_pii)]
        q_total = 135 - sum(pii)
        cuts = np.sort(rng.integers(10, q_total - 10, size=n_pii))
        qparts = np.split(_fill(rng, q_total), cuts)
        passages = [_fill(rng, int(rng.integers(100, 149))) for _ in range(10)]
        body = np.concatenate(passages)
        wp = [_fill(rng, k) for k in pii]
        rp = [_fill(rng, max(1, k + int(rng.integers(-2, 3)))) for k in pii]

        def build(piis):
            parts = [(system, 0)]
            for i in range(n_pii):
                parts.append((qparts[i], 0))
                parts.append((piis[i], 1))
            parts.append((np.concatenate([qparts[n_pii], body]), 0))
            return _build_request(parts)
        wreqs.append(build(wp)); rreqs.append(build(rp))
    wb = _make_batch(wreqs, np.arange(pairs) * 2, g.window_len)
    rb = _make_batch(rreqs, np.arange(pairs) * 2 + 1, g.window_len)
    cap = int(wb.span_len.sum()) + 4096
    return Workload("msmarco_rag", g, [(wb, rb)], pool_capacity_tokens=cap, max_span_len=2048,
                    notes="256 writer/reader pairs; writers inserted before the readers are matched")


def multidoc_workload(seed: int = 3, readers: int = 128, corpus: int = 512, per_reader: int = 7,
                      prompt_len: int = 4096, geometry: Optional[Geometry] = None,
                      passage_lo: int = 256, passage_hi: int = 768, zipf_s: float = 0.8,
                      origin_hi: int = 3584) -> Workload:
    """Config 3 (and, with the 70B geometry, config 4): multi-document RAG.

    Writers follow strict masking (Policy 3): each writer prompt is
    [masked user text of length o ~ U[0, origin_hi]] [one passage] [1 masked token],
    so each stored entry is exactly one passage at origin position o.  A
    system-prompt writer stores the shared 128-token system prompt at 0.
    Readers = [system 128] + `per_reader` passages (Zipf, random order) +
    a masked question filling up to `prompt_len`.
    """
    g = geometry or Geometry(32, 8, 128, "bf16", 500000.0)
    rng = np.random.default_rng(seed)
    system = _fill(rng, 128)
    wreqs = [_build_request([(system, 0), (_fill(rng, 1), 1)])]
    for pid in range(corpus):
        o = int(rng.integers(0, origin_hi + 1))
        wreqs.append(_build_request([(_fill(rng, o), 1), (_passage(seed, pid, passage_lo, passage_hi), 0),
                                     (_fill(rng, 1), 1)]))
    wb = _make_batch(wreqs, np.arange(len(wreqs)), g.window_len)
    rreqs = []
    for r in range(readers):
        pids = _zipf(rng, corpus, zipf_s, per_reader)
        parts = [(system, 0)]
        for pid in pids:
            parts.append((_passage(seed, int(pid), passage_lo, passage_hi), 0))
        used = sum(len(p[0]) for p in parts)
        parts.append((_fill(rng, max(8, prompt_len - used)), 1))
        rreqs.append(_build_request(parts))
    rb = _make_batch(rreqs, 100000 + np.arange(readers), g.window_len)
    cap = int(wb.span_len.sum()) + 4096
    return Workload("multidoc_shifted", g, [(wb, rb)], pool_capacity_tokens=cap,
                    max_span_len=max(passage_hi, 128) + 16,
                    notes="one entry per passage; readers reuse passages at shifted positions")


def churn_workload(seed: int = 5, batches: int = 40, per_batch: int = 256, corpus: int = 100000,
                   geometry: Optional[Geometry] = None, passages_per_req: int = 9,
                   capacity_tokens: int = 6_000_000) -> Workload:
    """Config 5: high-churn serving mix (10K requests in 40 batches of 256).

    Request = [system 128] then ~9 passages of 128-192 tokens from a 100K
    passage Zipf(1.1) corpus, each preceded by a sensitive run of 3-5 tokens
    (~2.3% of tokens).  Every request is first a reader (matched) and then a
    writer (its own segments are inserted), so rounds are (same batch, same batch).
    """
    g = geometry or Geometry(32, 8, 128, "bf16", 500000.0)
    rng = np.random.default_rng(seed)
    system = _fill(rng, 128)
    rounds = []
    wid = 0
    for b in range(batches):
        reqs = []
        for r in range(per_batch):
            pids = _zipf(rng, corpus, 1.1, passages_per_req)
            parts = [(system, 0)]
            for pid in pids:
                parts.append((_fill(rng, int(rng.integers(3, 6))), 1))
                parts.append((_passage(seed, int(pid), 128, 192), 0))
            reqs.append(_build_request(parts))
        bb = _make_batch(reqs, np.arange(wid, wid + per_batch), g.window_len)
        wid += per_batch
        rounds.append((bb, bb))
    return Workload("high_churn", g, rounds, pool_capacity_tokens=capacity_tokens, max_span_len=256,
                    notes="each batch is matched, then inserted (Duplicate/Stored/Supersede + LRU)")


CONFIGS = {
    1: "toy KV (2 layers, 2 KV heads, head_dim 64, fp32): 8 requests x 512 tokens",
    2: "Llama-3-8B-shaped KV, MSMARCO-style RAG prompts ~1.5K tokens, 256 requests, 1 B200",
    3: "Llama-3-8B-shaped KV, multi-document RAG, passages at shifted positions, 4K prompts",
    4: "Llama-3-70B-shaped KV (80 layers), 8K prompts, sharded by layer/head",
    5: "high-churn serving mix: 10K requests, 100K-span index, 2.3% sensitive tokens",
}


def make_workload(cfg: int, scale: float = 1.0, seed: Optional[int] = None, **kw) -> Workload:
    """scale < 1 shrinks request counts (parity tests at oracle-friendly sizes)."""
    s = lambda n: max(1, int(round(n * scale)))
    if cfg == 1:
        return toy_workload(seed if seed is not None else 1, **kw)
    if cfg == 2:
        return msmarco_workload(seed if seed is not None else 2, pairs=s(256), **kw)
    if cfg == 3:
        return multidoc_workload(seed if seed is not None else 3, readers=s(128), corpus=s(512), **kw)
    if cfg == 4:
        g = kw.pop("geometry", None) or Geometry(80, 8, 128, "bf16", 500000.0)
        return multidoc_workload(seed if seed is not None else 4, readers=s(64), corpus=s(1000),
                                 per_reader=14, prompt_len=8192, geometry=g, origin_hi=7168, **kw)
    if cfg == 5:
        return churn_workload(seed if seed is not None else 5, batches=s(40), per_batch=s(256),
                              corpus=max(1000, s(100000)), **kw)
    raise ValueError(cfg)


# ----------------------------------------------------------------------------
# counter-based KV payload (bit-identical in numpy and torch)
# ----------------------------------------------------------------------------
def splitmix64_np(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
        return z ^ (z >> np.uint64(31))


def _payload_key_np(writer, pos, layer, head, dim, kind):
    u = lambda a: np.asarray(a, dtype=np.uint64)
    return ((u(writer) << np.uint64(44)) | (u(pos) << np.uint64(24)) | (u(layer) << np.uint64(16))
            | (u(head) << np.uint64(9)) | (u(kind) << np.uint64(8)) | u(dim))


def payload_np(writer, pos, layer, head, dim, kind) -> np.ndarray:
    """fp32 payload value in [-2, 2), exactly representable in fp32.

    key packs (writer<2^20, pos<2^20, layer<256, head<128, kind in {0=K,1=V}, dim<256);
    value = ((splitmix64(key ^ SALT) >> 40) - 2^23) * 2^-22.
    """
    z = splitmix64_np(_payload_key_np(writer, pos, layer, head, dim, kind) ^ np.uint64(PAYLOAD_SALT))
    u = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return u.astype(np.float32) * np.float32(2.0 ** -22)


def bf16_bits_np(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern with round-to-nearest-even (finite inputs)."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = (b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_round_np(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 (RNE), returned as fp32 values."""
    return (bf16_bits_np(x).astype(np.uint32) << np.uint32(16)).view(np.float32)


def payload_torch(writer, pos, layer, head, dim, kind):
    """Same values as payload_np, computed with torch int64 ops (wrapping)."""
    import torch

    def s64(c):
        return c - (1 << 64) if c >= (1 << 63) else c

    def lsr(z, k):   # logical shift right on int64
        return (z >> k) & ((1 << (64 - k)) - 1)

    key = (writer << 44) | (pos << 24) | (layer << 16) | (head << 9) | (kind << 8) | dim
    z = key ^ s64(PAYLOAD_SALT)
    z = z + s64(_GOLDEN)
    z = (z ^ lsr(z, 30)) * s64(_MIX1)
    z = (z ^ lsr(z, 27)) * s64(_MIX2)
    z = z ^ lsr(z, 31)
    u = lsr(z, 40) - (1 << 23)
    return u.to(torch.float32) * (2.0 ** -22)


def fill_paged_kv_torch(k_layers, v_layers, block_tables, lens, writer_ids, geometry: Geometry,
                        layer_offset: int = 0, head_offset: int = 0, token_chunk: int = 1 << 16,
                        only_ranges=None):
    """Write the payload of every (request, position) into a paged KV cache.

    k_layers/v_layers: lists of torch tensors [num_blocks, block, H, d] (one per layer).
    block_tables: torch int32 [R, max_blocks] on the same device; lens: list of ints.
    only_ranges: optional list (per request) of (begin, end) position ranges to fill.
    """
    import torch
    dev = k_layers[0].device
    H, d, bs = geometry.num_kv_heads, geometry.head_dim, geometry.block_size
    tdt = torch.float32 if geometry.dtype == "fp32" else torch.bfloat16
    bt = block_tables.to(torch.int64)
    hh = (torch.arange(H, device=dev, dtype=torch.int64) + head_offset).view(1, H, 1)
    dd = torch.arange(d, device=dev, dtype=torch.int64).view(1, 1, d)
    for r, n in enumerate(lens):
        ranges = only_ranges[r] if only_ranges is not None else [(0, int(n))]
        for (lo, hi) in ranges:
            for c0 in range(lo, hi, token_chunk):
                c1 = min(hi, c0 + token_chunk)
                pos = torch.arange(c0, c1, device=dev, dtype=torch.int64)
                blk = bt[r, pos // bs]
                slot = pos % bs
                p3 = pos.view(-1, 1, 1)
                for li in range(len(k_layers)):
                    lay = li + layer_offset
                    for kind, dst in ((0, k_layers[li]), (1, v_layers[li])):
                        val = payload_torch(int(writer_ids[r]), p3, lay, hh, dd, kind).to(tdt)
                        dst[blk, slot] = val


# ----------------------------------------------------------------------------
# attention matrices (last-layer, head-aggregated, causal, row-stochastic)
# ----------------------------------------------------------------------------
def _attn_logits_np(n: int, segments, lam: float, seed: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64).reshape(-1, 1)
    j = np.arange(n, dtype=np.float64).reshape(1, -1)
    seg = np.full(n, -1, np.int64)
    for s, (a, b) in enumerate(segments):
        seg[a:b] = s
    same = (seg.reshape(-1, 1) == seg.reshape(1, -1)) & (seg.reshape(-1, 1) >= 0)
    key = (np.uint64(seed) << np.uint64(40)) ^ (np.arange(n * n, dtype=np.uint64).reshape(n, n))
    noise = (splitmix64_np(key) >> np.uint64(40)).astype(np.float64) / float(1 << 24)
    w = np.exp(-lam * (i - j)) * np.where(same, 4.0, 1.0) * (0.5 + noise)
    w[j > i] = 0.0
    return w


def attention_np(n: int, segments=(), lam: float = 0.01, seed: int = 0) -> np.ndarray:
    """fp32 [n, n] causal row-stochastic exp-decay attention with segment locality."""
    w = _attn_logits_np(n, segments, lam, seed)
    return (w / w.sum(axis=1, keepdims=True)).astype(np.float32)


def attention_torch(n: int, segments=(), lam: float = 0.01, seed: int = 0, device="cuda"):
    """Device-side version (values close to, not bit-identical with, attention_np).

    Parity tests copy the device matrix back and hand the same bytes to the oracle.
    """
    import torch
    i = torch.arange(n, device=device, dtype=torch.float32).view(-1, 1)
    j = torch.arange(n, device=device, dtype=torch.float32).view(1, -1)
    seg = torch.full((n,), -1, device=device, dtype=torch.int64)
    for s, (a, b) in enumerate(segments):
        seg[a:b] = s
    same = (seg.view(-1, 1) == seg.view(1, -1)) & (seg.view(-1, 1) >= 0)
    ii = torch.arange(n, device=device, dtype=torch.int64)
    noise = payload_torch(seed & 0xFFFFF, ii.view(-1, 1) & 0xFFFFF, 0, 0, ii.view(1, -1) & 0xFF, 0)
    noise = noise * 0.25 + 1.0
    w = torch.exp(-lam * (i - j)) * torch.where(same, 4.0, 1.0) * noise
    w = torch.tril(w)
    return (w / w.sum(dim=1, keepdim=True)).contiguous()
