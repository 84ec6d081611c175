"""Thin Python front-end over the C-ABI (include/cacheprune.h): argument marshalling only.

Every step of the hot path runs in libcacheprune.so kernels; torch supplies
device memory (workspaces, batches, paged caches) and streams.  Names follow
the C-ABI: insert / match_spans / gather_rerotate / score_deviation.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _i32(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs, dtype=np.int64).astype(np.int32)).reshape(-1)


def _offsets(ms: np.ndarray):
    """Per-span score offsets and packed-bit word offsets: int64 [S + 1] each (prefix sums)."""
    so = np.zeros(len(ms) + 1, np.int64)
    bo = np.zeros(len(ms) + 1, np.int64)
    np.cumsum(ms, out=so[1:])
    np.cumsum((ms.astype(np.int64) + 31) // 32, out=bo[1:])
    return so, bo


def _cptr(a: np.ndarray, ctype):
    """Host array pointer for the C-ABI (the caller keeps `a` alive across the call)."""
    return a.ctypes.data_as(C.POINTER(ctype))


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class IndexConfig:
    num_layers: int
    num_kv_heads: int
    head_dim: int
    dtype: str = "bf16"                  # "bf16" | "fp32"
    rope_theta: float = 500000.0
    rope_style: str = "neox"
    window_len: int = 128
    block_size: int = 16
    hash_seed: int = 42
    pool_capacity_tokens: int = 1 << 20
    max_entries: int = 8192
    max_span_len: int = 2048
    max_req_tokens: int = 10240
    max_batch_reqs: int = 1024
    max_batch_tokens: int = 1 << 21
    max_spans_per_insert: int = 4096
    layer_offset: int = 0
    head_offset: int = 0
    max_sessions: int = 0                 # same-user session store (R#33); 0 = off

    def c(self) -> L.CpConfig:
        return L.CpConfig(self.window_len, self.block_size, self.hash_seed, self.num_layers, self.num_kv_heads,
                          self.head_dim, self.layer_offset, self.head_offset,
                          L.CP_BF16 if self.dtype == "bf16" else L.CP_FP32,
                          L.CP_ROPE_GPTJ if self.rope_style == "gptj" else L.CP_ROPE_NEOX,
                          float(self.rope_theta), self.pool_capacity_tokens, self.max_entries, self.max_span_len,
                          self.max_req_tokens, self.max_batch_reqs, self.max_batch_tokens, self.max_spans_per_insert,
                          self.max_sessions)

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32


@dataclass
class DeviceBatch:
    tokens: torch.Tensor                  # int32 [T]
    offsets: torch.Tensor                 # int64 [R+1]
    mask: Optional[torch.Tensor]          # uint8 [T] or None
    max_req_len: int = 0
    session: Optional[torch.Tensor] = None   # int32 [R]: same-user session per request (R#33), or None

    @property
    def num_reqs(self) -> int:
        return int(self.offsets.numel() - 1)

    @property
    def total_tokens(self) -> int:
        return int(self.tokens.numel())

    def c(self, with_mask: bool = True) -> L.CpBatch:
        return L.CpBatch(self.num_reqs, self.total_tokens, _ptr(self.tokens), _ptr(self.offsets),
                         _ptr(self.mask) if (with_mask and self.mask is not None) else None, int(self.max_req_len),
                         _ptr(self.session))

    @staticmethod
    def from_numpy(tokens, offsets, mask, device="cuda", pin: bool = False, session=None) -> "DeviceBatch":
        import numpy as np
        lens = np.diff(offsets)
        t = torch.from_numpy(np.ascontiguousarray(tokens, dtype=np.int32))
        o = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64))
        m = None if mask is None else torch.from_numpy(np.ascontiguousarray(mask, dtype=np.uint8))
        ss = None if session is None else torch.from_numpy(np.ascontiguousarray(session, dtype=np.int32)).to(device)
        return DeviceBatch(t.to(device), o.to(device), None if m is None else m.to(device),
                           int(lens.max()) if len(lens) else 0, ss)


@dataclass
class PagedKV:
    k: List[torch.Tensor]                 # per layer [num_blocks, 16, H, d]
    v: List[torch.Tensor]
    block_tables: torch.Tensor            # int32 [R, max_blocks]
    _keep: list = field(default_factory=list)

    def c(self) -> L.CpPagedKV:
        kp = (C.c_void_p * len(self.k))(*[t.data_ptr() for t in self.k])
        vpp = (C.c_void_p * len(self.v))(*[t.data_ptr() for t in self.v])
        self._keep = [kp, vpp]
        return L.CpPagedKV(C.cast(kp, C.POINTER(C.c_void_p)), C.cast(vpp, C.POINTER(C.c_void_p)),
                           _ptr(self.block_tables), int(self.block_tables.shape[1]))

    @staticmethod
    def allocate(num_layers, num_blocks, H, d, dtype, block_tables, device="cuda", zero=True) -> "PagedKV":
        mk = torch.zeros if zero else torch.empty
        k = [mk((num_blocks, 16, H, d), dtype=dtype, device=device) for _ in range(num_layers)]
        v = [mk((num_blocks, 16, H, d), dtype=dtype, device=device) for _ in range(num_layers)]
        return PagedKV(k, v, block_tables.to(device=device, dtype=torch.int32).contiguous())


class Hits:
    """Device output buffers of cp_match_spans."""

    def __init__(self, max_hits: int, num_reqs: int, total_tokens: int, device="cuda"):
        z = lambda n, dt=torch.int32: torch.zeros(max(int(n), 1), dtype=dt, device=device)
        self.max_hits = int(max_hits)
        self.num_hits = z(1)
        self.req_hit_offsets = z(num_reqs + 1)
        self.hit_req, self.hit_entry, self.hit_slot = z(max_hits), z(max_hits), z(max_hits)
        self.hit_dst, self.hit_len, self.hit_delta = z(max_hits), z(max_hits), z(max_hits)
        self.plan = z(total_tokens, torch.uint8)
        self.req_covered, self.req_recompute, self.req_candidates = z(num_reqs), z(num_reqs), z(num_reqs)

    def c(self) -> L.CpHits:
        return L.CpHits(self.max_hits, *[_ptr(t) for t in (
            self.num_hits, self.req_hit_offsets, self.hit_req, self.hit_entry, self.hit_slot, self.hit_dst,
            self.hit_len, self.hit_delta, self.plan, self.req_covered, self.req_recompute, self.req_candidates)])

    def to_host(self) -> dict:
        n = int(self.num_hits.item())
        out = {k: getattr(self, k)[:n].cpu().numpy() for k in
               ("hit_req", "hit_entry", "hit_slot", "hit_dst", "hit_len", "hit_delta")}
        out["num_hits"] = n
        for k in ("req_hit_offsets", "plan", "req_covered", "req_recompute", "req_candidates"):
            out[k] = getattr(self, k).cpu().numpy()
        return out


class KVIndex:
    """A shared KV pool + its prefix index on one GPU (one shard of layers/heads)."""

    def __init__(self, cfg: IndexConfig, device="cuda", stream=None):
        self.cfg, self.device = cfg, torch.device(device)
        self._c = cfg.c()
        lib = L.lib()
        sizes = (C.c_size_t * L.CP_WS_COUNT)()
        L.check(lib.cp_index_workspace(C.byref(self._c), sizes), "cp_index_workspace")
        self.ws_sizes = [int(s) for s in sizes]
        # 256-B aligned byte workspaces (torch's caching allocator returns >= 512-B aligned blocks)
        self.ws = [torch.empty(max(s, 256), dtype=torch.uint8, device=self.device) for s in self.ws_sizes]
        ptrs = (C.c_void_p * L.CP_WS_COUNT)(*[t.data_ptr() for t in self.ws])
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(lib.cp_index_create(C.byref(self._c), ptrs, _stream(stream), C.byref(h)), "cp_index_create")
        self.h = h
        self.num_pages = int(lib.cp_pool_num_pages(C.byref(self._c)))
        self.max_pages_per_entry = int(lib.cp_max_pages_per_entry(C.byref(self._c)))
        self.B = int(lib.cp_index_hash_base(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.lib().cp_index_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def view(self, num_layers: int, num_kv_heads: int, layer_offset: int, head_offset: int,
             stream=None) -> "KVIndexView":
        """cp_index_create_view: a further (layer, head) rectangle of this rank served by this index's
        metadata (one match, one insert) with its own pool."""
        return KVIndexView(self, num_layers, num_kv_heads, layer_offset, head_offset)

    # --- pool views (for tests / diagnostics) ---
    def pool_views(self):
        c = self.cfg
        shape = (c.num_layers, self.num_pages, 16, c.num_kv_heads, c.head_dim)
        n = 1
        for s in shape:
            n *= s
        k = self.ws[0][: n * (4 if c.dtype == "fp32" else 2)].view(c.torch_dtype).view(shape)
        v = self.ws[1][: n * (4 if c.dtype == "fp32" else 2)].view(c.torch_dtype).view(shape)
        return k, v

    def insert(self, writers: DeviceBatch, writer_kv: PagedKV, span_req, span_begin, span_len,
               recompute_bits=None, bits_word_offsets=None, t: int = 0, stream=None, phase: Optional[str] = None,
               out=None):
        """cp_index_insert; phase "prepare" / "commit" calls the split halves (cp_index_insert_prepare /
        _commit, same arguments, stream-ordered by the caller).  out: (out_id, out_oc) int32 buffers."""
        S = int(span_req.numel())
        if out is None:
            out = (torch.full((max(S, 1),), -1, dtype=torch.int32, device=self.device),
                   torch.full((max(S, 1),), -1, dtype=torch.int32, device=self.device))
        out_id, out_oc = out
        fn = {None: "cp_index_insert", "prepare": "cp_index_insert_prepare", "commit": "cp_index_insert_commit"}[phase]
        wb, kv = writers.c(), writer_kv.c()
        rc = getattr(L.lib(), fn)(self.h, C.byref(wb), C.byref(kv), S, _ptr(span_req), _ptr(span_begin),
                                  _ptr(span_len), _ptr(recompute_bits), _ptr(bits_word_offsets), int(t),
                                  _ptr(out_id), _ptr(out_oc), _stream(stream))
        L.check(rc, fn)
        return out_id[:S], out_oc[:S]

    def insert_commit_rects(self, views: Sequence["KVIndexView"], writers: DeviceBatch, writer_kvs: Sequence[PagedKV],
                            span_req, span_begin, span_len, recompute_bits=None, bits_word_offsets=None, t: int = 0,
                            stream=None, out=None):
        """cp_index_insert_commit_rects: the commit half of a split insert whose copy-in fills this index's
        pool (writer_kvs[0]) and its views' (writer_kvs[1:], one per view, one block table) in one launch."""
        S = int(span_req.numel())
        if out is None:
            out = (torch.full((max(S, 1),), -1, dtype=torch.int32, device=self.device),
                   torch.full((max(S, 1),), -1, dtype=torch.int32, device=self.device))
        if len(writer_kvs) != len(views) + 1:
            raise ValueError("one writer cache per rectangle")
        out_id, out_oc = out
        vh = (C.c_void_p * max(1, len(views)))(*[v.h for v in views])
        kvs = (L.CpPagedKV * len(writer_kvs))(*[k.c() for k in writer_kvs])
        wb = writers.c()
        rc = L.lib().cp_index_insert_commit_rects(self.h, len(views), vh, C.byref(wb), kvs, S, _ptr(span_req),
                                                  _ptr(span_begin), _ptr(span_len), _ptr(recompute_bits),
                                                  _ptr(bits_word_offsets), int(t), _ptr(out_id), _ptr(out_oc),
                                                  _stream(stream))
        L.check(rc, "cp_index_insert_commit_rects")
        return out_id[:S], out_oc[:S]

    def insert_session(self, writers: DeviceBatch, writer_kv: PagedKV, t: int = 0, out=None, stream=None):
        """cp_index_insert_session (R#33): each request replaces its session's private entry.  `writers.session`
        (int32 [R], values 1..max_sessions) is required.  Returns (out_id, out_outcome) device tensors."""
        R = writers.num_reqs
        if out is None:
            out = tuple(torch.full((max(R, 1),), -1, dtype=torch.int32, device=self.device) for _ in range(2))
        wb, kv = writers.c(), writer_kv.c()
        L.check(L.lib().cp_index_insert_session(self.h, C.byref(wb), C.byref(kv), int(t), _ptr(out[0]), _ptr(out[1]),
                                                _stream(stream)), "cp_index_insert_session")
        return out[0][:R], out[1][:R]

    def match_spans(self, readers: DeviceBatch, t: int = 0, no_touch: bool = False, use_mask: bool = True,
                    hits: Optional[Hits] = None, stream=None, policy: Optional[str] = None) -> Hits:
        """policy None: the method (cross-user selective); "fixed_chunk" / "prefix_only": the NEXT-3
        baseline policies (CP_MATCH_FIXED_CHUNK / CP_MATCH_PREFIX_ONLY)."""
        flags = (L.CP_MATCH_NO_TOUCH if no_touch else 0) | {
            None: 0, "fixed_chunk": L.CP_MATCH_FIXED_CHUNK, "prefix_only": L.CP_MATCH_PREFIX_ONLY}[policy]
        if hits is None:
            hits = Hits(readers.total_tokens // self.cfg.window_len + readers.num_reqs + 1, readers.num_reqs,
                        readers.total_tokens, self.device)
        rb, hc = readers.c(use_mask), hits.c()
        rc = L.lib().cp_match_spans(self.h, C.byref(rb), int(t), flags, C.byref(hc), _stream(stream))
        L.check(rc, "cp_match_spans")
        return hits

    def gather_rerotate(self, readers: DeviceBatch, hits: Hits, dst_kv: PagedKV,
                        zero_recompute: bool = True, zero_uncovered: bool = False, skip_linked: bool = False,
                        reuse_worklist: bool = False, skip_recompute: bool = False, stream=None):
        """Placeholders (R#14): zero_recompute + zero_uncovered = the paper's zero placeholders for both
        kinds; skip_recompute leaves recompute-marked rows unwritten (plan codes as placeholders)."""
        flags = ((L.CP_ZERO_RECOMPUTE if zero_recompute else 0) | (L.CP_ZERO_UNCOVERED if zero_uncovered else 0) |
                 (L.CP_SKIP_LINKED if skip_linked else 0) | (L.CP_REUSE_WORKLIST if reuse_worklist else 0) |
                 (L.CP_SKIP_RECOMPUTE if skip_recompute else 0))
        rb, hc, kv = readers.c(), hits.c(), dst_kv.c()
        L.check(L.lib().cp_gather_rerotate(self.h, C.byref(rb), C.byref(hc), C.byref(kv), flags, _stream(stream)),
                "cp_gather_rerotate")

    def l2_persist(self, stream=None, hit_ratio: float = 1.0):
        """cp_index_l2_persist: keep this index's metadata L2-resident for kernels launched in `stream`."""
        L.check(L.lib().cp_index_l2_persist(self.h, _stream(stream), float(hit_ratio)), "cp_index_l2_persist")

    def gather_rerotate_rects(self, views: Sequence["KVIndexView"], readers: DeviceBatch, hits: Hits,
                              dst_kvs: Sequence[PagedKV], zero_recompute: bool = True, zero_uncovered: bool = False,
                              skip_linked: bool = False, skip_recompute: bool = False, stream=None):
        """cp_gather_rerotate_rects: this index's rectangle (dst_kvs[0]) and its pool views' (dst_kvs[1:],
        one per view, all on one block table) in one launch."""
        flags = ((L.CP_ZERO_RECOMPUTE if zero_recompute else 0) | (L.CP_ZERO_UNCOVERED if zero_uncovered else 0) |
                 (L.CP_SKIP_LINKED if skip_linked else 0) | (L.CP_SKIP_RECOMPUTE if skip_recompute else 0))
        if len(dst_kvs) != len(views) + 1:
            raise ValueError("one destination cache per rectangle")
        vh = (C.c_void_p * max(1, len(views)))(*[v.h for v in views])
        kvs = (L.CpPagedKV * len(dst_kvs))(*[k.c() for k in dst_kvs])
        rb, hc = readers.c(), hits.c()
        L.check(L.lib().cp_gather_rerotate_rects(self.h, len(views), vh, C.byref(rb), C.byref(hc), kvs, flags,
                                                 _stream(stream)), "cp_gather_rerotate_rects")

    def link_blocks(self, readers: DeviceBatch, hits: Hits, max_blocks: int, out: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
        """NEXT-2 (cp_link_blocks, R#31): int32 [R, max_blocks] pool page per linkable request block, -1
        otherwise.  Valid until the next insert on this index."""
        if out is None:
            out = torch.full((readers.num_reqs, max_blocks), -1, dtype=torch.int32, device=hits.plan.device)
        rb, hc = readers.c(), hits.c()
        L.check(L.lib().cp_link_blocks(self.h, C.byref(rb), C.byref(hc), _ptr(out), int(max_blocks), _stream(stream)),
                "cp_link_blocks")
        return out

    def commit_stats(self, stream=None):
        """(commits applied by the parallel path, by the sequential path, OR of the fallback reasons)
        -- cp_index_commit_stats."""
        out = (C.c_int32 * 3)()
        L.check(L.lib().cp_index_commit_stats(self.h, out, _stream(stream)), "cp_index_commit_stats")
        return int(out[0]), int(out[1]), int(out[2])

    def match_work(self, reset: bool = False, stream=None):
        """cp_index_match_work: (windows, candidates, full-hash-passed, tokens to verify) since the last reset."""
        out = (C.c_uint64 * 4)()
        L.check(L.lib().cp_index_match_work(self.h, out, int(reset), _stream(stream)), "cp_index_match_work")
        return tuple(int(x) for x in out)

    def pin_links(self, pages: torch.Tensor, delta: int, stream=None):
        """cp_pin_links (R#32): +delta pins on the entries owning the listed pool pages (a link table)."""
        p = pages.reshape(-1).contiguous()
        L.check(L.lib().cp_pin_links(self.h, _ptr(p), int(p.numel()), int(delta), _stream(stream)), "cp_pin_links")

    def set_clock(self, clock: Optional[torch.Tensor]):
        """cp_index_set_clock: read the logical time from a device uint64 (int64 storage) tensor, or None."""
        self._clock = clock
        L.check(L.lib().cp_index_set_clock(self.h, _ptr(clock)), "cp_index_set_clock")

    def last_error(self, stream=None) -> int:
        return int(L.lib().cp_index_last_error(self.h, _stream(stream)))

    def snapshot(self, with_tokens: bool = True, stream=None) -> dict:
        import numpy as np
        c = self.cfg
        S, MP, ML = c.max_entries, self.max_pages_per_entry, c.max_span_len
        arr = {
            "id": np.zeros(S, np.int32), "len": np.zeros(S, np.int32), "origin_pos": np.zeros(S, np.int32),
            "prefix_hash": np.zeros(S, np.uint64), "full_hash": np.zeros(S, np.uint64),
            "last_used": np.zeros(S, np.uint64), "digest": np.zeros(S * 32, np.uint8),
            "pages": np.zeros(S * MP, np.int32), "fifo": np.zeros(self.num_pages, np.int32),
            "pin": np.zeros(S, np.int32), "owner": np.zeros(S, np.int32),
        }
        if with_tokens:
            arr["tokens"] = np.zeros(S * ML, np.int32)
            arr["recompute"] = np.zeros(S * ML, np.uint8)
        ptr = lambda k: arr[k].ctypes.data_as(C.c_void_p) if k in arr else None
        snap = L.CpSnapshot(0, 0, 0, 0, 0, ptr("id"), ptr("len"), ptr("origin_pos"), ptr("prefix_hash"),
                            ptr("full_hash"), ptr("last_used"), ptr("digest"), ptr("pages"), ptr("tokens"),
                            ptr("recompute"), ptr("fifo"), ptr("pin"), ptr("owner"))
        L.check(L.lib().cp_index_snapshot(self.h, C.byref(snap), _stream(stream)), "cp_index_snapshot")
        n = snap.num_live
        out = dict(num_live=n, next_id=snap.next_id, live_tokens=snap.live_tokens, fifo_count=snap.fifo_count,
                   error=snap.error, fifo=arr["fifo"][:snap.fifo_count].copy(), entries=[])
        for q in range(n):
            ln = int(arr["len"][q])
            e = dict(id=int(arr["id"][q]), len=ln, origin_pos=int(arr["origin_pos"][q]),
                     prefix_hash=int(arr["prefix_hash"][q]), full_hash=int(arr["full_hash"][q]),
                     last_used=int(arr["last_used"][q]), digest=arr["digest"][32 * q:32 * q + 32].tobytes(),
                     pages=arr["pages"][q * MP:q * MP + (ln + 15) // 16].copy(), pin=int(arr["pin"][q]),
                     owner=int(arr["owner"][q]))
            if with_tokens:
                e["tokens"] = arr["tokens"][q * ML:q * ML + ln].copy()
                e["recompute"] = arr["recompute"][q * ML:q * ML + ln].astype(bool)
            out["entries"].append(e)
        return out


class KVIndexView(KVIndex):
    """A pool view (cp_index_create_view): own geometry + pool workspaces, the base's metadata."""

    def __init__(self, base: KVIndex, num_layers: int, num_kv_heads: int, layer_offset: int, head_offset: int):
        import dataclasses
        self.base, self.device = base, base.device
        self.cfg = dataclasses.replace(base.cfg, num_layers=num_layers, num_kv_heads=num_kv_heads,
                                       layer_offset=layer_offset, head_offset=head_offset)
        self._c = self.cfg.c()
        lib = L.lib()
        sizes = (C.c_size_t * L.CP_WS_COUNT)()
        L.check(lib.cp_index_workspace(C.byref(self._c), sizes), "cp_index_workspace")
        self.ws_sizes = [int(sizes[0]), int(sizes[1]), 0, 0]
        self.ws = [torch.empty(max(int(sizes[i]), 256), dtype=torch.uint8, device=self.device) for i in range(2)]
        h = C.c_void_p()
        L.check(lib.cp_index_create_view(base.h, num_layers, num_kv_heads, layer_offset, head_offset,
                                         _ptr(self.ws[0]), _ptr(self.ws[1]), C.byref(h)), "cp_index_create_view")
        self.h = h
        self.num_pages, self.max_pages_per_entry, self.B = base.num_pages, base.max_pages_per_entry, base.B

    def copy_in(self, writers: DeviceBatch, writer_kv: PagedKV, reuse_worklist: bool = False, stream=None):
        """cp_index_copy_in: this view's share of the base's last insert copy-in."""
        wb, kv = writers.c(), writer_kv.c()
        flags = L.CP_REUSE_WORKLIST if reuse_worklist else 0
        L.check(L.lib().cp_index_copy_in(self.h, C.byref(wb), C.byref(kv), flags, _stream(stream)),
                "cp_index_copy_in")


def score_deviation(attn: Sequence[torch.Tensor], n: Sequence[int], heads: Sequence[int], span_l: Sequence[int],
                    span_r: Sequence[int], rho_num: int = 1, rho_den: int = 4, out_scores=None, out_bits=None,
                    stream=None, mode: int = L.CP_SCORE_INTER_INTRA):
    """Recompute scores + top-rho bits for spans (cp_score_deviation).  Returns (scores, bits,
    score_offsets, bits_word_offsets); scores int64 concatenated, bits uint32 (as int32 storage)."""
    S = len(span_l)
    l_, r_ = _i32(span_l), _i32(span_r)
    ms = r_ - l_ + 1
    so, bo = _offsets(ms)
    dev = attn[0].device if S else torch.device("cuda")
    if out_scores is None:
        out_scores = torch.zeros(max(int(so[-1]), 1), dtype=torch.int64, device=dev)
    if out_bits is None:
        out_bits = torch.zeros(max(int(bo[-1]), 1), dtype=torch.int32, device=dev)
    A = np.fromiter((a.data_ptr() for a in attn), dtype=np.uint64, count=S) if S else np.zeros(1, np.uint64)
    n_, h_ = _i32(n), _i32(heads)
    rc = L.lib().cp_score_deviation(S, _cptr(A, C.c_void_p), _cptr(n_, C.c_int32), _cptr(h_, C.c_int32),
                                    _cptr(l_, C.c_int32), _cptr(r_, C.c_int32), rho_num, rho_den, mode,
                                    int(ms.max()) if S else 1, _ptr(out_scores), _cptr(so, C.c_int64),
                                    _ptr(out_bits), _cptr(bo, C.c_int64), _stream(stream))
    L.check(rc, "cp_score_deviation")
    return out_scores, out_bits, so.tolist(), bo.tolist()


def score_kv_deviation(span_req: Sequence[int], span_l: Sequence[int], span_r: Sequence[int],
                       reused_k: torch.Tensor, reused_v: torch.Tensor, reused_block_tables: torch.Tensor,
                       fresh_k: torch.Tensor, fresh_v: torch.Tensor, fresh_block_tables: torch.Tensor,
                       rho_num: int = 3, rho_den: int = 20, out_scores=None, out_bits=None, stream=None):
    """NEXT-4, CacheBlend's selector (cp_score_kv_deviation; R#30): per span token the L1 KV
    deviation between one layer of the reused cache and of a fresh recomputation ([blocks, 16, H, d]
    each), top ceil(rho*m) marked (default 15% = 3/20).  Returns (dev, bits, score_offsets,
    bits_word_offsets) like score_deviation."""
    S = len(span_l)
    q_, l_, r_ = _i32(span_req), _i32(span_l), _i32(span_r)
    ms = r_ - l_ + 1
    so, bo = _offsets(ms)
    dev = reused_k.device
    if out_scores is None:
        out_scores = torch.zeros(max(int(so[-1]), 1), dtype=torch.int64, device=dev)
    if out_bits is None:
        out_bits = torch.zeros(max(int(bo[-1]), 1), dtype=torch.int32, device=dev)
    for t in (reused_k, reused_v, fresh_k, fresh_v):
        if not t.is_contiguous() or t.shape[1:] != reused_k.shape[1:] or t.dtype != reused_k.dtype:
            raise ValueError("caches must be contiguous [blocks, 16, H, d] of one dtype")
    H, d = int(reused_k.shape[2]), int(reused_k.shape[3])
    rbt, fbt = reused_block_tables.contiguous(), fresh_block_tables.contiguous()
    rc = L.lib().cp_score_kv_deviation(S, _cptr(q_, C.c_int32), _cptr(l_, C.c_int32), _cptr(r_, C.c_int32),
                                       _ptr(reused_k), _ptr(reused_v), _ptr(rbt), int(rbt.shape[1]), _ptr(fresh_k),
                                       _ptr(fresh_v), _ptr(fbt), int(fbt.shape[1]), H, d,
                                       L.CP_BF16 if reused_k.dtype == torch.bfloat16 else L.CP_FP32,
                                       rho_num, rho_den, int(ms.max()) if S else 1, _ptr(out_scores),
                                       _cptr(so, C.c_int64), _ptr(out_bits), _cptr(bo, C.c_int64), _stream(stream))
    L.check(rc, "cp_score_kv_deviation")
    return out_scores, out_bits, so.tolist(), bo.tolist()


def annotate_spans(attn: Sequence[torch.Tensor], masks: Sequence[torch.Tensor], heads: Sequence[int],
                   min_len: int = 128, max_segments: int = 64, workspace_bytes: int = 4 << 30, stream=None):
    """NEXT-1 (cp_annotate_spans): per request, per coarse segment, the reusable span (l, r, diff) of
    C1 Steps 1-2, or (-1, -1, 0).  Requests are processed in chunks that fit `workspace_bytes`."""
    lib = L.lib()
    R = len(attn)
    ns = [int(a.shape[-1]) for a in attn]
    out = [None] * R
    dev = attn[0].device if R else torch.device("cuda")
    # the workspace is a sum of per-request (256-B aligned) terms: size each request once, then chunk
    per = [int(lib.cp_annotate_workspace(1, (C.c_int32 * 1)(n), max_segments)) for n in ns]
    i = 0
    while i < R:
        j, tot = i + 1, per[i]
        while j < R and tot + per[j] <= workspace_bytes:
            tot += per[j]
            j += 1
        k = j - i
        n_arr = (C.c_int32 * k)(*ns[i:j])
        need = int(lib.cp_annotate_workspace(k, n_arr, max_segments))
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        nseg = torch.zeros(k, dtype=torch.int32, device=dev)
        ol = torch.full((k * max_segments,), -1, dtype=torch.int32, device=dev)
        orr = torch.full((k * max_segments,), -1, dtype=torch.int32, device=dev)
        od = torch.zeros(k * max_segments, dtype=torch.int64, device=dev)
        A = (C.c_void_p * k)(*[a.data_ptr() for a in attn[i:j]])
        M = (C.c_void_p * k)(*[m.data_ptr() for m in masks[i:j]])
        h_arr = (C.c_int32 * k)(*[int(h) for h in heads[i:j]])
        L.check(lib.cp_annotate_spans(k, A, n_arr, h_arr, M, min_len, max_segments, _ptr(ws), need, _ptr(nseg),
                                      _ptr(ol), _ptr(orr), _ptr(od), _stream(stream)), "cp_annotate_spans")
        nseg_h, ol_h, or_h, od_h = nseg.cpu().numpy(), ol.cpu().numpy(), orr.cpu().numpy(), od.cpu().numpy()
        for q in range(k):
            c = int(nseg_h[q])
            if c < 0:
                raise L.CacheHitError("cp_annotate_spans: more coarse segments than max_segments")
            b = q * max_segments
            out[i + q] = [(int(ol_h[b + s]), int(or_h[b + s]), int(od_h[b + s])) for s in range(c)]
        i = j
    return out


def hash_prefix(batch: DeviceBatch, hash_seed: int, stream=None) -> torch.Tensor:
    out = torch.zeros(batch.total_tokens + batch.num_reqs, dtype=torch.int64, device=batch.tokens.device)
    rb = batch.c(False)
    L.check(L.lib().cp_hash_prefix(C.byref(rb), int(hash_seed), _ptr(out), _stream(stream)), "cp_hash_prefix")
    return out


def policy_spans(batch: DeviceBatch, policy: str, chunk_len: int, max_len: int = 1 << 30, stream=None):
    """NEXT-3: the spans a baseline policy stores for a writer batch (cp_policy_spans); returns
    (span_req, span_begin, span_len) device int32 tensors.  Synchronizes (the count sizes them)."""
    code = {"fixed_chunk": L.CP_POLICY_FIXED_CHUNK, "prefix_only": L.CP_POLICY_PREFIX_ONLY}[policy]
    dev = batch.tokens.device
    cap = batch.total_tokens // max(chunk_len, 1) + 1 if policy == "fixed_chunk" else batch.num_reqs + 1
    out = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(3)]
    cnt_d = torch.zeros(1, dtype=torch.int32, device=dev)
    cnt_h = C.c_int32(0)
    rb = batch.c(True)
    L.check(L.lib().cp_policy_spans(C.byref(rb), code, int(chunk_len), int(min(max_len, 2**31 - 1)), cap,
                                    _ptr(out[0]), _ptr(out[1]), _ptr(out[2]), _ptr(cnt_d), C.byref(cnt_h),
                                    _stream(stream)), "cp_policy_spans")
    n = int(cnt_h.value)
    return tuple(o[:n] for o in out)


def kernel_launch_count() -> int:
    return int(L.lib().cp_kernel_launch_count())
