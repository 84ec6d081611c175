"""GPU-vs-oracle parity harness (test infrastructure).

Runs the same seeded workload through the CUDA path (paper_2605_23640_b200, via the C-ABI) and
through the CPU oracle (oracle/), and compares:
  * insert outcomes and entry ids, and the whole live index (ids, lengths, origins, prefix/full
    hashes, SHA-256 digests, last_used, page lists, tokens, recompute bits, free-page FIFO) -- bit exact
  * hits (request, entry, dst, len, delta), per-request hit offsets, plan codes, covered /
    recompute / candidate counts -- bit exact
  * gathered rows: V (and K when delta == 0) bit exact, K within the north-star tolerance
    (fp32: max|dK| / max|K| <= 1e-5; bf16: max|dK| <= 2e-2), zero placeholders exactly +0.0,
    uncovered rows untouched.
No expected value comes from the CUDA path: the oracle replays the same inputs, and the expected
KV rows are the generator's payload re-rotated by the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

import oracle.oracle as O
from synth.gen import (Batch, Workload, bf16_round_np, fill_paged_kv_torch, make_workload,
                       payload_np)

SENTINEL = 5.0        # pre-filled into destination caches: outside every payload / rotated value


def rand_bits(spans_len: Sequence[int], rng: np.random.Generator, num: int = 1, den: int = 4):
    """Seeded recompute marks: exactly ceil(num*m/den) random positions per span (a generator, not N3)."""
    flags = []
    for m in spans_len:
        f = np.zeros(int(m), bool)
        k = -(-num * int(m) // den)
        f[rng.choice(int(m), size=k, replace=False)] = True
        flags.append(f)
    return flags


def block_tables(lens, rng, spans=None, reserve_dummy=True):
    """Each request gets ceil(n/16) blocks from a random permutation.  With `spans` (list per request
    of (begin, end)), blocks not overlapping any span all map to dummy block 0 (memory saving)."""
    R = len(lens)
    nb = [max(1, (int(n) + 15) // 16) for n in lens]
    need = []
    for r in range(R):
        if spans is None:
            need.append(np.ones(nb[r], bool))
        else:
            m = np.zeros(nb[r], bool)
            for (a, b) in spans[r]:
                m[a // 16:(b + 15) // 16] = True
            need.append(m)
    total = int(sum(int(x.sum()) for x in need))
    first = 1 if reserve_dummy else 0
    perm = rng.permutation(total) + first
    bt = np.zeros((R, max(nb)), np.int32)
    i = 0
    for r in range(R):
        for j in range(nb[r]):
            if need[r][j]:
                bt[r, j] = perm[i]; i += 1
    return bt, total + first


def payload_rows(writer: int, pos: np.ndarray, layer: int, H: int, d: int, head_offset: int, dtype: str,
                 kind: int) -> np.ndarray:
    v = payload_np(writer, pos.reshape(-1, 1, 1), layer, (np.arange(H) + head_offset).reshape(1, H, 1),
                   np.arange(d).reshape(1, 1, d), kind)
    return bf16_round_np(v) if dtype == "bf16" else v


@dataclass
class ParityReport:
    ok: bool = True
    notes: List[str] = field(default_factory=list)
    stats: Dict[str, float] = field(default_factory=dict)

    def fail(self, msg):
        self.ok = False
        self.notes.append(msg)


class Case:
    """A workload on one GPU shard + its oracle twin."""

    def __init__(self, wl: Workload, device="cuda", seed: int = 0, rho=(1, 4), layer_range=None,
                 head_range=None, sample_reqs: Optional[int] = None, sample_layers: Optional[Sequence[int]] = None,
                 use_reader_mask: bool = True, hash_seed: int = 42, policy: Optional[str] = None,
                 placeholders: str = "recompute", max_sessions: int = 0, batch_slack: int = 0):
        import torch
        import paper_2605_23640_b200 as cp
        self.torch, self.cp = torch, cp
        self.wl, self.device = wl, torch.device(device)
        g = wl.geometry
        self.l0, self.l1 = layer_range or (0, g.num_layers)
        self.h0, self.h1 = head_range or (0, g.num_kv_heads)
        self.g = g.shard(self.l0, self.l1, self.h0, self.h1)
        self.rng = np.random.default_rng(seed)
        self.rho = rho
        self.sample_reqs, self.sample_layers = sample_reqs, sample_layers
        self.use_reader_mask = use_reader_mask
        self.policy = policy                 # None: the method; "fixed_chunk" / "prefix_only": NEXT-3 baselines
        # R#14 zero placeholders: "recompute" (CP_ZERO_RECOMPUTE), "both" (+ CP_ZERO_UNCOVERED: paper-literal),
        # "none" (CP_SKIP_RECOMPUTE: recompute-marked rows left untouched)
        self.placeholders = placeholders
        lens = [int(b.lens.max()) for wb, rb in wl.rounds for b in (wb, rb) if b is not None]
        spans = [len(wb.span_len) for wb, rb in wl.rounds if wb is not None]
        if policy is not None:
            spans += [wb.total_tokens // g.window_len + wb.num_reqs for wb, rb in wl.rounds if wb is not None]
        reqs = [b.num_reqs for wb, rb in wl.rounds for b in (wb, rb) if b is not None]
        toks = [b.total_tokens for wb, rb in wl.rounds for b in (wb, rb) if b is not None]
        w = g.window_len
        self.cfg = cp.IndexConfig(
            num_layers=self.g.num_layers, num_kv_heads=self.g.num_kv_heads, head_dim=g.head_dim, dtype=g.dtype,
            rope_theta=g.rope_theta, rope_style=g.rope_style, window_len=w, hash_seed=hash_seed,
            pool_capacity_tokens=wl.pool_capacity_tokens,
            max_entries=min(131072, wl.pool_capacity_tokens // w + max(spans + [1]) + 64),
            max_span_len=wl.max_span_len, max_req_tokens=max(lens + [1]) + batch_slack,
            max_batch_reqs=max(reqs + [1]) + batch_slack, max_batch_tokens=max(toks + [1]) + 64 * batch_slack,
            max_spans_per_insert=max(spans + [1]), layer_offset=self.l0, head_offset=self.h0,
            max_sessions=max_sessions)
        self.dev = cp.KVIndex(self.cfg, self.device)
        self.orc = O.OracleIndex(w, hash_seed, wl.pool_capacity_tokens, self.dev.num_pages)
        self.calls: List[Batch] = []          # writer batch of each insert call (for payload identity)
        self.t = 0

    # ------------------------------------------------------------------ helpers
    def _dev_batch(self, b: Batch, with_mask=True, sessions=None):
        return self.cp.DeviceBatch.from_numpy(b.tokens, b.offsets, b.mask if with_mask else None, self.device,
                                              session=sessions)

    def insert_session(self, wb: Batch, sessions, rep: ParityReport):
        """R#33: every request of `wb` replaces its session's private entry, on the device and in the oracle."""
        self.t += 1
        t = self.t
        kv = self.writer_kv(wb)
        db = self._dev_batch(wb, sessions=np.asarray(sessions, np.int32))
        ids, oc = self.dev.insert_session(db, kv, t)
        err = self.dev.last_error()
        rc, oids, ooc = self.orc.insert_session(wb, sessions, t)
        if err != rc:
            rep.fail(f"insert_session t={t}: device status {err} != oracle {rc}")
            return
        if rc != 0:
            return
        self.calls.append(wb)
        ids, oc = ids.cpu().numpy(), oc.cpu().numpy()
        if not np.array_equal(oc, ooc) or not np.array_equal(ids, oids):
            rep.fail(f"insert_session t={t}: outcomes / ids differ: {oc[:6]} {ids[:6]} vs {ooc[:6]} {oids[:6]}")
        rep.stats["session_stored"] = rep.stats.get("session_stored", 0) + int(np.sum(ooc == O.STORED))
        del kv
        self.compare_index(rep, f"after insert_session t={t}")

    def _tdt(self):
        return self.torch.bfloat16 if self.g.dtype == "bf16" else self.torch.float32

    def writer_kv(self, wb: Batch, sparse: bool = False):
        torch = self.torch
        spans = None
        if sparse:
            spans = [[] for _ in range(wb.num_reqs)]
            for r, b0, m in zip(wb.span_req, wb.span_begin, wb.span_len):
                spans[int(r)].append((int(b0), int(b0) + int(m)))
        bt, nblocks = block_tables(wb.lens, self.rng, spans)
        kv = self.cp.PagedKV.allocate(self.g.num_layers, nblocks, self.g.num_kv_heads, self.g.head_dim,
                                      self._tdt(), torch.from_numpy(bt), self.device, zero=True)
        fill_paged_kv_torch(kv.k, kv.v, kv.block_tables, [int(x) for x in wb.lens], wb.writer_ids, self.g,
                            layer_offset=self.l0, head_offset=self.h0, only_ranges=spans)
        return kv

    def dst_kv(self, rb: Batch):
        torch = self.torch
        bt, nblocks = block_tables(rb.lens, self.rng)
        kv = self.cp.PagedKV.allocate(self.g.num_layers, nblocks, self.g.num_kv_heads, self.g.head_dim,
                                      self._tdt(), torch.from_numpy(bt), self.device, zero=False)
        for t in kv.k + kv.v:
            t.fill_(SENTINEL)
        return kv

    # ------------------------------------------------------------------ steps
    def policy_spans(self, wb: Batch, rep: ParityReport):
        """NEXT-3: each side derives the baseline store's spans on its own; they must agree exactly.
        Returns the writer batch with the oracle's spans (for the oracle and the payload) and the
        device's span tensors (for the device insert)."""
        import dataclasses
        db = self._dev_batch(wb)
        d_sr, d_sb, d_sl = self.cp.policy_spans(db, self.policy, self.g.window_len, self.wl.max_span_len)
        o_sr, o_sb, o_sl = O.policy_spans(wb, self.policy, self.g.window_len, self.wl.max_span_len)
        for name, d, o in (("req", d_sr, o_sr), ("begin", d_sb, o_sb), ("len", d_sl, o_sl)):
            if not np.array_equal(d.cpu().numpy(), o):
                rep.fail(f"policy_spans({self.policy}): span_{name} differs")
        rep.stats["policy_spans"] = rep.stats.get("policy_spans", 0) + len(o_sr)
        return dataclasses.replace(wb, span_req=o_sr, span_begin=o_sb, span_len=o_sl), (d_sr, d_sb, d_sl)

    def insert(self, wb: Batch, rep: ParityReport, bits_flags=None, sparse_kv=False, concurrent_readers=None,
               between=None):
        """concurrent_readers: a reader batch matched (NO_TOUCH) and gathered on the main stream while
        the device insert's read-only half (cp_index_insert_prepare) runs on a side stream; the commit
        follows both.  The oracle inserts sequentially (the NO_TOUCH match changes no state).
        between: a callable run after the device prepare and before the commit (it applies the same
        operation to the device and the oracle, e.g. a touching match or a pin); the oracle's insert
        follows it, so the device commit must decide as if the prepare had come after it."""
        torch = self.torch
        dev_spans = None
        if self.policy is not None:
            wb, dev_spans = self.policy_spans(wb, rep)
            if not rep.ok:
                return
        self.t += 1
        t = self.t
        if bits_flags is None:
            bits_flags = rand_bits(wb.span_len, self.rng, *self.rho)
        words, offs = O.pack_bits(bits_flags)
        kv = self.writer_kv(wb, sparse=sparse_kv)
        db = self._dev_batch(wb)
        sp = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(self.device)
        dwords = torch.from_numpy(words.view(np.int32).copy() if len(words) else np.zeros(1, np.int32)).to(self.device)
        doffs = torch.from_numpy(offs.astype(np.int64)).to(self.device)
        dsp = dev_spans if dev_spans is not None else (sp(wb.span_req), sp(wb.span_begin), sp(wb.span_len))
        if between is not None:
            self.dev.insert(db, kv, *dsp, dwords, doffs, t, phase="prepare")
            between()
            ids, oc = self.dev.insert(db, kv, *dsp, dwords, doffs, t, phase="commit")
        elif concurrent_readers is None:
            ids, oc = self.dev.insert(db, kv, *dsp, dwords, doffs, t)
        else:
            side, main = torch.cuda.Stream(), torch.cuda.current_stream()
            ready = torch.cuda.Event()
            ready.record(main)
            side.wait_event(ready)
            with torch.cuda.stream(side):
                self.dev.insert(db, kv, *dsp, dwords, doffs, t, phase="prepare")
            rdb = self._dev_batch(concurrent_readers, with_mask=self.use_reader_mask)
            hits = self.dev.match_spans(rdb, t, no_touch=True, use_mask=self.use_reader_mask, policy=self.policy)
            self.dev.gather_rerotate(rdb, hits, self.dst_kv(concurrent_readers), zero_recompute=True)
            main.wait_stream(side)
            ids, oc = self.dev.insert(db, kv, *dsp, dwords, doffs, t, phase="commit")
        err = self.dev.last_error()
        rc, oids, ooc = self.orc.insert(wb, words, offs, t)
        if err != rc:
            rep.fail(f"insert t={t}: device status {err} != oracle {rc}")
            return
        if rc != 0:
            return                          # rejected calls store nothing and are not counted by the oracle
        self.calls.append(wb)
        ids, oc = ids.cpu().numpy(), oc.cpu().numpy()
        if not np.array_equal(oc, ooc):
            rep.fail(f"insert t={t}: outcomes differ at {np.nonzero(oc != ooc)[0][:8]}")
        if not np.array_equal(ids, oids):
            rep.fail(f"insert t={t}: entry ids differ at {np.nonzero(ids != oids)[0][:8]}")
        rep.stats["stored"] = rep.stats.get("stored", 0) + int(np.sum((ooc == O.STORED) | (ooc == O.SUPERSEDED)))
        rep.stats["duplicate"] = rep.stats.get("duplicate", 0) + int(np.sum(ooc == O.DUPLICATE))
        del kv
        self.compare_index(rep, f"after insert t={t}")

    def compare_index(self, rep: ParityReport, where: str, tokens=True):
        snap = self.dev.snapshot(with_tokens=tokens)
        live = self.orc.live_entries()
        if snap["error"]:
            rep.fail(f"{where}: device error word {snap['error']}")
        if snap["num_live"] != len(live):
            rep.fail(f"{where}: live entries {snap['num_live']} != oracle {len(live)}")
            return
        if snap["live_tokens"] != self.orc.live_tokens:
            rep.fail(f"{where}: live tokens {snap['live_tokens']} != {self.orc.live_tokens}")
        if not np.array_equal(snap["fifo"], self.orc.fifo()):
            rep.fail(f"{where}: free-page FIFO differs")
        for de, oe in zip(snap["entries"], live):
            for k in ("id", "len", "origin_pos", "prefix_hash", "full_hash", "last_used", "digest", "pin", "owner"):
                if de[k] != oe[k]:
                    rep.fail(f"{where}: entry {oe['id']} field {k}: {de[k]!r} != {oe[k]!r}")
            if not np.array_equal(de["pages"], oe["pages"]):
                rep.fail(f"{where}: entry {oe['id']} page list differs")
            if tokens:
                if not np.array_equal(de["tokens"], oe["tokens"]):
                    rep.fail(f"{where}: entry {oe['id']} tokens differ")
                if not np.array_equal(de["recompute"], oe["recompute"]):
                    rep.fail(f"{where}: entry {oe['id']} recompute bits differ")
        rep.stats["live_entries"] = len(live)

    def match_and_gather(self, rb: Batch, rep: ParityReport, check_kv=True, no_touch=False, sessions=None):
        torch = self.torch
        self.t += 1
        t = self.t
        db = self._dev_batch(rb, with_mask=self.use_reader_mask,
                             sessions=None if sessions is None else np.asarray(sessions, np.int32))
        hits = self.dev.match_spans(db, t, no_touch=no_touch, use_mask=self.use_reader_mask, policy=self.policy)
        dst = self.dst_kv(rb) if check_kv else None
        if check_kv:
            ph = self.placeholders
            self.dev.gather_rerotate(db, hits, dst, zero_recompute=ph != "none", zero_uncovered=ph == "both",
                                     skip_recompute=ph == "none")
        err = self.dev.last_error()
        if err:
            rep.fail(f"match t={t}: device error {err}")
            return
        res = self.orc.match(rb, t, no_touch=no_touch, use_mask=self.use_reader_mask, policy=self.policy,
                             sessions=sessions)
        h = hits.to_host()
        if h["num_hits"] != res.num_hits:
            rep.fail(f"match t={t}: num_hits {h['num_hits']} != {res.num_hits}")
            return
        for k, ok in (("hit_req", res.hit_req), ("hit_entry", res.hit_entry), ("hit_dst", res.hit_dst),
                      ("hit_len", res.hit_len), ("hit_delta", res.hit_delta)):
            if not np.array_equal(h[k], ok):
                rep.fail(f"match t={t}: {k} differs")
        R = rb.num_reqs
        if not np.array_equal(h["req_hit_offsets"][:R + 1], res.req_hit_offsets):
            rep.fail(f"match t={t}: req_hit_offsets differ")
        if not np.array_equal(h["plan"][:rb.total_tokens], res.plan):
            rep.fail(f"match t={t}: plan codes differ at {np.nonzero(h['plan'][:rb.total_tokens] != res.plan)[0][:8]}")
        for k, ok in (("req_covered", res.req_covered), ("req_recompute", res.req_recompute),
                      ("req_candidates", res.req_candidates)):
            if not np.array_equal(h[k][:R], ok):
                rep.fail(f"match t={t}: {k} differs: {h[k][:R][:6]} vs {ok[:6]}")
        cov = int(res.req_covered.sum())
        rep.stats["covered"] = rep.stats.get("covered", 0) + cov
        rep.stats["tokens"] = rep.stats.get("tokens", 0) + rb.total_tokens
        rep.stats["hits"] = rep.stats.get("hits", 0) + res.num_hits
        rep.stats["moved_hits"] = rep.stats.get("moved_hits", 0) + int(np.sum(res.hit_delta != 0))
        if self.policy == "prefix_only":          # hits shorter than their entry (partial prefixes)
            rep.stats["partial_hits"] = rep.stats.get("partial_hits", 0) + sum(
                int(res.hit_len[i]) < self.orc.entry(int(res.hit_entry[i]))["len"] for i in range(res.num_hits))
        if check_kv:
            self.compare_kv(rb, res, dst, rep)
        self.compare_index(rep, f"after match t={t}", tokens=False)

    def compare_links(self, rb: Batch, rep: ParityReport):
        """NEXT-2: link table of a NO_TOUCH match of `rb` vs the oracle's (R#31)."""
        self.t += 1
        db = self._dev_batch(rb, with_mask=self.use_reader_mask)
        hits = self.dev.match_spans(db, self.t, no_touch=True, use_mask=self.use_reader_mask, policy=self.policy)
        res = self.orc.match(rb, self.t, no_touch=True, use_mask=self.use_reader_mask, policy=self.policy)
        maxb = max(1, int(max((int(n) + 15) // 16 for n in rb.lens)))
        got = self.dev.link_blocks(db, hits, maxb).cpu().numpy()
        if self.dev.last_error():
            rep.fail(f"link t={self.t}: device error {self.dev.last_error()}")
            return
        exp = self.orc.link_blocks(rb, res, maxb)
        if not np.array_equal(got, exp):
            rep.fail(f"link t={self.t}: link tables differ at {np.argwhere(got != exp)[:4].tolist()}")
        rep.stats["linked_blocks"] = rep.stats.get("linked_blocks", 0) + int((exp >= 0).sum())

    def _entry_origin(self, eid):
        e = self.orc.entry(int(eid))
        wb = self.calls[e["origin_call"]]
        return int(wb.writer_ids[e["origin_req"]]), e["origin_pos"]

    def compare_kv(self, rb: Batch, res, dst, rep: ParityReport):
        torch = self.torch
        g = self.g
        H, d = g.num_kv_heads, g.head_dim
        reqs = list(range(rb.num_reqs))
        if self.sample_reqs is not None and len(reqs) > self.sample_reqs:
            reqs = sorted(self.rng.choice(len(reqs), size=self.sample_reqs, replace=False).tolist())
        layers = list(range(g.num_layers)) if self.sample_layers is None else [l for l in self.sample_layers if l < g.num_layers]
        bt = dst.block_tables.cpu().numpy()
        max_dk, max_k = 0.0, 0.0
        for r in reqs:
            n = int(rb.lens[r])
            q = np.arange(n)
            blk = torch.from_numpy(bt[r, q // 16].astype(np.int64)).to(self.device)
            slot = torch.from_numpy((q % 16).astype(np.int64)).to(self.device)
            plan = res.plan[rb.offsets[r]:rb.offsets[r + 1]]
            hs = [i for i in range(res.num_hits) if res.hit_req[i] == r]
            for l in layers:
                gotK = dst.k[l][blk, slot].float().cpu().numpy()
                gotV = dst.v[l][blk, slot].float().cpu().numpy()
                expK = np.full((n, H, d), SENTINEL, np.float32)
                expV = np.full((n, H, d), SENTINEL, np.float32)
                for i in hs:
                    k0, m, delta = int(res.hit_dst[i]), int(res.hit_len[i]), int(res.hit_delta[i])
                    writer, origin = self._entry_origin(res.hit_entry[i])
                    pos = origin + np.arange(m)
                    lay = l + self.l0
                    kraw = payload_rows(writer, pos, lay, H, d, self.h0, g.dtype, 0)
                    vraw = payload_rows(writer, pos, lay, H, d, self.h0, g.dtype, 1)
                    krot = O.rerotate_rows(kraw, H, d, g.rope_theta, delta, g.dtype == "bf16", g.rope_style == "gptj")
                    expK[k0:k0 + m] = krot
                    expV[k0:k0 + m] = vraw
                zero = plan == 2 if self.placeholders != "none" else np.zeros_like(plan, bool)
                if self.placeholders == "none":                       # recompute rows untouched
                    expK[plan == 2] = SENTINEL
                    expV[plan == 2] = SENTINEL
                if self.placeholders == "both":                       # unmatched rows zeroed too
                    zero = zero | (plan == 0)
                expK[zero] = 0.0
                expV[zero] = 0.0
                if not np.array_equal(gotV.view(np.uint32), expV.view(np.uint32)):
                    bad = np.nonzero(np.any(gotV != expV, axis=(1, 2)))[0]
                    rep.fail(f"gather: V differs req {r} layer {l} at positions {bad[:8]}")
                untouched = (plan == 0) if self.placeholders != "both" else np.zeros_like(plan, bool)
                if self.placeholders == "none":
                    untouched = untouched | (plan == 2)
                if not np.array_equal(gotK[untouched], expK[untouched]) or not np.array_equal(
                        gotK[zero].view(np.uint32), expK[zero].view(np.uint32)):
                    rep.fail(f"gather: K placeholder / untouched rows differ req {r} layer {l}")
                live = plan == 1
                if live.any():
                    dk = np.abs(gotK[live] - expK[live]).max()
                    max_dk = max(max_dk, float(dk)); max_k = max(max_k, float(np.abs(expK[live]).max()))
                # delta == 0 hits are bit copies
                for i in hs:
                    if int(res.hit_delta[i]) == 0:
                        k0, m = int(res.hit_dst[i]), int(res.hit_len[i])
                        sel = live[k0:k0 + m]
                        if not np.array_equal(gotK[k0:k0 + m][sel].view(np.uint32), expK[k0:k0 + m][sel].view(np.uint32)):
                            rep.fail(f"gather: delta=0 K not a bit copy req {r} layer {l}")
        rep.stats["max_abs_dK"] = max(rep.stats.get("max_abs_dK", 0.0), max_dk)
        rep.stats["max_abs_K"] = max(rep.stats.get("max_abs_K", 0.0), max_k)
        if g.dtype == "bf16":
            if max_dk > 2e-2:
                rep.fail(f"gather: bf16 K max-abs error {max_dk} > 2e-2")
        elif max_k > 0 and max_dk / max_k > 1e-5:
            rep.fail(f"gather: fp32 K relative error {max_dk / max_k} > 1e-5")

    def score_parity(self, wb: Batch, rep: ParityReport, max_spans: Optional[int] = None, lam=0.01):
        """N3 on device-generated attention (copied back for the oracle: a generator output)."""
        torch = self.torch
        from synth.gen import attention_torch
        idx = list(range(len(wb.span_len)))
        if max_spans is not None and len(idx) > max_spans:
            idx = sorted(self.rng.choice(len(idx), size=max_spans, replace=False).tolist())
        mats, ns, hs, ls, rs = {}, [], [], [], []
        for s in idx:
            r = int(wb.span_req[s])
            if r not in mats:
                mats[r] = attention_torch(int(wb.lens[r]), wb.segments[r] if wb.segments else (), lam, seed=r,
                                          device=self.device)
            ns.append(int(wb.lens[r])); hs.append(1)
            ls.append(int(wb.span_begin[s])); rs.append(int(wb.span_begin[s] + wb.span_len[s] - 1))
        attn = [mats[int(wb.span_req[s])] for s in idx]
        sc, bits, so, bo = self.cp.score_deviation(attn, ns, hs, ls, rs, *self.rho)
        sc, bits = sc.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
        host = {r: A.cpu().numpy() for r, A in mats.items()}
        for q, s in enumerate(idx):
            A = host[int(wb.span_req[s])]
            osc, obits = O.score(A, ls[q], rs[q], *self.rho)
            m = rs[q] - ls[q] + 1
            if not np.array_equal(sc[so[q]:so[q] + m], osc):
                rep.fail(f"score: span {s} scores differ")
            if not np.array_equal(bits[bo[q]:bo[q] + (m + 31) // 32], obits):
                rep.fail(f"score: span {s} bits differ")
        rep.stats["score_spans"] = rep.stats.get("score_spans", 0) + len(idx)


def ToyCase(device="cuda"):
    return Case(make_workload(1), device=device)


def run_round_parity(case: Case, rounds: Optional[int] = None, check_kv=True, score=True) -> dict:
    rep = ParityReport()
    for i, (wb, rb) in enumerate(case.wl.rounds[:rounds]):
        if wb is not None:
            case.insert(wb, rep)
            if score:
                case.score_parity(wb, rep)
        case.match_and_gather(rb, rep, check_kv=check_kv)
    out = dict(ok=rep.ok, notes=rep.notes[:20])
    out.update(rep.stats)
    return out
