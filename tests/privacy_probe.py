"""Desk-scale reuse-oracle probing: the privacy pin of SURVEY §8(c) (test infrastructure).

The side channel is the binary reuse oracle R(p) = "the match of probe p has a hit" (SPEC S:L402-419,
`reuse_oracle`: "returns 1 iff match_request(probe).match_rate > 0; this is the only signal exposed to
the attack harness").  The adversary is the strongest black-box one at desk scale (SPEC S:L537-546,
`attack_probe_loop`; "a strong adversary with unlimited probing capability"): it knows
every writer's prompt except the sensitive tokens, and for every position p and every substring
[a, b) of the prompt that contains p (w <= b - a <= Lmax, Lmax = the longest stored segment) it probes
all V values v of the token at p.  A token is DIRECTLY RECOVERED iff some such substring gives
R(true value) = 1 and R(v) = 0 for some other v -- the reuse signal singles the true token out.

Workloads: vocabulary V = 16, public text in [0, 12) built from a few shared motifs (so stored segments
recur across writers), sensitive runs of 1-3 tokens drawn from [12, 16) (fresh values, as PII is:
a public segment can never reproduce a secret by coincidence).  Insert-time masks are the ground
truth with a fraction `fn_rate` of the sensitive tokens missed by the detector (false negatives,
SPEC acceptance 2 / PAPER Fig. 8-a): those are stored and become recoverable.

PAPER Table 4: "Direct Recovery" 0% on every dataset; SPEC acceptance 1.
Positive control: the same attack recovers the public tokens inside stored segments.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Tuple

import numpy as np

from synth.gen import Batch, pack_batches

V, PUBLIC, W = 16, 12, 4


@dataclass
class ProbeWorkload:
    writers: Batch                 # tokens, INSERT-time mask, spans = mask-0 runs >= W
    truth: np.ndarray              # ground-truth sensitive mask, per token of `writers`
    lmax: int


def make_workload(seed: int, n_writers: int = 6, fn_rate: float = 0.0, fn_order_seed: int = 0) -> ProbeWorkload:
    rng = np.random.default_rng(seed)
    motifs = [rng.integers(0, PUBLIC, int(rng.integers(W, 9))).astype(np.int32) for _ in range(4)]
    reqs = []
    for _ in range(n_writers):
        toks, sens = [], []
        n_target = int(rng.integers(20, 33))
        while sum(len(t) for t in toks) < n_target:
            if rng.random() < 0.55:
                t = motifs[int(rng.integers(0, len(motifs)))]
            else:
                t = rng.integers(0, PUBLIC, int(rng.integers(1, 7))).astype(np.int32)
            toks.append(t); sens.append(np.zeros(len(t), np.uint8))
            if rng.random() < 0.6:
                k = int(rng.integers(1, 4))
                toks.append(rng.integers(PUBLIC, V, k).astype(np.int32)); sens.append(np.ones(k, np.uint8))
        reqs.append((np.concatenate(toks), np.concatenate(sens)))
    truth = np.concatenate([s for _, s in reqs]).astype(np.uint8)
    # detector false negatives: a nested prefix of a fixed permutation of the sensitive positions
    sens_pos = np.nonzero(truth)[0]
    perm = np.random.default_rng(10_000 + fn_order_seed).permutation(len(sens_pos))
    missed = sens_pos[perm[: int(round(fn_rate * len(sens_pos)))]]
    mask = truth.copy()
    mask[missed] = 0
    parts, off = [], 0
    for r, (t, _) in enumerate(reqs):
        m = mask[off:off + len(t)]
        off += len(t)
        runs, i = [], 0
        while i < len(t):
            if m[i]:
                i += 1
                continue
            j = i
            while j < len(t) and not m[j]:
                j += 1
            runs.append((i, j))
            i = j
        sp = [(a, b - a) for a, b in runs if b - a >= W]
        parts.append(Batch(tokens=t.astype(np.int32), offsets=np.array([0, len(t)], np.int64), mask=m.copy(),
                           writer_ids=np.array([r], np.int64),
                           span_req=np.zeros(len(sp), np.int32), span_begin=np.array([a for a, _ in sp], np.int32),
                           span_len=np.array([l for _, l in sp], np.int32), segments=[runs]))
    wb = pack_batches(parts)
    lmax = int(wb.span_len.max()) if len(wb.span_len) else W
    return ProbeWorkload(wb, truth, lmax)


def probe_batch(wl: ProbeWorkload, positions: List[Tuple[int, int]]):
    """All probes for the listed (request, position) targets: every substring [a, b) of the request that
    contains the position, W <= b - a <= Lmax, with every value v at the position.  Returns the CSR
    probe batch (no mask: the adversary's probes carry none) and, per probe, (target index, substring
    index, v)."""
    wb = wl.writers
    toks, offs, meta = [], [0], []
    for ti, (r, p) in enumerate(positions):
        base = int(wb.offsets[r])
        n = int(wb.offsets[r + 1] - base)
        req = wb.tokens[base:base + n]
        si = 0
        for a in range(max(0, p - wl.lmax + 1), p + 1):
            for b in range(max(p + 1, a + W), min(n, a + wl.lmax) + 1):
                for v in range(V):
                    q = req[a:b].copy()
                    q[p - a] = v
                    toks.append(q); offs.append(offs[-1] + len(q)); meta.append((ti, si, v))
                si += 1
    batch = Batch(tokens=np.concatenate(toks).astype(np.int32) if toks else np.zeros(0, np.int32),
                  offsets=np.array(offs, np.int64), mask=np.zeros(offs[-1], np.uint8),
                  writer_ids=np.zeros(len(offs) - 1, np.int64))
    return batch, np.array(meta, np.int64).reshape(-1, 3)


def recovered(positions, meta: np.ndarray, oracle_bits: np.ndarray, true_vals) -> np.ndarray:
    """Per target: True iff some substring has R(true) = 1 and R(v) = 0 for another v."""
    out = np.zeros(len(positions), bool)
    if len(meta) == 0:
        return out
    R = oracle_bits.astype(bool)
    for ti in range(len(positions)):
        sel = meta[:, 0] == ti
        sub, vals, rr = meta[sel, 1], meta[sel, 2], R[sel]
        for s in np.unique(sub):
            k = sub == s
            rv = dict(zip(vals[k].tolist(), rr[k].tolist()))
            if rv.get(int(true_vals[ti]), False) and not all(rv.values()):
                out[ti] = True
                break
    return out


def attack(wl: ProbeWorkload, reuse_oracle: Callable[[Batch], np.ndarray], which: str = "sensitive",
           limit: int = 0):
    """Run the attack on the ground-truth sensitive positions ('sensitive') or on the public tokens
    inside stored segments ('public', positive control).  reuse_oracle(batch) -> uint8 per request.
    Returns (recovered, total, probes issued)."""
    wb = wl.writers
    positions, truev = [], []
    covered = np.zeros(wb.total_tokens, bool)
    for r, b0, m in zip(wb.span_req, wb.span_begin, wb.span_len):
        covered[int(wb.offsets[r]) + int(b0): int(wb.offsets[r]) + int(b0) + int(m)] = True
    for r in range(wb.num_reqs):
        base = int(wb.offsets[r])
        for p in range(int(wb.offsets[r + 1] - base)):
            g = base + p
            if (which == "sensitive" and wl.truth[g]) or (which == "public" and covered[g] and not wl.truth[g]):
                positions.append((r, p)); truev.append(int(wb.tokens[g]))
    if limit:
        positions, truev = positions[:limit], truev[:limit]
    if not positions:
        return 0, 0, 0
    batch, meta = probe_batch(wl, positions)
    bits = reuse_oracle(batch)
    rec = recovered(positions, meta, bits, truev)
    return int(rec.sum()), len(positions), int(batch.num_reqs)
