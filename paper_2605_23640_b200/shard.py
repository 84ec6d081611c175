"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed for plumbing).

Partitioning: the KV pool and every request's paged cache are split by LAYER
(or by KV head) across ranks; the index metadata (prefix table, entry table, token store, page
lists) is replicated and kept bit-identical on every rank because every rank applies the same
inserts in the same order and runs the same deterministic matcher.  No KV byte crosses NVLink.

The one real exchange step is the recompute marks: the final-layer attention that N3 scores
("attention scores of the final transformer layer only") lives on the rank that owns
the last layer, so that rank runs cp_score_deviation and broadcasts the packed bits (an index
update) to every other rank before the insert.  `broadcast_update` is that collective; it works
with NCCL on device tensors and with gloo on CPU tensors (tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    layer_lo: int
    layer_hi: int
    head_lo: int
    head_hi: int

    @property
    def num_layers(self) -> int:
        return self.layer_hi - self.layer_lo

    @property
    def num_heads(self) -> int:
        return self.head_hi - self.head_lo


def _split(n: int, parts: int, i: int) -> Tuple[int, int]:
    base, rem = divmod(n, parts)
    lo = i * base + min(i, rem)
    return lo, lo + base + (1 if i < rem else 0)


def make_shard(rank: int, world: int, num_layers: int, num_heads: int, by: str = "layer") -> Shard:
    """Contiguous layer ranges (by='layer') or KV-head ranges (by='head') per rank."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if by == "layer":
        if world > num_layers:
            raise ValueError("more ranks than layers")
        lo, hi = _split(num_layers, world, rank)
        return Shard(rank, world, lo, hi, 0, num_heads)
    if by == "head":
        if world > num_heads:
            raise ValueError("more ranks than KV heads")
        lo, hi = _split(num_heads, world, rank)
        return Shard(rank, world, 0, num_layers, lo, hi)
    raise ValueError(by)


def _rects(u0: int, u1: int, num_heads: int) -> List[Tuple[int, int, int, int]]:
    """Decompose the flat (layer, head) unit range [u0, u1) (unit = layer * H + head) into at most
    three rectangles (layer_lo, layer_hi, head_lo, head_hi): a trailing head range of the first layer,
    whole layers, a leading head range of the last layer."""
    H = num_heads
    out = []
    l0, h0 = divmod(u0, H)
    l1, h1 = divmod(u1, H)
    if u1 <= u0:
        return out
    if l0 == l1:
        return [(l0, l0 + 1, h0, h1)]
    if h0 > 0:
        out.append((l0, l0 + 1, h0, H))
        l0 += 1
    if l1 > l0:
        out.append((l0, l1, 0, H))
    if h1 > 0:
        out.append((l1, l1 + 1, 0, h1))
    return out


def balanced_units(world: int, num_layers: int, num_heads: int, owner_extra_units: float) -> List[Tuple[int, int]]:
    """Flat unit ranges per rank of the load-balanced layer layout.  Units (one KV head of one layer)
    are dealt out contiguously in (layer, head) order; the last rank owns the final layer (it holds the
    final-layer attention N3 scores) and carries N3's cost, `owner_extra_units` gather units'
    worth, so it gets that many fewer units -- but never less than the whole final layer."""
    U = num_layers * num_heads
    if world == 1:
        return [(0, U)]
    if U - num_heads < world - 1:
        raise ValueError("too few (layer, head) units: the owner keeps the final layer, every other rank needs one")
    target = (U + owner_extra_units) / world
    own = int(round(target - owner_extra_units))
    own = max(num_heads, min(U - (world - 1), own))
    rest = U - own
    ranges = [_split(rest, world - 1, r) for r in range(world - 1)]
    return ranges + [(rest, U)]


def make_layout(rank: int, world: int, num_layers: int, num_heads: int, by: str = "layer",
                owner_extra_units: float = 0.0) -> List[Shard]:
    """This rank's rectangles of the (layer, KV head) grid.  'layer' / 'head': one rectangle
    (make_shard).  'balanced': the layer layout with the N3 owner's share reduced by N3's cost
    (balanced_units), cut at head granularity -- up to three rectangles per rank, served by one
    index (the first rectangle) plus pool views (cp_index_create_view) for the others."""
    if by != "balanced":
        return [make_shard(rank, world, num_layers, num_heads, by)]
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if world > num_layers * num_heads:
        raise ValueError("more ranks than (layer, head) units")
    u0, u1 = balanced_units(world, num_layers, num_heads, owner_extra_units)[rank]
    return [Shard(rank, world, a, b, c, d) for a, b, c, d in _rects(u0, u1, num_heads)]


def score_owner(world: int, num_layers: int, by: str = "layer") -> int:
    """Rank holding the final layer's attention (runs N3).  Head sharding: rank 0 by convention
    (it must then hold the head-aggregated attention; see DESIGN.md multi-GPU)."""
    if by == "balanced":
        return world - 1
    if by == "layer":
        for r in range(world):
            if make_shard(r, world, num_layers, 1, "layer").layer_hi == num_layers:
                return r
    return 0


def broadcast_update(bits, src: int, group=None):
    """Broadcast the packed recompute bits of an insert (index update) from `src` to all ranks.
    `bits` must have the same shape/dtype on every rank; returns it (filled on non-src ranks)."""
    import torch.distributed as dist
    if bits.is_cuda and dist.get_backend(group) == "gloo":      # test configuration: stage through host
        host = bits.cpu()
        dist.broadcast(host, src=src, group=group)
        bits.copy_(host)
        return bits
    dist.broadcast(bits, src=src, group=group)
    return bits
