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
from typing import Tuple


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


def score_owner(world: int, num_layers: int, by: str = "layer") -> int:
    """Rank holding the final layer's attention (runs N3).  Head sharding: rank 0 by convention
    (it must then hold the head-aggregated attention; see DESIGN.md multi-GPU)."""
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
