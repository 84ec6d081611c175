"""Multi-process (world size 2, gloo, CPU) tests of the sharding + index-update protocol.

On the GPU box each rank runs the CUDA path on its layer shard; here the control protocol is
exercised with CPU tensors: the score owner (last-layer rank) computes the recompute bits from
the final-layer attention and broadcasts them; every rank applies the same inserts and must end
with a bit-identical index (checked with the oracle as the per-rank index model)."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_23640_b200.shard import broadcast_update, make_shard, score_owner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shards_partition_layers_and_heads():
    for L, H in [(32, 8), (80, 8), (2, 2)]:
        for world in [1, 2, 4, 8]:
            if world > L:
                continue
            shs = [make_shard(r, world, L, H, "layer") for r in range(world)]
            got = [l for s in shs for l in range(s.layer_lo, s.layer_hi)]
            assert got == list(range(L))
            assert all(s.head_lo == 0 and s.head_hi == H for s in shs)
            assert max(s.num_layers for s in shs) - min(s.num_layers for s in shs) <= 1
            own = score_owner(world, L, "layer")
            assert shs[own].layer_hi == L
            if world <= H:
                hs = [make_shard(r, world, L, H, "head") for r in range(world)]
                assert [h for s in hs for h in range(s.head_lo, s.head_hi)] == list(range(H))
    with pytest.raises(ValueError):
        make_shard(2, 2, 32, 8)


def test_balanced_layout_partitions_the_unit_grid():
    """The balanced layout (shard.make_layout 'balanced'): every (layer, head) unit on exactly one rank,
    each rank's rectangles contiguous in (layer, head) order, at most three per rank, the owner (last
    rank) holding the whole final layer and about `extra` units fewer than the others."""
    from paper_2605_23640_b200.shard import balanced_units, make_layout
    for L, H in [(32, 8), (80, 8), (2, 2), (32, 1)]:
        for world in [1, 2, 3, 4, 8]:
            if world > 1 and L * H - H < world - 1:
                with pytest.raises(ValueError):
                    make_layout(0, world, L, H, "balanced", 1.0)
                continue
            for extra in [0.0, 2.5, 6.0]:
                seen = []
                for r in range(world):
                    rects = make_layout(r, world, L, H, "balanced", extra)
                    assert 1 <= len(rects) <= 3
                    units = [l * H + h for s in rects for l in range(s.layer_lo, s.layer_hi)
                             for h in range(s.head_lo, s.head_hi)]
                    assert units == list(range(units[0], units[0] + len(units)))
                    seen += units
                assert seen == list(range(L * H))
                own = make_layout(world - 1, world, L, H, "balanced", extra)
                assert own[-1].layer_hi == L and any(s.layer_lo <= L - 1 < s.layer_hi and s.head_lo == 0
                                                     and s.head_hi == H for s in own)
                sizes = [b - a for a, b in balanced_units(world, L, H, extra)]
                if world > 1 and sizes[-1] > H:
                    others = sizes[:-1]
                    assert max(others) - min(others) <= 1
                    assert abs((sizes[-1] + extra) - sum(others) / len(others)) <= 1.0 + 1e-9


def _snapshot_digest(idx):
    h = hashlib.sha256()
    for e in idx.live_entries():
        h.update(repr((e["id"], e["len"], e["origin_pos"], e["prefix_hash"], e["full_hash"], e["last_used"],
                       e["digest"], e["pages"].tolist(), e["recompute"].tolist())).encode())
    h.update(np.asarray(idx.fifo()).tobytes())
    return h.hexdigest()


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle.oracle as O
        from synth.gen import attention_np, make_workload
        wl = make_workload(2, scale=0.03)
        g = wl.geometry
        sh = make_shard(rank, world, g.num_layers, g.num_kv_heads, "layer")
        owner = score_owner(world, g.num_layers, "layer")
        wb, rb = wl.rounds[0]
        w = g.window_len
        pages = (wl.pool_capacity_tokens + wl.max_span_len + 15) // 16 + (wl.pool_capacity_tokens + w - 1) // w + 1
        idx = O.OracleIndex(w, 42, wl.pool_capacity_tokens, pages)
        t = 0
        for batch in (wb, rb):                       # writers, then the readers' own segments
            t += 1
            m = [int(x) for x in batch.span_len]
            nwords = sum((x + 31) // 32 for x in m)
            bits = torch.zeros(max(nwords, 1), dtype=torch.int32)
            if rank == owner:                        # only the last-layer rank holds the attention
                flags = []
                for s in range(len(m)):
                    r = int(batch.span_req[s])
                    A = attention_np(int(batch.lens[r]), batch.segments[r], 0.01, seed=r)
                    b0 = int(batch.span_begin[s])
                    _, bw = O.score(A, b0, b0 + m[s] - 1, 1, 4)
                    flags.append(O.bits_to_bool(bw, m[s]))
                words, offs = O.pack_bits(flags)
                bits[:len(words)] = torch.from_numpy(words.view(np.int32))
            broadcast_update(bits, owner)            # C1: the index update crosses ranks
            words = bits.numpy().view(np.uint32)[:nwords]
            offs = np.concatenate([[0], np.cumsum([(x + 31) // 32 for x in m])]).astype(np.int64)
            rc, ids, oc = idx.insert(batch, words, offs, t)
            assert rc == 0
            t += 1
            idx.match(rb, t=t)                       # every rank matches redundantly (identical touches)
        dg = _snapshot_digest(idx)
        out = [None] * world
        dist.all_gather_object(out, (sh.layer_lo, sh.layer_hi, dg, len(idx.live_entries())))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_index_update_broadcast_keeps_replicas_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q), nprocs=2, join=True)
    out = q.get(timeout=60)
    (l0, h0, d0, n0), (l1, h1, d1, n1) = out
    assert (l0, h0, l1, h1) == (0, 16, 16, 32)
    assert d0 == d1 and n0 == n1 and n0 > 0
