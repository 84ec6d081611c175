"""Hot-path-only driver for compute-sanitizer --tool initcheck: config-1 rounds of insert -> match ->
gather -> score -> link -> split insert, without the diagnostic snapshot (which copies whole
workspace arrays, unused slots included, to the host).  Round 2 adds: the paper-literal placeholders
(uncovered list), CP_SKIP_RECOMPUTE, a pool view (copy-in + gather with the reused work list), pins,
session inserts and session-tagged matching, and the matcher work counters."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from synth.gen import attention_torch, make_workload  # noqa: E402
from tests.harness import Case  # noqa: E402


def main():
    wl = make_workload(1)
    case = Case(wl, max_sessions=16, batch_slack=8)
    dev = case.device
    # a pool view of layer 1, created with the index: every insert's copy-in also fills it
    v = case.dev.view(1, case.cfg.num_kv_heads, 1, 0)
    one = lambda p: cp.PagedKV(p.k[1:2], p.v[1:2], p.block_tables)
    for k, (wb, rb) in enumerate(wl.rounds):
        kv = case.writer_kv(wb)
        db = case._dev_batch(wb)
        sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev) for a in (wb.span_req, wb.span_begin, wb.span_len)]
        attn = [attention_torch(int(wb.lens[int(r)]), wb.segments[int(r)], 0.01, seed=int(r), device=dev) for r in wb.span_req]
        ls = [int(b) for b in wb.span_begin]
        rs = [int(b) + int(m) - 1 for b, m in zip(wb.span_begin, wb.span_len)]
        _, bits, so, bo = cp.score_deviation(attn, [int(wb.lens[int(r)]) for r in wb.span_req], [1] * len(ls), ls, rs)
        boff = torch.tensor(bo[:-1] or [0], dtype=torch.int64, device=dev)
        if k % 2:
            case.dev.insert(db, kv, *sp, bits, boff, 2 * k + 1, phase="prepare")
            case.dev.insert(db, kv, *sp, bits, boff, 2 * k + 1, phase="commit")
        else:
            case.dev.insert(db, kv, *sp, bits, boff, 2 * k + 1)
        v.copy_in(db, one(kv), reuse_worklist=True)
        rdb = case._dev_batch(rb)
        hits = case.dev.match_spans(rdb, 2 * k + 2)
        dst = case.dst_kv(rb)
        link = case.dev.link_blocks(rdb, hits, dst.block_tables.shape[1])
        case.dev.gather_rerotate(rdb, hits, dst, skip_linked=True)
        case.dev.gather_rerotate(rdb, hits, dst, zero_recompute=True, zero_uncovered=True)
        case.dev.gather_rerotate(rdb, hits, dst, skip_recompute=True)
        case.dev.pin_links(link, 1)
        case.dev.match_work()
        torch.cuda.synchronize()
        assert case.dev.last_error() == 0
        # same-user sessions: the writers are their sessions' last turns; readers of those sessions
        ss = np.arange(1, wb.num_reqs + 1, dtype=np.int32)
        sdb = cp.DeviceBatch.from_numpy(wb.tokens, wb.offsets, wb.mask, dev, session=ss)
        case.dev.insert_session(sdb, kv, 2 * k + 2)
        v.copy_in(sdb, one(kv), reuse_worklist=True)
        rs = cp.DeviceBatch.from_numpy(rb.tokens, rb.offsets, rb.mask, dev,
                                       session=(np.arange(rb.num_reqs) % (wb.num_reqs + 1)).astype(np.int32))
        h2 = case.dev.match_spans(rs, 2 * k + 3)
        case.dev.gather_rerotate(rs, h2, dst)
        case.dev.pin_links(link, -1)
        torch.cuda.synchronize()
        assert case.dev.last_error() == 0
    # the view gathers with the base's hits and the reused work list
    wb, rb = wl.rounds[-1]
    kv = case.writer_kv(wb)
    db = case._dev_batch(wb)
    sp = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev) for a in (wb.span_req, wb.span_begin, wb.span_len)]
    case.dev.insert(db, kv, *sp, None, None, 100)
    v.copy_in(db, one(kv), reuse_worklist=True)
    rdb = case._dev_batch(rb)
    hits = case.dev.match_spans(rdb, 101)
    dst = case.dst_kv(rb)
    case.dev.gather_rerotate(rdb, hits, dst)
    v.gather_rerotate(rdb, hits, one(dst), reuse_worklist=True)
    torch.cuda.synchronize()
    assert case.dev.last_error() == 0
    print("initcheck path OK")


if __name__ == "__main__":
    main()
