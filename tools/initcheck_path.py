"""Hot-path-only driver for compute-sanitizer --tool initcheck: config-1 rounds of insert -> match ->
gather -> score -> link -> split insert, without the diagnostic snapshot (which copies whole
workspace arrays, unused slots included, to the host)."""
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
    case = Case(wl)
    dev = case.device
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
        rdb = case._dev_batch(rb)
        hits = case.dev.match_spans(rdb, 2 * k + 2)
        dst = case.dst_kv(rb)
        case.dev.link_blocks(rdb, hits, dst.block_tables.shape[1])
        case.dev.gather_rerotate(rdb, hits, dst, skip_linked=True)
        torch.cuda.synchronize()
        assert case.dev.last_error() == 0
    print("initcheck path OK")


if __name__ == "__main__":
    main()
