"""A/B of the N3 row kernels (cp_set_score_variant: 0 a row per 8-lane group, 4 vectors per lane in flight, 4 CTAs/SM; 5: 16-lane groups; 6: 6 vectors at 3 CTAs/SM; 7: 4-lane groups; 4 the round-1 warp-per-row kernel, 1-3 its occupancy variants) on the bench's config-2
score call (512 spans of the 256 reader prompts, synthetic final-layer attention), CUDA events.
Prints ms and GB/s of algorithmic bytes (the row prefixes A[i][0..i] read)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402
from paper_2605_23640_b200 import _lib as L  # noqa: E402
from synth.gen import attention_torch, make_workload  # noqa: E402


def main():
    wl = make_workload(2)
    _, rb = wl.rounds[0]
    attn = {r: attention_torch(int(rb.lens[r]), rb.segments[r], 0.01, seed=r, device="cuda")
            for r in sorted(set(int(x) for x in rb.span_req))}
    args = ([attn[int(r)] for r in rb.span_req], [int(rb.lens[int(r)]) for r in rb.span_req], [1] * len(rb.span_req),
            [int(b) for b in rb.span_begin], [int(b) + int(m) - 1 for b, m in zip(rb.span_begin, rb.span_len)])
    nbytes = sum(4 * (i + 1) for l, r in zip(args[3], args[4]) for i in range(l, r + 1))
    L.check(L.lib().cp_set_score_variant(4))             # the register-staged row kernel as the reference
    sc, bits, so, bo = cp.score_deviation(*args, 1, 4)
    ref = (sc.clone(), bits.clone())
    # marshal once (the binding rebuilds 512-entry ctypes arrays per call; time the kernels, not that)
    import ctypes as C
    S = len(args[3])
    A = (C.c_void_p * S)(*[a.data_ptr() for a in args[0]])
    a32 = lambda xs: (C.c_int32 * S)(*[int(x) for x in xs])
    a64 = lambda xs: (C.c_int64 * S)(*[int(x) for x in xs])
    n_, h_, l_, r_ = a32(args[1]), a32(args[2]), a32(args[3]), a32(args[4])
    so_, bo_ = a64(so[:-1]), a64(bo[:-1])
    maxm = max(r - l + 1 for l, r in zip(args[3], args[4]))
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def call():
        L.check(L.lib().cp_score_deviation(S, A, n_, h_, l_, r_, 1, 4, 0, maxm, C.c_void_p(sc.data_ptr()), so_,
                                           C.c_void_p(bits.data_ptr()), bo_, stream))
    for v in (4, 0, 5, 6, 7):
        L.check(L.lib().cp_set_score_variant(v))
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        same = torch.equal(sc, ref[0]) and torch.equal(bits, ref[1])
        print(f"variant {v}: {ms:.4f} ms  {nbytes / ms / 1e6:.0f} GB/s  identical={same}")


if __name__ == "__main__":
    main()
