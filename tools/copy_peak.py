"""Copy-roofline reference: torch copy_ vs the gather's LDG.128.nc / STG.128.cs streaming copy
(cp_copy_diag) on 2 x 8 GiB buffers; prints GB/s (read + write bytes)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_23640_b200 import _lib as L  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    n = 8 << 30
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    a.random_(0, 255)
    out = {}
    ms = timed(lambda: b.copy_(a))
    out["torch_copy_"] = round(2 * n / ms / 1e6, 1)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for cps in (1, 2, 4, 8):
        ms = timed(lambda: L.lib().cp_copy_diag(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), n, cps, st))
        out[f"ldg_stg_stream_x{cps}"] = round(2 * n / ms / 1e6, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
