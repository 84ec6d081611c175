"""NEXT-4 timing: CacheBlend KV-deviation selector (cp_score_kv_deviation; R#30) on the
config-2 shape: 256 requests x ~1.5K tokens, Llama-3-8B first-layer KV (8 heads x 128, bf16), one
span per request covering its passages (what CacheBlend would score), rho = 15%.

Algorithmic bytes per span token: 4 rows (reused K, V; fresh K, V) x H*d*2 B = 8 KiB; the kernel
is HBM-bound.  Writes gpurun_out/kvdev_bench.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23640_b200 as cp  # noqa: E402


def main():
    R, H, d = 256, 8, 128
    rng = np.random.default_rng(0)
    lens = rng.integers(1400, 1670, R)
    nb = [(int(n) + 15) // 16 for n in lens]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    caches = []
    for _ in range(2):
        perm = torch.from_numpy(rng.permutation(sum(nb)).astype(np.int32))
        bt = torch.zeros((R, max(nb)), dtype=torch.int32)
        o = 0
        for r, k in enumerate(nb):
            bt[r, :k] = perm[o:o + k]
            o += k
        K = torch.randn((sum(nb), 16, H, d), generator=gen, device="cuda").to(torch.bfloat16)
        V = torch.randn((sum(nb), 16, H, d), generator=gen, device="cuda").to(torch.bfloat16)
        caches.append((K, V, bt.cuda()))
    req = list(range(R))
    ls = [295] * R                                   # after the system prompt and question
    rs = [int(n) - 1 for n in lens]
    (rK, rV, rbt), (fK, fV, fbt) = caches
    args = (req, ls, rs, rK, rV, rbt, fK, fV, fbt, 3, 20)
    dev, bits, so, bo = cp.score_kv_deviation(*args)
    ref = (dev.clone(), bits.clone())
    variants = {}
    for var in ("1", "2", "3", "0"):                  # A/B of (loads per lane, CTAs per SM); 0 = default
        os.environ["CP_KVDEV_VARIANT"] = var
        for _ in range(2):
            cp.score_kv_deviation(*args, out_scores=dev, out_bits=bits)
        torch.cuda.synchronize()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            cp.score_kv_deviation(*args, out_scores=dev, out_bits=bits)
        e1.record()
        torch.cuda.synchronize()
        variants[var] = round(e0.elapsed_time(e1) / reps, 4)
        assert torch.equal(dev, ref[0]) and torch.equal(bits, ref[1])
    os.environ.pop("CP_KVDEV_VARIANT")
    ms = variants["0"]
    tokens = sum(r - l + 1 for l, r in zip(ls, rs))
    nbytes = tokens * 4 * H * d * 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = {"what": "cp_score_kv_deviation (rows + top-k), config-2 shape, bf16 8x128 first layer, rho 3/20",
           "spans": R, "span_tokens": tokens, "algorithmic_bytes": nbytes, "ms": round(ms, 4),
           "GBps": round(nbytes / ms / 1e6, 1), "peak_GBps": peak, "frac": round(nbytes / ms / 1e6 / peak, 4),
           "variants_ms": variants}
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "kvdev_bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
