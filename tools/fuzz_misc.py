"""Long randomized GPU-vs-oracle runs of the NEXT rows' kernels (beyond the test suite's seeds):
  * annotator (cp_annotate_spans, NEXT-1): random causal matrices (1-3 heads, quantized values for
    ties, row-stochastic or not), random masks (including long runs), random min_len;
  * KV deviation (cp_score_kv_deviation, NEXT-4): random geometries / dtypes / spans / rho;
  * N3 score + top-k (cp_score_deviation): random spans up to 4000 rows, 1-2 heads, ties, rho 0..1.
Usage: python tools/fuzz_misc.py [seeds].  Writes gpurun_out/fuzz_misc.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle.oracle as O  # noqa: E402
import paper_2605_23640_b200 as cp  # noqa: E402


def annotate_case(seed):
    rng = np.random.default_rng(seed)
    min_len = int(rng.choice([1, 2, 5, 8, 16, 33]))
    mats, masks, heads, exp = [], [], [], []
    for _ in range(int(rng.integers(1, 10))):
        n = int(rng.integers(1, 400))
        h = int(rng.integers(1, 4))
        A = rng.uniform(0, 1, (h, n, n))
        if rng.random() < 0.4:
            A = np.floor(A * 4) / 4
        A = np.tril(A).astype(np.float32)
        if rng.random() < 0.5:
            A /= np.maximum(A.sum(-1, keepdims=True), 1e-6)
        m = (rng.random(n) < rng.uniform(0, 0.15)).astype(np.uint8)
        if rng.random() < 0.2 and n > 10:
            a = int(rng.integers(0, n - 5)); m[a:a + int(rng.integers(1, 40))] = 1
        mats.append(A); masks.append(m); heads.append(h)
        exp.append(O.annotate(A, m, min_len))
    dA = [torch.from_numpy(np.ascontiguousarray(A)).cuda() for A in mats]
    dM = [torch.from_numpy(m).cuda() for m in masks]
    os.environ["CP_ANN_VARIANT"] = str(seed % 3)          # auto / flat / split row walk
    got = cp.annotate_spans(dA, dM, heads, min_len=min_len, max_segments=256)
    os.environ.pop("CP_ANN_VARIANT")
    return got == exp


def kvdev_case(seed):
    rng = np.random.default_rng(seed)
    H, d = [(1, 8), (2, 64), (8, 128), (3, 16), (4, 32)][seed % 5]
    dt = torch.bfloat16 if seed % 2 else torch.float32
    if dt == torch.float32 and (H * d * 4) % 16:
        return True
    lens = [int(x) for x in rng.integers(1, 600, int(rng.integers(1, 6)))]
    gen = torch.Generator(device="cuda"); gen.manual_seed(seed)
    caches = []
    for _ in range(2):
        nb = [(n + 15) // 16 for n in lens]
        perm = torch.from_numpy(rng.permutation(sum(nb)).astype(np.int32))
        bt = torch.zeros((len(lens), max(nb)), dtype=torch.int32)
        o = 0
        for r, k in enumerate(nb):
            bt[r, :k] = perm[o:o + k]; o += k
        K = (torch.randn((sum(nb), 16, H, d), generator=gen, device="cuda") * float(rng.uniform(0.1, 4))).to(dt)
        V = (torch.randn((sum(nb), 16, H, d), generator=gen, device="cuda") * float(rng.uniform(0.1, 4))).to(dt)
        caches.append((K, V, bt.cuda()))
    (rK, rV, rbt), (fK, fV, fbt) = caches
    for r, n in enumerate(lens):                       # share some rows so deviations tie at 0
        q = torch.arange(n, device="cuda")
        keep = torch.from_numpy(rng.random(n) < 0.5).cuda()
        rb, fb = rbt[r, q // 16].long(), fbt[r, q // 16].long()
        fK[fb[keep], (q % 16)[keep]] = rK[rb[keep], (q % 16)[keep]]
        fV[fb[keep], (q % 16)[keep]] = rV[rb[keep], (q % 16)[keep]]
    spans = []
    for _ in range(int(rng.integers(1, 8))):
        r = int(rng.integers(len(lens))); lo = int(rng.integers(lens[r])); hi = int(rng.integers(lo, lens[r]))
        spans.append((r, lo, hi))
    num, den = [(3, 20), (1, 4), (0, 5), (5, 5), (2, 7)][seed % 5]
    req, ls, rs = zip(*spans)
    dev, bits, so, bo = cp.score_kv_deviation(req, ls, rs, rK, rV, rbt, fK, fV, fbt, num, den)
    dev, bits = dev.cpu().numpy(), bits.cpu().numpy().view(np.uint32)

    def rows(T, bt, r, lo, hi):
        q = torch.arange(lo, hi + 1, device="cuda")
        return T[bt[r, q // 16].long(), q % 16].float().reshape(len(q), -1).cpu().numpy()
    for s, (r, lo, hi) in enumerate(spans):
        m = hi - lo + 1
        od, ob = O.kv_deviation(rows(rK, rbt, r, lo, hi), rows(rV, rbt, r, lo, hi), rows(fK, fbt, r, lo, hi),
                                rows(fV, fbt, r, lo, hi), num, den)
        if not (np.array_equal(dev[so[s]:so[s] + m], od) and np.array_equal(bits[bo[s]:bo[s] + (m + 31) // 32], ob)):
            return False
    return True


def score_case(seed):
    rng = np.random.default_rng(seed)
    mats, ns, hs, ls, rs = [], [], [], [], []
    big = seed % 10 == 0
    for _ in range(int(rng.integers(1, 4 if big else 12))):
        n = int(rng.integers(1, 4000 if big else 600))
        h = int(rng.integers(1, 3))
        A = rng.uniform(0, 1, (h, n, n)).astype(np.float32)
        if rng.random() < 0.5:
            A = np.floor(A * 8) / 8
        A = np.tril(A).astype(np.float32)
        l = int(rng.integers(0, n)); r = int(rng.integers(l, n))
        mats.append(torch.from_numpy(A).cuda()); ns.append(n); hs.append(h); ls.append(l); rs.append(r)
    num, den = [(1, 4), (3, 20), (0, 3), (3, 3), (5, 11)][seed % 5]
    sc, bits, so, bo = cp.score_deviation(mats, ns, hs, ls, rs, num, den)
    sc, bits = sc.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
    for q in range(len(ns)):
        m = rs[q] - ls[q] + 1
        osc, ob = O.score(mats[q].cpu().numpy(), ls[q], rs[q], num, den)
        if not (np.array_equal(sc[so[q]:so[q] + m], osc) and np.array_equal(bits[bo[q]:bo[q] + (m + 31) // 32], ob)):
            return False
    return True


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    t0 = time.time()
    fails = {"annotate": [], "kvdev": [], "score": []}
    for s in range(seeds):
        if not score_case(70000 + s):
            fails["score"].append(70000 + s)
        if not annotate_case(50000 + s):
            fails["annotate"].append(50000 + s)
        if not kvdev_case(60000 + s):
            fails["kvdev"].append(60000 + s)
    out = {"seeds_each": seeds, "failures": fails, "seconds": round(time.time() - t0, 1)}
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fuzz_misc.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
