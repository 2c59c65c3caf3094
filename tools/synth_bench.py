"""Search-path stage timings on a random index with the configs[2] shape,
built in seconds instead of bench.py's ~5-minute trained build: K = 2^20
random unit centroids, their exact 64-NN lists, rows spread uniformly over
the K x L groups (~15 rows per group at 1B rows, as in the trained index),
random codes.  Recall is meaningless here; timings of the probe, planner and
scan follow the shape (region / group / segment sizes, budget).  Small
enough to run under ncu (-k regex:<kernel> -s <skip> -c 1).

    python tools/synth_bench.py [--n 1000000000] [--k 1048576] [--nq 10000]
        [--nprobe 64] [--candidates 10000] [--steps 3] [--dedup]
"""

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(n, k, l, m, d, seed, log=print):
    import torch

    from paper_1802_02422_b200.builder import neighbor_centroids, norm_terms
    from paper_1802_02422_b200.device_index import IndexArrays

    t0 = time.perf_counter()
    g = torch.Generator(device="cuda").manual_seed(seed)
    cent = torch.randn(k, d, device="cuda", generator=g)
    cent /= cent.norm(dim=1, keepdim=True)
    nbr = neighbor_centroids(cent, l)
    alphas = 0.05 + 0.55 * torch.rand(k, device="cuda", generator=g)
    nt = norm_terms(cent, nbr, alphas)
    log(f"[synth] centroids + neighbors {time.perf_counter() - t0:.1f}s")
    # rows -> groups: sorted uniform keys, in chunks (1B int64 keys = 8 GB)
    gsize = torch.zeros(k * l, dtype=torch.int64, device="cuda")
    step = 1 << 28
    for s in range(0, n, step):
        c = min(step, n - s)
        key = torch.randint(0, k * l, (c,), device="cuda", generator=g, dtype=torch.int64)
        gsize += torch.bincount(key, minlength=k * l)
        del key
    gsize = gsize.reshape(k, l).int()
    offs = torch.zeros(k + 1, dtype=torch.int64, device="cuda")
    offs[1:] = torch.cumsum(gsize.sum(1).long(), 0)
    codes = torch.randint(0, 256, (n, m), device="cuda", generator=g, dtype=torch.uint8)
    cbytes = torch.randint(0, 256, (n,), device="cuda", generator=g, dtype=torch.uint8)
    pids = torch.randperm(n, device="cuda", dtype=torch.int32) if n <= (1 << 30) else \
        torch.arange(n, device="cuda", dtype=torch.int32)
    cw = 0.05 * torch.randn(m, 256, d // m, device="cuda", generator=g)
    arr = IndexArrays(
        centroids=cent.cpu().numpy(), alphas=alphas.cpu().numpy(),
        neighbor_ids=nbr.int().cpu().numpy(), norm_terms=nt.cpu().numpy(),
        group_sizes=gsize.cpu().numpy(), region_offsets=offs.cpu().numpy(), point_ids=pids,
        codes=codes, const_bytes=cbytes, codewords=cw.cpu().numpy(), rotation=None,
        const_lo=-0.5, const_hi=0.5, grouping=True)
    log(f"[synth] index arrays {time.perf_counter() - t0:.1f}s")
    return arr, cent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000_000)
    ap.add_argument("--k", type=int, default=1 << 20)
    ap.add_argument("--l", type=int, default=64)
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--d", type=int, default=96)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--nprobe", type=int, default=64)
    ap.add_argument("--tau", type=float, default=0.5)
    ap.add_argument("--candidates", type=int, default=10_000)
    ap.add_argument("--topk", type=int, default=100)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dedup", action="store_true", help="report neighbor-id duplication")
    args = ap.parse_args()
    import torch

    from paper_1802_02422_b200 import SearchParams, _native
    from paper_1802_02422_b200.device_index import DeviceIndex
    from paper_1802_02422_b200.query import search_batch

    arr, cent = build(args.n, args.k, args.l, args.m, args.d, args.seed)
    g = torch.Generator(device="cuda").manual_seed(args.seed + 1)
    src = torch.randint(0, args.k, (args.nq,), device="cuda", generator=g)
    q = cent[src] + 0.03 * torch.randn(args.nq, args.d, device="cuda", generator=g)
    q /= q.norm(dim=1, keepdim=True)
    dev = DeviceIndex(arr)
    del arr
    torch.cuda.empty_cache()
    p = SearchParams(nprobe=args.nprobe, tau=args.tau, candidates=args.candidates)
    ids = torch.empty(args.nq, args.topk, dtype=torch.int32, device="cuda")
    dists = torch.empty(args.nq, args.topk, dtype=torch.float32, device="cuda")
    stats = torch.empty(args.nq, 4, dtype=torch.int64, device="cuda")
    search_batch(dev, q, p, k=args.topk, out=(ids, dists, stats))
    torch.cuda.synchronize()
    if args.dedup:
        from paper_1802_02422_b200.query import probe

        regions, _ = probe(dev, q[:200].cpu().numpy(), args.nprobe)
        nbr = dev.arrays.neighbor_ids if hasattr(dev, "arrays") else None
        if nbr is not None:
            u = [len(np.unique(nbr[r].ravel())) for r in regions]
            print(f"[synth] unique neighbor ids per query: {np.mean(u):.0f} of "
                  f"{args.nprobe * args.l} ({np.mean(u) / (args.nprobe * args.l):.2f})")
    _native.profile_enable(True)
    _native.profile_read()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        search_batch(dev, q, p, k=args.topk, out=(ids, dists, stats))
    b.record()
    torch.cuda.synchronize()
    st = _native.profile_read()
    ms = a.elapsed_time(b) / args.steps
    print(f"[synth] n={args.n} K={args.k} nq={args.nq} P={args.nprobe}: {ms:.3f} ms/step "
          f"({args.nq / ms * 1e3 / 1e6:.3f}M q/s); "
          + ", ".join(f"{k} {v[0] / args.steps:.3f}" for k, v in st.items() if v[1])
          + f"; fallbacks {dev.fallback_counts()}; codes/query "
          f"{stats[:, 3].float().mean().item():.0f}")


if __name__ == "__main__":
    main()
