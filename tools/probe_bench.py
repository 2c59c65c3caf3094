"""Probe stage alone at a benchmark shape (K centroids, nq queries): times
givf_probe (K1a GEMM + select + recheck) with CUDA events; small enough to
run under ncu.

    python tools/probe_bench.py [--k 1048576] [--nq 10000] [--nprobe 64] [--reps 5]
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=1 << 20)
    ap.add_argument("--d", type=int, default=96)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--nprobe", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_1802_02422_b200 import _native
    from paper_1802_02422_b200.device_index import DeviceIndex, IndexArrays
    from paper_1802_02422_b200.query import probe

    rng = np.random.default_rng(0)
    k, d, m = args.k, args.d, 16
    c = rng.standard_normal((k, d)).astype(np.float32)
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    q = (c[rng.integers(0, k, args.nq)] + 0.03 * rng.standard_normal((args.nq, d))).astype(np.float32)
    arr = IndexArrays(
        centroids=c, alphas=np.zeros(k, np.float32), neighbor_ids=None, norm_terms=None,
        group_sizes=np.zeros((k, 1), np.int32), region_offsets=np.zeros(k + 1, np.int64),
        point_ids=np.zeros(0, np.int32), codes=np.zeros((0, m), np.uint8),
        const_bytes=np.zeros(0, np.uint8),
        codewords=rng.standard_normal((m, 256, d // m)).astype(np.float32), rotation=None,
        const_lo=0.0, const_hi=1.0, grouping=False)
    dev = DeviceIndex(arr)
    qd = torch.from_numpy(q).cuda()
    probe(dev, q, args.nprobe)
    torch.cuda.synchronize()
    _native.profile_enable(True)
    _native.profile_read()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        probe(dev, q, args.nprobe)
    b.record()
    torch.cuda.synchronize()
    st = _native.profile_read()
    print(f"probe K={k} nq={args.nq} P={args.nprobe}: {a.elapsed_time(b) / args.reps:.3f} ms/call; "
          + ", ".join(f"{n} {v[0] / args.reps:.3f}" for n, v in st.items() if v[1])
          + f"; fallbacks {dev.fallback_counts()}")


if __name__ == "__main__":
    main()
