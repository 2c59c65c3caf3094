"""Builder throughput on the GPU: KA (nearest centroid) TFLOP/s at a
benchmark shape, KE rows/s, knn_exact, and optionally one full workload
build with its stage log.

    python tools/build_timing.py [--rows R] [--k K] [--d D] [--workload c3mini]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=3):
    import torch

    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1 << 22)
    ap.add_argument("--k", type=int, default=1 << 20)
    ap.add_argument("--d", type=int, default=96)
    ap.add_argument("--workload", default="")
    ap.add_argument("--noise", default="per_coord")
    args = ap.parse_args()
    import torch

    from paper_1802_02422_b200.builder import Model, assign_nearest, encode_rows, knn_exact

    out = {}
    x = torch.randn(args.rows, args.d, device="cuda")
    c = torch.randn(args.k, args.d, device="cuda")
    ms = timed(lambda: assign_nearest(x, c))
    flops = 2.0 * args.rows * args.k * args.d
    out["assign"] = {"rows": args.rows, "k": args.k, "d": args.d, "ms": ms,
                     "tflops_d": flops / ms / 1e9,
                     "tflops_mma": 2.0 * args.rows * args.k * ((args.d + 31) // 32 * 32) / ms / 1e9}
    print(json.dumps(out["assign"]), flush=True)
    k2 = 1 << 16
    cent = c[:k2].contiguous()
    nbr = torch.randint(0, k2, (k2, 64), device="cuda", dtype=torch.int32)
    md = Model(cent, nbr, torch.rand(k2, device="cuda"), torch.randn(16, 256, args.d // 16, device="cuda"),
               -1.0, 1.0, True, 64)
    reg = torch.randint(0, k2, (args.rows,), device="cuda", dtype=torch.int32)
    ms = timed(lambda: encode_rows(x, reg, md))
    out["encode"] = {"rows": args.rows, "ms": ms, "rows_per_s": args.rows / ms * 1e3}
    print(json.dumps(out["encode"]), flush=True)
    q = torch.randn(10_000, args.d, device="cuda")
    base = x[: 1 << 20].contiguous()
    ms = timed(lambda: knn_exact(q, base, 10))
    out["knn"] = {"nq": 10_000, "nb": 1 << 20, "ms": ms}
    print(json.dumps(out["knn"]), flush=True)
    del x, c
    torch.cuda.empty_cache()
    if args.workload:
        import bench
        from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic

        w = bench.WORKLOADS[args.workload]
        data = SynthSpec(d=w["d"], n_clusters=w["n_clusters"], sigma=0.3, noise=args.noise, seed=0,
                         kind=w.get("kind", "gauss"))
        spec = BuildSpec(n=w["n"], k=w["k"], l=w["l"], m=w["m"], n_learn=w["n_learn"],
                         kmeans_iters=w["kmeans_iters"], pq_iters=w["pq_iters"], seed=0)
        t0 = time.perf_counter()
        arr, qq, gt = build_synthetic(data, spec, w["nq"], device="cuda",
                                      log=lambda m: print(m, flush=True), rows_on_device=True)
        torch.cuda.synchronize()
        out["build"] = {"workload": args.workload, "s": time.perf_counter() - t0,
                        "max_group": int(arr.group_sizes.max()),
                        "nonempty_groups": int((arr.group_sizes > 0).sum())}
        print(json.dumps(out["build"]), flush=True)


if __name__ == "__main__":
    main()
