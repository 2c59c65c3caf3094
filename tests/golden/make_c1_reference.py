"""BASELINE configs[0] (C1) built and searched by the REFERENCE itself, for
the recall side of the metric.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c1_reference.py [--n 1000000]

1. C1 data: 1M x 96 rows from 4096 unit-norm cluster means plus gaussian
   noise (total sigma 0.3), L2-normalised (BASELINE configs[0]); a held-out
   learn set and 1000 queries from the same mixture; seed 0.
2. The reference's own build: train_kmeans (K = 4096), build_graph (its HNSW
   over the centroids), build_index (L = 64, M = 8, grouping on).
3. The reference's own search() at configs[0]'s parameters (nprobe 32,
   tau 0.5, 10k candidates), as shipped (ef_search = 128, the approximate
   graph probe) and with ef_search = K (exact probe), recall@1/10/100 against
   datasets.exact_ground_truth.
4. Writes data/c1_ref/ (git-ignored; gpurun ships it): the index in the
   reference's .givf format (storage.save_index), queries, ground truth, and
   the reference's recall / timing as JSON.  profiles/r02_c1_reference.json
   keeps the numbers.  The GPU side (tools/c1_recall.py) loads the same file
   through our storage reader and searches it.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from givf.datasets import exact_ground_truth  # noqa: E402
from givf.graph import build_graph  # noqa: E402
from givf.index import build_index  # noqa: E402
from givf.kmeans import train_kmeans  # noqa: E402
from givf.search import SearchParams, recall_at_r, search  # noqa: E402
from givf.storage import save_index  # noqa: E402
from givf.util import derive_seed  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def mixture(rng, means, n, sigma_total):
    lab = rng.integers(0, means.shape[0], n)
    x = means[lab] + np.float32(sigma_total / np.sqrt(means.shape[1])) * \
        rng.standard_normal((n, means.shape[1])).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=1000)
    ap.add_argument("--n-learn", type=int, default=200_000)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--kmeans-iters", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "data", "c1_ref"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    t00 = time.perf_counter()
    rng = np.random.default_rng(0)
    d = 96
    means = rng.standard_normal((4096, d)).astype(np.float32)
    means /= np.linalg.norm(means, axis=1, keepdims=True)
    base = mixture(rng, means, args.n, 0.3)
    learn = mixture(rng, means, args.n_learn, 0.3)
    queries = mixture(rng, means, args.nq, 0.3)
    log = lambda m: print(f"[{time.perf_counter() - t00:7.1f}s] {m}", flush=True)  # noqa: E731
    log("data")
    gt = exact_ground_truth(base, queries, k=100)
    log("ground truth")
    coarse = train_kmeans(learn, args.k, iters=args.kmeans_iters, seed=0)
    log("kmeans")
    graph = build_graph(coarse, max_links=32, ef_construction=256, seed=derive_seed(0, "graph"))
    log("graph")
    ix = build_index(base, coarse, graph, learn, l=64, m=8, grouping=True, seed=0,
                     progress=log)
    log("index")
    save_index(ix, os.path.join(args.out, "c1.givf"))
    np.save(os.path.join(args.out, "queries.npy"), queries)
    np.save(os.path.join(args.out, "gt.npy"), gt)
    out = {"config": "BASELINE configs[0] (C1)", "n": args.n, "d": d, "K": args.k, "L": 64, "M": 8,
           "nq": args.nq, "noise": "total sigma 0.3", "kmeans_iters": args.kmeans_iters,
           "build": "reference train_kmeans + build_graph(32, 256) + build_index", "runs": []}
    for ef, label in ((128, "as shipped (HNSW probe, ef_search=128)"),
                      (args.k, "exact probe (ef_search=K)")):
        p = SearchParams(nprobe=32, tau=0.5, candidates=10_000, ef_search=ef)
        t0 = time.perf_counter()
        res = [search(ix, q, p) for q in queries]
        dt = time.perf_counter() - t0
        rec = {f"recall@{r}": float(recall_at_r([x.ids for x in res], gt, r)) for r in (1, 10, 100)}
        out["runs"].append(dict(label=label, ef_search=ef, nprobe=32, tau=0.5, candidates=10_000,
                                qps_1core=args.nq / dt, **rec))
        log(f"{label}: {rec}, {args.nq / dt:.1f} q/s")
    with open(os.path.join(args.out, "reference.json"), "w") as f:
        json.dump(out, f, indent=1)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r02_c1_reference.json"), "w") as f:
        json.dump(out, f, indent=1)
    log("done")


if __name__ == "__main__":
    main()
