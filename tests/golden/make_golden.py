"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture stores (1) the index arrays produced by the reference's own
`build_index` (index.py:249-380) and (2) the reference's own `search`
results (search.py:93-163) for a grid of SearchParams on a set of queries.
Searches run with `ef_search = index.k`, the reference configuration whose
probe is exact; one as-shipped grid point (ef_search=128) is
stored as well for information.  The GPU box never runs this script: the
`.npz` files travel, the reference does not.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from givf.datasets import synth_clustered  # noqa: E402
from givf.graph import build_graph  # noqa: E402
from givf.index import build_index  # noqa: E402
from givf.kmeans import train_kmeans  # noqa: E402
from givf.search import SearchParams, search  # noqa: E402
from givf.util import derive_seed  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def index_arrays(ix) -> dict:
    g = bool(ix.params.grouping)
    k = ix.k
    ngrp = ix.groups_per_region
    return {
        "ix_centroids": ix.coarse.centroids.astype(np.float32),
        "ix_alphas": ix.alphas.astype(np.float32),
        "ix_neighbor_ids": ix.neighbor_ids.astype(np.int32) if g else np.zeros((k, 0), np.int32),
        "ix_norm_terms": ix.norm_terms.astype(np.float32) if g else np.zeros((k, 0), np.float32),
        "ix_group_sizes": ix.group_sizes.astype(np.int32).reshape(k, ngrp),
        "ix_region_offsets": ix.region_offsets.astype(np.int64),
        "ix_point_ids": ix.point_ids.astype(np.int32),
        "ix_codes": ix.codes.astype(np.uint8),
        "ix_const_bytes": ix.const_bytes.astype(np.uint8),
        "ix_codewords": ix.pq.codewords.astype(np.float32),
        "ix_rotation": ix.pq.rotation.astype(np.float32) if ix.pq.rotation is not None
        else np.zeros((0, 0), np.float32),
        "ix_const_lohi": np.array([ix.const_quant.lo, ix.const_quant.hi], np.float64),
        "ix_grouping": np.array([1 if g else 0], np.int32),
    }


def run_grid(ix, queries, grid) -> dict:
    out = {}
    for j, p in enumerate(grid):
        ids, dists, offs, stats = [], [], [0], []
        for q in queries:
            r = search(ix, q, p)
            ids.append(r.ids.astype(np.int32))
            dists.append(r.distances.astype(np.float32))
            offs.append(offs[-1] + r.ids.shape[0])
            s = r.stats
            stats.append([s.regions_visited, s.subregions_visited,
                          s.subregions_pruned, s.codes_scanned])
        out[f"r{j}_ids"] = np.concatenate(ids) if ids else np.empty(0, np.int32)
        out[f"r{j}_dists"] = np.concatenate(dists) if dists else np.empty(0, np.float32)
        out[f"r{j}_offs"] = np.asarray(offs, np.int64)
        out[f"r{j}_stats"] = np.asarray(stats, np.int64)
    return out


def params_json(grid) -> str:
    return json.dumps([
        dict(nprobe=p.nprobe, tau=p.tau, candidates=p.candidates,
             ef_search=p.ef_search, rerank=p.rerank, prune=p.prune)
        for p in grid
    ])


def save(name, ix, queries, grid, note):
    t0 = time.perf_counter()
    data = index_arrays(ix)
    data["queries"] = np.asarray(queries, np.float32)
    data.update(run_grid(ix, queries, grid))
    data["meta"] = np.array(json.dumps({"name": name, "note": note,
                                        "params": json.loads(params_json(grid))}))
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **data)
    print(f"{name}: {os.path.getsize(path)/1e3:.0f} kB, grid {len(grid)}, "
          f"{len(queries)} queries, {time.perf_counter()-t0:.1f}s", flush=True)


def unit_mixture(rng, n, d, n_clusters, sigma, per_coord=True):
    """C1-family data: unit-norm means, gaussian noise, L2-normalised rows."""
    means = rng.standard_normal((n_clusters, d)).astype(np.float32)
    means /= np.linalg.norm(means, axis=1, keepdims=True)
    lab = rng.integers(0, n_clusters, n)
    s = sigma if per_coord else sigma / np.sqrt(d)
    x = means[lab] + np.float32(s) * rng.standard_normal((n, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(np.float32)


def fixture_small():
    # the reference's own test world (pkg/tests/conftest.py:32-72)
    data = synth_clustered(12_000, 16, 60, spread=0.4, seed=11)
    base, learn, queries = data[:10_000], data[10_000:11_900], data[11_900:]
    coarse = train_kmeans(learn, 48, iters=8, seed=5)
    graph = build_graph(coarse, max_links=8, ef_construction=48, seed=derive_seed(5, "graph"))
    k = 48
    grid = [
        SearchParams(nprobe=8, tau=0.5, candidates=300, ef_search=k),
        SearchParams(nprobe=4, tau=1.0, candidates=50, ef_search=k, rerank=False),
        SearchParams(nprobe=48, tau=1.0, candidates=10**9, ef_search=k),
        SearchParams(nprobe=16, tau=0.4, candidates=10**9, ef_search=k),
        SearchParams(nprobe=12, tau=0.7, candidates=900, ef_search=k, prune=False),
        SearchParams(nprobe=48, tau=0.4, candidates=2500, ef_search=k),
        SearchParams(nprobe=1, tau=1.0, candidates=137, ef_search=k),
        SearchParams(nprobe=8, tau=0.6, candidates=2000, ef_search=k, rerank=False),
        SearchParams(nprobe=48, tau=0.3, candidates=700, ef_search=k, rerank=False),
        SearchParams(nprobe=8, tau=0.5, candidates=300),  # as shipped (graph ef=128)
    ]
    ix = build_index(base, coarse, graph, learn, l=6, m=4, grouping=True, seed=5)
    save("small_grouped", ix, queries[:16], grid, "conftest world, grouped L=6 M=4")
    flat = build_index(base, coarse, graph, learn, l=6, m=4, grouping=False, seed=5)
    save("small_flat", flat, queries[:16], grid[:4], "conftest world, grouping off")


def fixture_kat():
    # test_search.py:157-170: one exactly representable point per centroid
    rng = np.random.default_rng(0)
    centers = rng.random((300, 6)).astype(np.float32)
    coarse = train_kmeans(centers, 300, iters=3, seed=1)
    graph = build_graph(coarse, max_links=6, ef_construction=24, seed=2)
    ix = build_index(centers, coarse, graph, centers, l=3, m=2, seed=3)
    grid = [SearchParams(nprobe=300, tau=1.0, candidates=300, ef_search=300),
            SearchParams(nprobe=17, tau=0.5, candidates=40, ef_search=300)]
    save("kat", ix, centers[[0, 111, 299, 5, 77]], grid, "exact reconstruction KAT")


def fixture_c1like(m, name, rotation=False, d=96, k=256, l=16, nq=16):
    rng = np.random.default_rng(1234 + m + (7 if rotation else 0) + d)
    x = unit_mixture(rng, 60_000 + nq, d, 400, 0.3, per_coord=False)
    base, learn, queries = x[:40_000], x[40_000:60_000], x[60_000:]
    coarse = train_kmeans(learn, k, iters=8, seed=3)
    graph = build_graph(coarse, max_links=12, ef_construction=64, seed=derive_seed(3, "graph"))
    ix = build_index(base, coarse, graph, learn, l=l, m=m, grouping=True, seed=3,
                     learn_rotation=rotation, pq_iters=8, rotation_rounds=2)
    grid = [
        SearchParams(nprobe=32, tau=0.5, candidates=10_000, ef_search=k),
        SearchParams(nprobe=16, tau=0.25, candidates=2_000, ef_search=k),
        SearchParams(nprobe=k, tau=0.5, candidates=5_000, ef_search=k),
        SearchParams(nprobe=64, tau=1.0, candidates=800, ef_search=k, prune=False),
        SearchParams(nprobe=24, tau=0.5, candidates=3_000, ef_search=k, rerank=False),
        SearchParams(nprobe=7, tau=0.9, candidates=150, ef_search=k),
        SearchParams(nprobe=32, tau=0.5, candidates=10_000),  # as shipped
    ]
    save(name, ix, queries, grid, f"C1-family d={d} K={k} L={l} M={m} rotation={rotation}")


def fixture_givf():
    """The conftest-world indexes (same seeds as fixture_small) written by the
    reference's own save_index (storage.py:114-127): byte-level fixtures for
    the .givf reader/writer.  Their arrays equal those stored in the .npz."""
    from givf.storage import save_index

    data = synth_clustered(12_000, 16, 60, spread=0.4, seed=11)
    base, learn = data[:10_000], data[10_000:11_900]
    coarse = train_kmeans(learn, 48, iters=8, seed=5)
    graph = build_graph(coarse, max_links=8, ef_construction=48, seed=derive_seed(5, "graph"))
    for name, grouping in (("small_grouped", True), ("small_flat", False)):
        ix = build_index(base, coarse, graph, learn, l=6, m=4, grouping=grouping, seed=5)
        ref = np.load(os.path.join(OUT, f"{name}.npz"))
        for key, val in index_arrays(ix).items():
            assert np.array_equal(ref[key], val), (name, key)
        path = os.path.join(OUT, f"{name}.givf")
        size = save_index(ix, path)
        print(f"{name}.givf: {size} bytes", flush=True)


def main():
    which = sys.argv[1:] or ["small", "kat", "m8", "m16", "rot", "givf"]
    if "small" in which:
        fixture_small()
    if "kat" in which:
        fixture_kat()
    if "m8" in which:
        fixture_c1like(8, "c1like_m8")
    if "m16" in which:
        fixture_c1like(16, "c1like_m16")
    if "rot" in which:
        fixture_c1like(8, "rot_m8", rotation=True, d=32, k=64, l=8, nq=10)
    if "givf" in which:
        fixture_givf()


if __name__ == "__main__":
    main()
