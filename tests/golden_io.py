"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""

import json
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["small_grouped", "small_flat", "kat", "c1like_m8", "c1like_m16", "rot_m8"]


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    rot = z["ix_rotation"]
    lo, hi = z["ix_const_lohi"]
    ix = SimpleNamespace(
        centroids=z["ix_centroids"],
        alphas=z["ix_alphas"],
        neighbor_ids=z["ix_neighbor_ids"] if int(z["ix_grouping"][0]) else None,
        norm_terms=z["ix_norm_terms"] if int(z["ix_grouping"][0]) else None,
        group_sizes=z["ix_group_sizes"],
        region_offsets=z["ix_region_offsets"],
        point_ids=z["ix_point_ids"],
        codes=z["ix_codes"],
        const_bytes=z["ix_const_bytes"],
        codewords=z["ix_codewords"],
        rotation=rot if rot.size else None,
        const_lo=float(lo),
        const_hi=float(hi),
        grouping=bool(int(z["ix_grouping"][0])),
    )
    runs = []
    for j, p in enumerate(meta["params"]):
        offs = z[f"r{j}_offs"]
        ids, dists = z[f"r{j}_ids"], z[f"r{j}_dists"]
        per_q = [(ids[offs[i]:offs[i + 1]], dists[offs[i]:offs[i + 1]])
                 for i in range(len(offs) - 1)]
        runs.append(SimpleNamespace(params=SimpleNamespace(**p), results=per_q,
                                    stats=z[f"r{j}_stats"]))
    return SimpleNamespace(name=name, index=ix, queries=z["queries"], runs=runs,
                           note=meta["note"])


def exact_runs(fx):
    """Grid points run with the exact probe (ef_search == K)."""
    k = fx.index.centroids.shape[0]
    return [r for r in fx.runs if r.params.ef_search >= k or r.params.nprobe == k]
