"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): golden-fixture searches through every search-path kernel (probe,
planner, LUTs, scan, full-mode rerank, scan order), the query-sharded plan /
localize / merge path, and -- with GIVF_PROBE=fused -- the fused probe and
K3a-from-fp16-rows.  Exits non-zero on any mismatch with the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
    GIVF_PROBE=fused compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import golden_io
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex
    from paper_1802_02422_b200.query import compact_plans, plan_batch, search_planned
    from paper_1802_02422_b200.sharded import merge_topk

    fx = golden_io.load("c1like_m16")
    q = fx.queries[:12]
    for p in (SearchParams(nprobe=32, tau=0.5, candidates=3000),
              SearchParams(nprobe=16, tau=1.0, candidates=800, rerank=False)):
        wi, wd, ws = so.search_topk(fx.index, q, so.Params(**vars(p)), 50)
        if p.rerank:  # top-k = the head of the reranked list
            ids, d, st = search_batch(fx.index, q, p, k=50)
            assert np.array_equal(st, ws), "stats"
            assert np.mean(ids == wi) > 0.99, "top-k ids"
        full = search_batch(fx.index, q, p)
        assert all(r.stats.codes_scanned == s[3] for r, s in zip(full, ws))
    # query-sharded plans over 2 shards on this device, K7 merge
    p = SearchParams(nprobe=32, tau=0.5, candidates=3000)
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32)).cuda()
    want_i, want_d, _ = search_batch(DeviceIndex(fx.index), qd, p, k=50)
    shards = [DeviceIndex(fx.index, shard=(g, 2)) for g in range(2)]
    it, n, _ = plan_batch(shards[0], qd, p)
    offs, flat = compact_plans(it, n)
    parts = [search_planned(s, qd, p, offs, flat, 50) for s in shards]
    mi, md = merge_topk(torch.stack([x[0] for x in parts]), torch.stack([x[1] for x in parts]), 50)
    assert torch.equal(mi, want_i) and torch.equal(md, want_d), "sharded merge"
    torch.cuda.synchronize()
    print("sanitize case ok", os.environ.get("GIVF_PROBE", "default"))


if __name__ == "__main__":
    main()
