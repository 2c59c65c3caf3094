"""Recall on the REFERENCE-built configs[0] index (tests/golden/
make_c1_reference.py writes data/c1_ref/: the reference's own .givf file,
queries, exact ground truth and the reference's recall / speed), searched by
this package on the GPU: the same index, the same queries, the reference's
as-shipped recall beside ours.

    python tools/c1_recall.py [--dir data/c1_ref] [--out profiles/r02_c1_recall.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default=os.path.join(ROOT, "data", "c1_ref"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_c1_recall.json"))
    args = ap.parse_args()
    import torch

    from paper_1802_02422_b200 import SearchParams, load_index, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex
    from paper_1802_02422_b200.query import recall_at_r

    ref = json.load(open(os.path.join(args.dir, "reference.json")))
    arr = load_index(os.path.join(args.dir, "c1.givf"))
    q = np.load(os.path.join(args.dir, "queries.npy"))
    gt = np.load(os.path.join(args.dir, "gt.npy"))
    dev = DeviceIndex(arr)
    out = {"index": "reference-built configs[0] (data/c1_ref/c1.givf, reference storage format)",
           "reference": ref["runs"], "ours": []}
    for ef in (128, arr.k):
        p = SearchParams(nprobe=32, tau=0.5, candidates=10_000, ef_search=ef)
        qd = torch.from_numpy(q).cuda()
        search_batch(dev, qd, p, k=100)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            ids, _, _ = search_batch(dev, qd, p, k=100)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        ids = ids.cpu().numpy()
        rec = {f"recall@{r}": float(recall_at_r(ids, gt, r)) for r in (1, 10, 100)}
        full = search_batch(dev, q, p)  # the reference's full result form
        rec_full = {f"full_recall@{r}": float(recall_at_r(full, gt, r)) for r in (1, 10, 100)}
        out["ours"].append(dict(ef_search=ef, nprobe=32, tau=0.5, candidates=10_000,
                                probe="exact (ef_search is validated, the probe is exact)",
                                qps_device_resident=len(q) / dt, **rec, **rec_full))
        print(ef, rec, rec_full, f"{len(q) / dt:.0f} q/s", flush=True)
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
