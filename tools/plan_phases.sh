#!/bin/bash
# Cycle split of k_plan_approx by phase (builds a -DGIVF_PHASES library).
cd "$(dirname "$0")/.."
make clean > /dev/null && make -j16 EXTRA=-DGIVF_PHASES > /dev/null 2>&1 || exit 1
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1802_02422_b200 import SearchParams
from paper_1802_02422_b200.device_index import DeviceIndex
from paper_1802_02422_b200 import _native
w = bench.WORKLOADS['c2']
arr, q, gt, _ = bench.load_or_build(w, 'per_coord', 0, 'cuda:0')
dev = DeviceIndex(arr)
p = SearchParams(nprobe=w['nprobe'], tau=w['tau'], candidates=w['candidates'])
from paper_1802_02422_b200.query import search_batch
qt = torch.from_numpy(q).cuda()
search_batch(dev, qt, p, k=100); torch.cuda.synchronize()
out = np.zeros(32, np.int64)
_native.check(_native.load().givf_index_counters(dev.handle, out.ctypes.data, 32))
before = out.copy()
search_batch(dev, qt, p, k=100); torch.cuda.synchronize()
_native.check(_native.load().givf_index_counters(dev.handle, out.ctypes.data, 32))
ph = (out - before)[8:24]
names = ['stage(q,regions)', 'w:classify', 'levels', 'bucket+walk', 'w:walk+cert', 'emit', 'rescore', 'w:f64 score',
         'stage:items', '-', 'w:gather', 'w:sort', 'emit:A compact', '-', '-', '-']
tot = ph.sum()
for n, v in zip(names, ph):
    print(f"PHASE {n:14s} {100*v/max(tot,1):5.1f}%  {v/q.shape[0]:10.0f} cycles/query")
print("fallbacks", (out-before)[:2], "window items/query", (out-before)[24] / q.shape[0], "begun/query", (out-before)[25] / q.shape[0])
PY
make clean > /dev/null && make -j16 > /dev/null 2>&1
