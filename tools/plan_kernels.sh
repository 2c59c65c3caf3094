#!/bin/bash
# Per-launch durations of the planner kernels (ncu launch list, cold-cache,
# serialised) for the C2 bench; run after the same bench exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan|probe|scan" -c 60 --csv \
  --log-file gpurun_out/plan_kernels.csv python bench.py --workload c2 --steps 1 --warmup 3 \
  --no-cpu-baseline > gpurun_out/plan_kernels.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/plan_kernels.csv")) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows:
    v = float(r[vi].replace(",", "")); v = v / 1e3 if r[ui] == "nsecond" else v
    agg[r[ki].split("(")[0][:60]].append(v)
for k, v in agg.items():
    print(f"{k:60s} n={len(v):3d} mean_us={sum(v)/len(v):9.1f}")
PY
