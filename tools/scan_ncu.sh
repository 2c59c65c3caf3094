#!/bin/bash
# One ncu --set full capture of the warp scan on the C2 bench (after the same
# command ran clean without ncu); report in gpurun_out/scan_full.ncu-rep.
# usage: tools/scan_ncu.sh [env settings...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline"
env "$@" $CMD > gpurun_out/scan_plain.log 2>&1 && \
env "$@" ncu --set full --clock-control none --import-source on -k regex:k_scan_warp -s 2 -c 1 \
    -f -o gpurun_out/scan_full $CMD > gpurun_out/scan_ncu.log 2>&1
echo "scan ncu rc=$?"
