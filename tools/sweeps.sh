#!/bin/bash
# BASELINE configs[1] nprobe x tau sweep and configs[4] batch x budget latency
# sweep on the C2 index, plus a C4 rehearsal (SIFT-like uint8, 50M x 128).
# Lines land in gpurun_out/; copy them to profiles/ to keep them.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --latency-sweep \
  --sweep 16:0.5,32:0.5,64:0.25,128:0.5,128:0.25,256:0.5,256:0.25 \
  > gpurun_out/sweep_c2.json 2> gpurun_out/sweep_c2.err
echo "c2 sweeps rc=$?"
timeout 1500 python bench.py --workload c4mini --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_c4mini.json 2> gpurun_out/bench_c4mini.err
echo "c4mini rc=$?"
