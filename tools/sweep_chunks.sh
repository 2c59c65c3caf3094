#!/bin/bash
# qps and per-stage ms for a range of chunk sizes / stream counts (C2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for s in ${STREAMS:-2}; do for c in ${CHUNKS:-256 512 1024 2500 5000}; do
GIVF_STREAMS=$s GIVF_CHUNK_QUERIES=$c timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json;d=json.load(open('gpurun_out/b.json'))
print('S=$s C=$c', round(d['value']), {k: round(v, 3) for k, v in d['stage_ms_per_step'].items()}, d.get('fallback_queries_per_step'))" || tail -3 gpurun_out/b.err
done; done
