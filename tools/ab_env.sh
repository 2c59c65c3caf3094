#!/bin/bash
# A/B a list of environment settings on the C2 bench: tools/ab_env.sh "A=1" "A=2 B=3" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'))
print('$cfg'.ljust(36), round(d['value']), {k: round(v, 3) for k, v in d['stage_ms_per_step'].items()}, d.get('fallback_queries_per_step'))" || tail -3 gpurun_out/ab.err
done
