#!/bin/bash
# A/B environment settings on the C2 bench, device-resident and end-to-end:
# tools/ab_e2e.sh "A=1" "A=2 B=3" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg timeout 400 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'))
print('$cfg'.ljust(40), 'dev', round(d['value']), 'e2e', round(d['e2e']['value']))" || tail -3 gpurun_out/ab.err
done
