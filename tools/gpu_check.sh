#!/bin/bash
# One gpurun round trip: GPU tests (summary line) + a C2 bench (compact line).
# usage: tools/gpu_check.sh [bench args...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
echo "TESTS: $(tail -1 gpurun_out/gpu_tests.log)"
grep -E "^FAILED|Error" gpurun_out/gpu_tests.log | head -5
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline "$@" \
  > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench_c2.json"))
    print("BENCH:", round(d["value"]), "qps  e2e", round(d["e2e"]["value"] or 0), " r@10", d["config"]["recall@10"], d.get("fallback_queries_per_step"),
          {k: round(v, 3) for k, v in d["stage_ms_per_step"].items()})
except Exception as e:
    print("BENCH failed:", e)
    print(open("gpurun_out/bench_c2.err").read()[-2000:])
PY
