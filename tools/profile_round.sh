#!/bin/bash
# Round evidence on one B200: full bench line (with CPU baseline), reference
# arm, per-launch kernel list, and one ncu --set full capture of the top
# kernels (each only after the same command exited 0 without ncu).
# Everything lands in gpurun_out/; tools/summarize_profiles.py turns it into
# profiles/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_scan_warp|k_probe_gemm_tc|k_plan_approx|k_probe_select|k_plan_rescore|k_plan_scores_approx|k_probe_recheck|k_build_luts" \
    -s 8 -c 8 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
