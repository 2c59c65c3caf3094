timeout 600 python tools/synth_bench.py --dedup > gpurun_out/synth1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_warp|k_plan_scores_direct|k_plan_approx|k_plan_rescore" -s 4 -c 4 -o gpurun_out/synth_prof python tools/synth_bench.py --steps 1 > gpurun_out/synth_ncu.log 2>&1
tail -3 gpurun_out/synth1.log; tail -3 gpurun_out/synth_ncu.log
