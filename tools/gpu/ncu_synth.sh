ARGS="--steps 1"
python tools/synth_bench.py $ARGS > gpurun_out/s_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(probe_filter|probe_thresh|probe_pick|query_f16|plan_scores|plan_approx|plan_rescore|scan_lean|build_luts|collect_failed)" -c 40 --csv \
  --log-file gpurun_out/r02_launches_c3synth.csv python tools/synth_bench.py $ARGS > gpurun_out/ncu_l.log 2>&1
tail -n 1 gpurun_out/s_plain.log
