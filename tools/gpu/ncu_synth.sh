ARGS="--steps 1"
python tools/synth_bench.py $ARGS > gpurun_out/s_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(probe|plan|scan|build_luts|query_f16|items|localize|collect|gather|merge|full)" -c 40 --csv \
  --log-file gpurun_out/r02_launches_c3synth.csv python tools/synth_bench.py $ARGS > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_scan_lean|k_probe_filter|k_plan_scores_direct|k_plan_approx" -s 5 -c 5 \
  -o gpurun_out/r02_c3synth_full python tools/synth_bench.py $ARGS > gpurun_out/ncu_f.log 2>&1
for f in gpurun_out/ncu_l.log gpurun_out/ncu_f.log; do tail -n 2 $f; done
