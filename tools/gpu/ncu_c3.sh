ARGS="--steps 1 --warmup 1 --no-sweeps --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/b1.json 2> gpurun_out/b1.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(probe|plan|scan|build_luts|query_f16|items|localize|collect|gather|merge|full)" -c 60 --csv \
  --log-file gpurun_out/r02_launches_c3.csv python bench.py $ARGS > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_scan_lean|k_probe_filter|k_plan_scores_direct" -s 3 -c 3 \
  -o gpurun_out/r02_c3_full python bench.py $ARGS > gpurun_out/ncu_f.log 2>&1
tail -2 gpurun_out/ncu_l.log gpurun_out/ncu_f.log
