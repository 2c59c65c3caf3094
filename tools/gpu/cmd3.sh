GIVF_FILTER_MB=1 timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1
for MB in 2 4; do
GIVF_FILTER_MB=$MB python tools/probe_bench.py --nprobe 64 --reps 1 > gpurun_out/plain$MB.log 2>&1 && GIVF_FILTER_MB=$MB ncu --set full --clock-control none --import-source on -k regex:k_probe_filter -s 1 -c 1 -o gpurun_out/filter_mb$MB python tools/probe_bench.py --nprobe 64 --reps 1 > gpurun_out/ncu_mb$MB.log 2>&1
done
