for MB in 4 2 1; do
  GIVF_FILTER_MB=$MB timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1
done
GIVF_FILTER_MB=2 timeout 300 python tools/probe_bench.py --nprobe 512 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_kernels.py -k "fused or modes" 2>&1 | tail -4
