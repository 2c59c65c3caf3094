for S in 2x64 2x128 4x64 4x32 1x128; do
  echo "shape $S"; GIVF_FILTER_SHAPE=$S timeout 120 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1
done
GIVF_FILTER_SHAPE=2x64 timeout 120 python tools/probe_bench.py --nprobe 512 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_kernels.py -k "fused or modes" 2>&1 | tail -4
