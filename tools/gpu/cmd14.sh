for S in 2x128 4x64 1x128; do GIVF_FILTER_SHAPE=$S timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1 | sed "s/^/$S /"; done
timeout 300 python tools/probe_bench.py --nprobe 512 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_kernels.py -k "fused or modes" 2>&1 | tail -2
