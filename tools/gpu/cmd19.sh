for W in 8 16; do GIVF_FILTER_WARPS=$W timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1 | cut -c1-200 | sed "s/^/EW=$W /"; done
GIVF_FILTER_WARPS=16 timeout 300 python tools/probe_bench.py --nprobe 512 2>&1 | tail -1 | cut -c1-200
timeout 300 python tools/probe_bench.py --nprobe 512 2>&1 | tail -1 | cut -c1-200
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_kernels.py -k "fused or modes" 2>&1 | tail -2
GIVF_FILTER_WARPS=16 timeout 900 python -m pytest -q -x tests/test_gpu_fused.py 2>&1 | tail -2
