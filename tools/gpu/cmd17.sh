for P in 64 512; do timeout 300 python tools/probe_bench.py --nprobe $P 2>&1 | tail -1 | cut -c1-220; done
for S in 4x64 1x128; do GIVF_FILTER_SHAPE=$S timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1 | cut -c1-200; done
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_kernels.py -k "fused or modes" 2>&1 | tail -2
timeout 900 python -m pytest -q -x tests/test_gpu_parity_scale.py -k "retry or probe_lists" 2>&1 | tail -2
