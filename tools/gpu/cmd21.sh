for P in 64 512; do timeout 300 python tools/probe_bench.py --nprobe $P 2>&1 | tail -1 | cut -c1-200; done
timeout 600 python tools/synth_bench.py 2>&1 | tail -1 | cut -c1-300
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_kernels.py -k "fused or modes" 2>&1 | tail -3
