timeout 600 python tools/synth_bench.py 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_gpu_fused.py tests/test_gpu_parity_scale.py -k "suite or 128-0.25 or probe_lists" 2>&1 | tail -3
