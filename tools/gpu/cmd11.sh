timeout 600 python tools/synth_bench.py 2>&1 | tail -1 | cut -c1-250
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py 2>&1 | tail -2
