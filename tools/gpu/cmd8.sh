timeout 600 python tools/synth_bench.py 2>&1 | tail -1
GIVF_SCAN=warp timeout 600 python tools/synth_bench.py 2>&1 | tail -1
timeout 1500 python -m pytest -q -x tests -m gpu 2>&1 | tail -4
