for PP in 0 2 3 4; do GIVF_PIPE=$PP timeout 300 python tools/synth_bench.py 2>&1 | tail -1 | cut -c1-120 | sed "s/^/PIPE=$PP /"; done
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py -k "modes" 2>&1 | tail -2
