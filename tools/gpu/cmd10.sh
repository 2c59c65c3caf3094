for D in 2 3 4; do GIVF_SCAN_DEPTH=$D timeout 600 python tools/synth_bench.py 2>&1 | tail -1 | sed "s/^/D=$D /" | cut -c1-200; done
