for S in 2x128 1x256 4x64; do for P in 64 512; do GIVF_FILTER_SHAPE=$S timeout 300 python tools/probe_bench.py --nprobe $P 2>&1 | tail -1 | cut -c1-170 | sed "s/^/$S /"; done; done
