for T in 3 2 1; do for P in 64 512; do GIVF_FUSED_TARGET=$T timeout 300 python tools/probe_bench.py --nprobe $P 2>&1 | tail -1 | sed "s/^/T=$T /" | cut -c1-220; done; done
