for D in 0 1 2; do
GIVF_FILTER_DBG=$D GIVF_FILTER_MB=2 timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1
done
GIVF_FILTER_DBG=2 GIVF_FILTER_MB=4 timeout 300 python tools/probe_bench.py --nprobe 64 2>&1 | tail -1
