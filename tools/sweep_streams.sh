cd $GRAFT_REPO_ROOT
./tools/gpu_check.sh | grep -E "TESTS|BENCH|FAIL"
for s in 1 2 3 4; do for c in 512 1024 2048 5000; do
GIVF_STREAMS=$s GIVF_CHUNK_QUERIES=$c timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b.json'));print('S=$s C=$c', round(d['value']))"
done; done
