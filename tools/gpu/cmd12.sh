timeout 600 python tools/c1_recall.py > gpurun_out/c1_recall.log 2>&1; tail -5 gpurun_out/c1_recall.log
timeout 1500 python -m pytest -q -x tests/test_gpu_sharded.py tests/test_dropin_surface.py tests/test_gpu_fused.py 2>&1 | tail -4
