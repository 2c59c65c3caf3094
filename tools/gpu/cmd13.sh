python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && GIVF_PROBE=fused python tools/sanitize_case.py >> gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_case.py > gpurun_out/memcheck_default.log 2>&1; echo rc=$? >> gpurun_out/memcheck_default.log
GIVF_PROBE=fused timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_case.py > gpurun_out/memcheck_fused.log 2>&1; echo rc=$? >> gpurun_out/memcheck_fused.log
for f in gpurun_out/san_plain.log gpurun_out/memcheck_default.log gpurun_out/memcheck_fused.log; do echo == $f; tail -n 4 $f; done
