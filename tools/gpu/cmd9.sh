timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_lean" -s 1 -c 1 -o gpurun_out/lean_prof python tools/synth_bench.py --steps 1 > gpurun_out/lean_ncu.log 2>&1
tail -2 gpurun_out/lean_ncu.log
