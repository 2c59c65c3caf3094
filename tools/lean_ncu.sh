#!/bin/bash
# ncu --set full (source counters) of one kernel on the configs[2]-shaped
# synthetic index, after the same command ran clean without ncu.
# usage: tools/lean_ncu.sh <kernel-regex> <out-name> [env settings...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
KREG=$1; OUT=$2; shift 2
CMD="python tools/synth_bench.py --steps 1"
env "$@" $CMD > gpurun_out/${OUT}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${OUT}_plain.log; exit 1; }
tail -1 gpurun_out/${OUT}_plain.log
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREG" -s 1 -c 1 \
    -f -o gpurun_out/$OUT $CMD > gpurun_out/${OUT}_ncu.log 2>&1
echo "ncu rc=$?"
