#!/bin/bash
# one full c3 step under ncu --set full (after a plain run of the same command exits 0)
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 1 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 16 -c 12 -o gpurun_out/c3_step $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"; tail -5 gpurun_out/ncu.log
