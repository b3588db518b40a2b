#!/bin/bash
# one `ncu --set full` capture of the first launch matching a kernel regex (after a plain run exits 0)
# usage: ncu_one.sh <tag> <regex> [bench args]
TAG=$1; KRE=$2; shift 2
CMD="python bench.py --profile-only --steps 1 --warmup 3 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s 3 -c 1 \
    -o gpurun_out/one_$TAG $CMD > gpurun_out/ncu_one.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_one.log
