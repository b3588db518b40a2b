#!/bin/bash
# Round profile artefacts: bench line, launch list (gpu__time_duration, cold/serialised) and
# one `ncu --set full` capture of the dominant kernel.  Usage: profile_round.sh <tag> <kernel-regex> [bench args]
TAG=$1; KRE=$2; shift 2
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_$TAG.json
CMD="python bench.py --profile-only --steps 2 --warmup 3 $*"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s 2 -c 1 \
    -o gpurun_out/top_$TAG $CMD > gpurun_out/ncu_top.log 2>&1
echo "ncu-full rc=$?"
