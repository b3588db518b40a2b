#!/bin/bash
# `ncu --set full` of one step's launches of the three c3 LOCAL hot kernels (after a plain run exits 0)
# usage: ncu_three.sh <tag> [bench args]
TAG=${1:-c3_three}; shift
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_rows_inv_b<.int.128, .int.4>|k_cols<.int.256, .int.4, .int.1>|k_rows_fwd<.int.128, .int.4, .int.0>" \
    -s 15 -c ${NCU_C:-5} -o gpurun_out/$TAG $CMD > gpurun_out/ncu_three.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_three.log; ls -la gpurun_out/$TAG.ncu-rep
