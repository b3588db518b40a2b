#!/bin/bash
mkdir -p gpurun_out/final
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3"
$CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_cols<\(int\)256, \(int\)4, \(int\)1>' -s 2 -c 1 -o gpurun_out/final/c3_cols256 $CMD > gpurun_out/final/ncu_cols.log 2>&1
echo "ncu cols rc=$?"; tail -2 gpurun_out/final/ncu_cols.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_rows_inv_b<\(int\)128' -s 2 -c 1 -o gpurun_out/final/c3_rows_inv_b $CMD > gpurun_out/final/ncu_rinv.log 2>&1
echo "ncu rows_inv rc=$?"; tail -2 gpurun_out/final/ncu_rinv.log
