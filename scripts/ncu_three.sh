#!/bin/bash
# one `ncu --set full` capture of each of the three c3 LOCAL hot kernels (after a plain run exits 0)
CMD="python bench.py --config c3 --profile-only --steps 1 --warmup 3 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_rows_inv<.int.128, .int.4, .int.0>|k_cols<.int.256, .int.4, .int.1>|k_rows_fwd<.int.128, .int.4, .int.0>" \
    -s 12 -c 3 -o gpurun_out/c3_three $CMD > gpurun_out/ncu_three.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_three.log; ls -la gpurun_out/c3_three.ncu-rep
