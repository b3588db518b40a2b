#!/bin/bash
# ncu --set full of the split-3 row kernels beside their power-of-two counterparts (c3)
mkdir -p gpurun_out
cap() { # tag mixed_last regex
  PCB_MIXED_LAST=$2 python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/plain.log 2>&1 || { echo plain failed; return; }
  PCB_MIXED_LAST=$2 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$3" -s 2 -c 1 \
    -o gpurun_out/s3b_$1 -f python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
  python scripts/ncu_summary.py gpurun_out/s3b_$1.ncu-rep
}
cap inv128 0 'k_rows_inv_b<\(int\)128, \(int\)4, \(int\)0>'
cap inv96 2 'k_rows_inv_b<\(int\)96, \(int\)8, \(int\)0>'
cap fwd128 0 'k_rows_fwd<\(int\)128, \(int\)4, \(int\)0>'
cap fwd96 2 'k_rows_fwd<\(int\)96, \(int\)8, \(int\)0>'
