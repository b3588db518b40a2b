#!/bin/bash
# A/B: twiddle recurrence in radix-16 stages / cols register caps
mkdir -p gpurun_out
CFGS="c3 c2 c4" bash scripts/ab_bench.sh
for lib in build/ab/*.so; do PCB_LIB_PATH=$PWD/$lib timeout 300 python scripts/quick_parity.py 2>&1 | grep -E "apply|ERR" | head -3; done
