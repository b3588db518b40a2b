#!/bin/bash
# parity (test_gpu_parity.py) + bench for the in-tree library and every build/ab/*.so variant
mkdir -p gpurun_out
for lib in default build/ab/*.so; do
  if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
  echo "== $lib: $(timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1)"
done
unset PCB_LIB_PATH
CFGS="${CFGS:-c3 c4 c2 c1}" bash scripts/ab_bench.sh
