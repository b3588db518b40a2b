#!/bin/bash
# quick sweep used during development: bench lines for several configs/modes
set -x
mkdir -p gpurun_out
for args in "--config c3 --mode local" "--config c3 --mode global" "--config c4 --mode local" "--config c1" "--config c2"; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args 2>&1 | tail -3
done
