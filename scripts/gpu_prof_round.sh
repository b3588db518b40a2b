#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak | tee gpurun_out/fp64_peak.json
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
bash scripts/ncu_c3.sh
