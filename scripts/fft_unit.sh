#!/bin/bash
# FFT engine unit test for every element-count setting the product compiles (fft.cuh PCB_E2/PCB_E3)
mkdir -p gpurun_out
for cfg in "16 24" "8 24" "8 12"; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 --expt-relaxed-constexpr -DPCB_E2=$1 -DPCB_E3=$2 \
       -Ipaper_1805_06018_b200/csrc -Iinclude scripts/fft_unit.cu -o gpurun_out/fft_unit_$1_$2 || exit 1
  echo "E2=$1 E3=$2: $(./gpurun_out/fft_unit_$1_$2 | tail -1)"
done
