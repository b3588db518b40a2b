#!/bin/bash
# FFT engine unit test for every element-count setting the product compiles (fft.cuh PCB_E2/PCB_E3/
# PCB_E2_SMALL_MAX): rows 8/24, cols 16/24 with 8 for lengths <= 64, mid 8/12
mkdir -p gpurun_out
for cfg in "16 24 64 96 0" "16 24 0 0 0" "8 24 0 0 1" "8 24 0 0 0" "8 12 0 0 0"; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 --expt-relaxed-constexpr -DPCB_E2=$1 -DPCB_E3=$2 \
       -DPCB_E2_SMALL_MAX=$3 -DPCB_E3_SMALL_MAX=$4 -DPCB_RADIX_DESC=$5 -Ipaper_1805_06018_b200/csrc -Iinclude tests/cuda/fft_unit.cu -o gpurun_out/fft_unit_$1_$2_$3_$4_$5 || exit 1
  echo "E2=$1 E3=$2 small<=$3,$4 desc=$5: $(./gpurun_out/fft_unit_$1_$2_$3_$4_$5 | tail -1)"
done
