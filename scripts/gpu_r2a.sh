#!/bin/bash
# round 2: full GPU suite + bench (c3 default) + launch list with DRAM bytes -> traffic json
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
lscpu > gpurun_out/lscpu.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
