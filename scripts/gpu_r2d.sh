#!/bin/bash
# round 2 (d): guard bands, c5 (classify + tiled), parity of blocks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tools.py tests/test_gpu_headline.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "guard or c5 or blocks or nccl or host_pipeline" > gpurun_out/pytest_d.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_d.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; cat gpurun_out/c5_time.json | head -8
