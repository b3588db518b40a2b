#!/bin/bash
# round 2 (h): c5 kernel (TMA zero blocks + gather queue): parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_hmatrix.py tests/test_gpu_tools.py -q -p no:cacheprovider -k "c5 or blocks or guard or hmatrix or cur" > gpurun_out/pytest_h.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_h.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; head -6 gpurun_out/c5_time.json
python scripts/c5_time.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blocks_tiled -s 3 -c 1 -o gpurun_out/r02h_c5 python scripts/c5_time.py > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
