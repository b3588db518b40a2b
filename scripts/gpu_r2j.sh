#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_tools.py tests/test_gpu_hmatrix.py -q -p no:cacheprovider -k "c5 or blocks or guard or hmatrix or cur" > gpurun_out/pytest_j.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_j.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; head -6 gpurun_out/c5_time.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches_j.csv python scripts/c5_time.py > /dev/null 2>&1; echo "ncu rc=$?"
