#!/bin/bash
mkdir -p gpurun_out
for z in 4 0 3; do
  PCB_C5_ZERO=$z timeout 300 python scripts/c5_time.py > gpurun_out/c5_$z.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/c5_time.json'));print('zero', $z, round(d['ms_per_call']*1e3,1), 'us/call', {k: round(v*1e3,1) for k,v in d['split_ms'].items()}, round(d['frac_hbm'],3))"
  cp gpurun_out/c5_time.json gpurun_out/c5_time_z$z.json
done
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_tools.py tests/test_gpu_hmatrix.py -q -p no:cacheprovider -k "c5 or blocks or guard or hmatrix or cur" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v.log
