#!/bin/bash
mkdir -p gpurun_out
for z in 0 1 2; do
  PCB_C5_ZERO=$z timeout 300 python scripts/c5_time.py > gpurun_out/c5_$z.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/c5_time.json'));print('zero', $z, round(d['kernel_ms']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['split_ms'].items()}, round(d['kernel_frac_hbm'],3))"
  cp gpurun_out/c5_time.json gpurun_out/c5_time_z$z.json
done
PCB_C5_ZERO=2 timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "c5 or blocks" > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_l.log
