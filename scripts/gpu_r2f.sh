#!/bin/bash
# round 2 (f): host pipeline (pooled pageable copies), c5 timing, bench c3 + reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tools.py tests/test_gpu_headline.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "host_pipeline or c5 or blocks or guard or cpp" > gpurun_out/pytest_f.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_f.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; head -12 gpurun_out/c5_time.json
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_f_c3.json 2> gpurun_out/bench_f_c3.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_f_c3.json'));print(round(d['value']), d['e2e'])"
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err
echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"; tail -c 1800 gpurun_out/ref_c3.json
