#!/bin/bash
# round 2 (e): full GPU suite, c5 timing, bench lines for every config, reference arm timing
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_e.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_e.log
timeout 300 python scripts/c5_time.py > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; head -8 gpurun_out/c5_time.json
for cfg in c1 c2 c4 c3; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/bench_e_$cfg.json 2> gpurun_out/bench_e_$cfg.err
  echo "bench $cfg rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_e_$cfg.json'));print('$cfg', round(d['value']), 'e2e', round(d['e2e']['value']), 'pageable', round(d['e2e']['pageable_value']), 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'], d['kernels_ms_per_step'], d['cpu_baseline'] and d['cpu_baseline'].get('value'))" || tail -3 gpurun_out/bench_e_$cfg.err
done
/usr/bin/time -v timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err
echo "ref rc=$?"; tail -c 1500 gpurun_out/ref_c3.json; grep -E "Elapsed|Maximum resident" gpurun_out/ref_c3.err
