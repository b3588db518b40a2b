#!/bin/bash
# round 2 (m): full GPU suite, estimator timing (mt19937 vs philox probes), c3/c4 bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_m.log
timeout 600 python scripts/estimator_time.py > gpurun_out/est.log 2>&1; echo "est rc=$?"; tail -2 gpurun_out/est.log
for cfg in c3 c4; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/bench_m_$cfg.json 2> gpurun_out/bench_m_$cfg.err
  echo "bench $cfg rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_m_$cfg.json'));print('$cfg', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['pageable_value']), 'frac', round(d['roofline']['frac'],3), d['roofline']['traffic_note'][:60])"
done
