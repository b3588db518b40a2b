#!/bin/bash
# development loop: parity quick check + c3/c4 bench lines
[ -z "$NOPARITY" ] && timeout 300 python scripts/quick_parity.py 2>&1 | tail -12
for args in "$@"; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args 2>&1 | tail -2 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config']['workload'], d['config']['mode'], 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms/step', round(d['ms_per_step'],3), d['kernels_ms_per_step'], 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))
"
done
