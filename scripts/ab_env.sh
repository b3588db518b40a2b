#!/bin/bash
# A/B of a runtime switch: ENVVAR=0/1 over configs (bench only). usage: VAR=PCB_BUNDLE CFGS="c3 c2" bash scripts/ab_env.sh
mkdir -p gpurun_out
for cfg in ${CFGS:-c3 c2 c4 c1}; do
  for val in ${VALS:-0 1}; do
    env $VAR=$val python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abe_${cfg}_$val.json 2> gpurun_out/abe_${cfg}_$val.err
    python -c "import json;d=json.load(open('gpurun_out/abe_${cfg}_$val.json'));print('$cfg $VAR=$val', round(d['value']), round(d['e2e']['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/abe_${cfg}_$val.err
  done
done
