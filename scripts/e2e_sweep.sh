#!/bin/bash
# e2e sub-batch size sweep on c3 (PCB_SUB_MB), device value unaffected; REPS runs per size
mkdir -p gpurun_out
for mb in ${MBS:-16 32 64 128}; do
  for rep in $(seq ${REPS:-1}); do
    PCB_SUB_MB=$mb python bench.py --config ${CFG:-c3} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$mb.json 2> gpurun_out/e2e_$mb.err
    python -c "import json;d=json.load(open('gpurun_out/e2e_$mb.json'));print($mb, round(d['value']), round(d['e2e']['value']))"
  done
done
