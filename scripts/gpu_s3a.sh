#!/bin/bash
# round-2 session 3: split-3 row engine -- parity, then A/B of the R2C-axis size rule (PCB_MIXED_LAST 0 / 2)
# and of the split-3 CTA size (build/ab variants)
mkdir -p gpurun_out
echo "== parity (default = mixed_last 2): $(timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3)"
for lib in default build/ab/*.so; do
  if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
  tag=$(basename $lib .so)
  for ml in 0 2; do
    if [ "$lib" != default ] && [ $ml = 0 ]; then continue; fi
    for cfg in c3 c2; do
      PCB_MIXED_LAST=$ml python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3a_${cfg}_${tag}_$ml.json 2>gpurun_out/s3a_${cfg}_${tag}_$ml.err
      python -c "import json;d=json.load(open('gpurun_out/s3a_${cfg}_${tag}_$ml.json'));print('$cfg $tag mixed_last=$ml', round(d['value']), round(d['e2e']['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3a_${cfg}_${tag}_$ml.err
    done
  done
done
