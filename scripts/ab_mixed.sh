#!/bin/bash
# parity + c3/c4 bench of each build/ab variant with and without 3-smooth sizes on the R2C axis
mkdir -p gpurun_out
for lib in default build/ab/*.so; do
  if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
  tag=$(basename $lib .so)
  echo "== $tag parity(mixed): $(PCB_MIXED_LAST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1)"
  for ml in 0 1; do
    for cfg in c3 c2 c4; do
      PCB_MIXED_LAST=$ml python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abm_${cfg}_${tag}_$ml.json 2>/dev/null
      python -c "import json;d=json.load(open('gpurun_out/abm_${cfg}_${tag}_$ml.json'));print('$cfg $tag mixed_last=$ml', round(d['value']), d['config']['fft_size'], {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
    done
  done
done
