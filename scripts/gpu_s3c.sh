#!/bin/bash
# split-3 row engine, second pass: parity, A/B (PCB_MIXED_LAST 0 / 2, CTA-size variants), launch list at mixed_last = 2
mkdir -p gpurun_out
echo "== parity: $(timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2)"
for lib in default build/ab/*.so; do
  if [ "$lib" = default ]; then unset PCB_LIB_PATH; else export PCB_LIB_PATH=$PWD/$lib; fi
  tag=$(basename $lib .so)
  for ml in 0 2; do
    if [ "$lib" != default ] && [ $ml = 0 ]; then continue; fi
    for cfg in c3 c2; do
      PCB_MIXED_LAST=$ml python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3c_${cfg}_${tag}_$ml.json 2>gpurun_out/s3c_${cfg}_${tag}_$ml.err
      python -c "import json;d=json.load(open('gpurun_out/s3c_${cfg}_${tag}_$ml.json'));print('$cfg $tag mixed_last=$ml', round(d['value']), round(d['e2e']['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3c_${cfg}_${tag}_$ml.err
    done
  done
done
unset PCB_LIB_PATH
for ml in 0 2; do
PCB_MIXED_LAST=$ml timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/s3c_launches_$ml.csv python bench.py --config c3 --profile-only --steps 1 --warmup 1 > gpurun_out/s3c_ncu_$ml.log 2>&1
python scripts/launch_share.py gpurun_out/s3c_launches_$ml.csv 2 | head -24
done
