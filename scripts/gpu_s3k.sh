#!/bin/bash
# row passes: 16 elements per thread at 8 / 4 CTAs per SM (erows16b), ascending stage radices (rdesc0)
mkdir -p gpurun_out
run() { tag=$1; cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/s3k_${cfg}_$tag.json 2>gpurun_out/s3k_${cfg}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/s3k_${cfg}_$tag.json'));print('$cfg $tag', round(d['value']), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" || tail -3 gpurun_out/s3k_${cfg}_$tag.err
}
for cfg in c3 c2; do
run base $cfg A=1
for lib in build/ab/*.so; do run $(basename $lib .so) $cfg PCB_LIB_PATH=$PWD/$lib; done
done
